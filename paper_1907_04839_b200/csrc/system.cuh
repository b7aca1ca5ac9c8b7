// Host-side engine behind the C ABI: device-resident state, launch plans, the evaluation graph.
// Mirrors HamiltonianSystem<T,D> (shooting.hpp:104-344) and the objective closure
// (registration.cpp:58-74); see include/lmshoot_b200.h for the per-call citations.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lmshoot_b200.h"
#include "nccl_dyn.h"
#include "pair_kernels.cuh"
#include "small_kernels.cuh"

namespace lms {

struct CudaFailure {
  cudaError_t err;
  const char* what;
  int line;
};

#define LMS_CUDA(expr)                                          \
  do {                                                          \
    cudaError_t lms_e_ = (expr);                                \
    if (lms_e_ != cudaSuccess) throw CudaFailure{lms_e_, #expr, __LINE__}; \
  } while (0)

struct StatusError {
  int code;
  const char* msg;
};

constexpr unsigned long long kNotDiverged = ~0ull;
constexpr int kRowAlign = 512;  // planes are padded to a multiple of the largest row tile

// Loopback transport for the row partition: `world` ranks are handles in ONE process (one host thread each,
// typically all on the same GPU).  Same schedule and the same in-place slice layout as the NCCL path; the
// exchange is a rendezvous plus device-to-device copies.  It exists so that a single-GPU box can run the
// partitioned evaluation with world > 1 for real (tests/test_gpu_parity.py::test_row_partition_loopback).
struct LocalGroup {
  explicit LocalGroup(int w) : world(w), lists(w) {}
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  std::vector<std::vector<std::pair<char*, size_t>>> lists;  // per rank: (buffer base, slice bytes)
  bool failed = false;

  void barrier()
  {
    std::unique_lock<std::mutex> lock(m);
    const unsigned long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return generation != gen; });
    }
  }
};

// Abstract interface the C ABI talks to (one concrete System<T,D> per precision x dim).
class SystemBase {
 public:
  virtual ~SystemBase() = default;
  virtual void hamiltonian(const double* q, const double* p, double* out) = 0;
  virtual void derivatives(const double* q, const double* p, double* hq, double* hp) = 0;
  virtual void integrate_forward(const double* q0, const double* p0, int timesteps, double* tq, double* tp) = 0;
  virtual void adjoint_step(const double* q, const double* p, const double* alpha, const double* beta,
                            double* da, double* db) = 0;
  virtual void mismatch_sq(const double* a, const double* b, double* out) = 0;
  virtual void bind(const double* q0, const double* target, double lambda, int timesteps) = 0;
  virtual void eval(const double* x, double* grad, double* scalars, bool device_ptrs) = 0;
  virtual void final_q(double* out) = 0;
  virtual void registration_metrics(double* out) = 0;  // {avg, max} template-target, {avg, max} q(1)-target
  virtual void velocities(const double* q, const double* p, size_t m, const double* pts, double* out) = 0;
  virtual void warp_stored(size_t m, const double* pts, double* out) = 0;
  virtual void comm_init(const unsigned char* id, int rank, int world) = 0;
  virtual void join_local_group(LocalGroup* group, int rank) = 0;
  // peer-push exchange for the row partition (see System::p2p_export)
  virtual void p2p_export(int rank, int world, unsigned char* blob) = 0;
  virtual void p2p_connect(const unsigned char* blobs) = 0;
  // population batches: `count` problems listed in ids (all when ids == nullptr); arrays are full-batch sized
  virtual void eval_batch(const double* x, double* grad, double* scalars, int* diverged_step, int count,
                          const int* ids) = 0;
  virtual void final_q_batch(double* out) = 0;
  virtual cudaStream_t stream_handle() const = 0;
  virtual const double* staging_scratch() const = 0;
  virtual const double* last_x_device() const = 0;  // the point of the last single-problem evaluation (device copy), or null  // device scratch of the host<->plane conversions (trace builds read it)
  int batch = 1;
  // scratch owned by the device-resident L-BFGS driver (device_lbfgs.cu), kept across lms_register_device calls:
  // cudaMalloc / cudaFree cost milliseconds (and synchronise the device) next to an 8 ms evaluation
  std::shared_ptr<void> lbfgs_workspace;

  lms_config cfg{};
  int last_diverged_step = -1;
  long long last_diverged_point = -1;
  std::string last_message;
  std::string kernel_names_;  // "<forward> / <adjoint>" shapes this handle launches
  double last_eval_ms = 0.0;
  int last_eval_launches = 0;
  bool kernel_timing = false;
  double last_kernel_ms[2] = {0.0, 0.0};
  // bound registration (host copies feed lms_register's x0 = (target - q0)/T, registration.cpp:47-52)
  bool bound = false;
  std::vector<double> host_q0, host_target;
  double lambda = 0.0;
  int timesteps = 0;
};

// ---- kernel variants --------------------------------------------------------------------------
template <typename T>
struct KernelChoice {
  void (*fn)(PairArgs<T>) = nullptr;
  void (*fn_cluster)(PairArgs<T>) = nullptr;  // same shape with the cluster combine (small problems), or null
  void (*fn_peers)(PairArgs<T>) = nullptr;    // same shape with the peer-push stores in its epilogues (row partition), or null
  int rows_per_thread = 0;
  void (*fn_thin)(PairArgs<T>) = nullptr;     // same shape with the thin-last-row-tile code (PairArgs::thin_split), or null:
                                              // launched only when the plan has a thin tile, so launches without one
                                              // (other sizes, batches, row partitions) run the kernel they always ran
  const char* name = "";
};

template <typename T, int D, int MODE, int R, int JU, int MINB, bool PACKED = false, int UNR = 1, bool BULK = false,
          bool AOS = false, bool WITH_CLUSTER = false, bool WITH_PEERS = false, bool WITH_THIN = false>
KernelChoice<T> make_choice(const char* name)
{
  KernelChoice<T> c;
  c.fn = pair_kernel<T, D, MODE, R, JU, MINB, PACKED, UNR, BULK, AOS>;
  if constexpr (WITH_THIN) c.fn_thin = pair_kernel<T, D, MODE, R, JU, MINB, PACKED, UNR, BULK, AOS, false, false, true>;
  if constexpr (WITH_CLUSTER) c.fn_cluster = pair_kernel<T, D, MODE, R, JU, MINB, PACKED, UNR, BULK, AOS, true>;
  if constexpr (WITH_PEERS) c.fn_peers = pair_kernel<T, D, MODE, R, JU, MINB, PACKED, UNR, BULK, AOS, false, true>;
  c.rows_per_thread = R;
  c.name = name;
  return c;
}

// variant 0 is the library default; the others exist so one GPU session can A/B them.
template <typename T, int D, int MODE>
KernelChoice<T> pick_kernel(int variant);
// specialised in system_{f32,f64}_d{2,3}.cu
#define LMS_DECLARE_PICKS(T, D)                              \
  template <> KernelChoice<T> pick_kernel<T, D, kFwd>(int);  \
  template <> KernelChoice<T> pick_kernel<T, D, kAdj>(int);  \
  template <> KernelChoice<T> pick_kernel<T, D, kVel>(int);
LMS_DECLARE_PICKS(float, 3)
LMS_DECLARE_PICKS(double, 3)
LMS_DECLARE_PICKS(float, 2)
LMS_DECLARE_PICKS(double, 2)
#undef LMS_DECLARE_PICKS

struct LaunchPlan {
  int grid = 0;
  int n_row_tiles = 0;
  int n_j_tiles = 0;
  int tiles_per_problem = 1;
  int thin_split = 1;  // > 1: the last row tile is thin (PairArgs::thin_split)
  int thin_period = 0; // phantom-cell period of the thin tile (PairArgs::thin_period)
  bool cluster = false;  // launch fn_cluster as clusters of kClusterSize CTAs, one cluster per row tile
  int bm = 0;
  size_t partial_elems = 0;
  int combine_segments = 0;  // partial segments the combine lands in dynamic shared memory per round trip (0: registers)
  size_t dyn_smem = 0;       // dynamic shared memory of the launch (the combine's landing zone)
};

template <typename T, int D>
class System final : public SystemBase {
 public:
  System(const lms_config& c, int batch_count);
  ~System() override;

  void hamiltonian(const double* q, const double* p, double* out) override;
  void derivatives(const double* q, const double* p, double* hq, double* hp) override;
  void integrate_forward(const double* q0, const double* p0, int timesteps, double* tq, double* tp) override;
  void adjoint_step(const double* q, const double* p, const double* alpha, const double* beta, double* da,
                    double* db) override;
  void mismatch_sq(const double* a, const double* b, double* out) override;
  void bind(const double* q0, const double* target, double lambda, int timesteps) override;
  void eval(const double* x, double* grad, double* scalars, bool device_ptrs) override;
  void final_q(double* out) override;
  void registration_metrics(double* out) override;
  void velocities(const double* q, const double* p, size_t m, const double* pts, double* out) override;
  void warp_stored(size_t m, const double* pts, double* out) override;
  void comm_init(const unsigned char* id, int rank, int world) override;
  void join_local_group(LocalGroup* group, int rank) override;
  void p2p_export(int rank, int world, unsigned char* blob) override;
  void p2p_connect(const unsigned char* blobs) override;
  void eval_batch(const double* x, double* grad, double* scalars, int* diverged_step, int count,
                  const int* ids) override;
  void final_q_batch(double* out) override;
  cudaStream_t stream_handle() const override { return stream_; }
  const double* staging_scratch() const override { return d_io_; }
  const double* last_x_device() const override { return stored_t_ == timesteps && bound && d_x_current_ ? d_x_ : nullptr; }

 private:
  static constexpr int kState = 2 * D;  // planes per (q,p) or (alpha,beta) state

  T* snapshot(int t) const { return traj_ + (long long)t * kState * stride_; }
  int n() const { return (int)cfg.n; }

  template <int MODE>
  LaunchPlan plan_for(const KernelChoice<T>& k, int n_rows, int row_tile0 = -1, int row_tiles = -1,
                      int batch_count = 1);
  template <int MODE>
  void launch(const KernelChoice<T>& k, PairArgs<T> a, const LaunchPlan& plan);
  void alloc_partials();
  PairArgs<T> base_args() const;

  void upload(const double* host, T* planes, long long stride, int count, int ncomp, bool check, int step,
              int batch_count = 1, long long dst_bs = 0);
  void download(const T* planes, long long stride, double* host, int count, int ncomp);
  void reset_diverged();
  void read_diverged_or_throw();
  void sync() { LMS_CUDA(cudaStreamSynchronize(stream_)); }
  void enqueue_eval(bool timed, int count = -1, const int* d_ids = nullptr);
  void require_single(const char* what) const;
  void destroy_graph();
  void ensure_points(size_t m);
  void all_gather_state(T* state_planes);
  void all_gather_doubles(double* buf);
  void gather_inplace(const std::vector<std::pair<char*, size_t>>& buffers);
  void relayout_for_world(int world, int rank);
  void pick_kernels(bool partitioned);
  void alloc_exchange_arena();
  void plan_small();
  void launch_small(bool host_io = false);
  void p2p_exchange();
  void p2p_disconnect();

  cudaStream_t stream_ = nullptr;
  int num_sms_ = 0;
  // programmatic dependent launch between the pair kernels (see the constructor): on for single unpartitioned
  // problems of 2400 to 8000 landmarks since round 2 (a loss in round 1, when the kernels were 4-5 x larger); LMS_PDL overrides
  bool pdl_ = false;
  // cluster combine for small single problems (pair_kernel<..., CLUSTER>): opt-in with LMS_CLUSTER=1.  It is worth
  // 8-12 % below N = 1500 in fp32 (plan_for), but it changes the summation order of those sizes (the partitioned and
  // unpartitioned paths then no longer agree bit for bit) and must stay off for several ranks on one GPU.
  bool cluster_combine_ = false;
  long long stride_ = 0;
  long long row_align_ = kRowAlign;  // plane padding: lcm of kRowAlign and the row tiles in use
  long long bs_traj_ = 0;   // elements between consecutive problems' trajectories
  long long bs_state_ = 0;  // ... between their (alpha,beta) states
  long long bs_vec_ = 0;    // ... between their D-plane vectors (hp0, target, q0)
  int max_t_ = 0;
  int* d_ids_ = nullptr;
  T inv_sig2_{}, kexp_{};

  KernelChoice<T> k_fwd_, k_adj_, k_vel_;

  T* traj_ = nullptr;
  T* adj_[2] = {nullptr, nullptr};
  T* hp0_ = nullptr;
  T* target_ = nullptr;
  T* q0_ = nullptr;
  T* scratch_in_ = nullptr;
  T* scratch_out_ = nullptr;
  T* points_[2] = {nullptr, nullptr};
  size_t points_cap_ = 0;
  long long points_stride_ = 0;
  T* partials_ = nullptr;
  size_t partials_cap_ = 0;
  int* counters_ = nullptr;
  int counters_cap_ = 0;
  double* h_part_ = nullptr;
  double* mm_part_ = nullptr;
  int part_tiles_ = 0;
  double* d_scalars_ = nullptr;
  unsigned long long* d_diverged_ = nullptr;
  double* d_io_ = nullptr;  // 4 x (n*D) doubles of conversion staging
  double* d_x_ = nullptr;
  bool d_x_current_ = false;  // d_x_ holds the point of the last evaluation (not after a zero-copy host-buffer call)
  double* d_grad_ = nullptr;
  double* h_scalars_ = nullptr;  // pinned: 3 doubles + the divergence word
  double* d_metrics_ = nullptr;  // registration_metrics: {avg, max} before and after
  size_t io_cap_ = 0;

  // bound problem
  T dt_{}, two_lambda_{};
  bool q0_bad_ = false;
  std::vector<char> q0_bad_problem_;
  bool traj0_is_q0_ = false;
  int stored_t_ = -1;  // timesteps of the trajectory currently in traj_ (-1: none)
  int final_adj_ = 0;  // which adj_ buffer holds (alpha_0, beta_0) after an eval
  LaunchPlan plan_fwd_, plan_adj_;
  cudaGraphExec_t graph_ = nullptr;
  int graph_launches_ = 0;
  std::vector<cudaEvent_t> events_;
  cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr;

  // small single problems: the whole evaluation as one persistent cooperative kernel (small_kernels.cuh)
  bool small_enabled_ = true;     // LMS_SMALL=0 pins the tiled path
  int small_max_n_ = 0;           // largest n the persistent kernel is chosen for (LMS_SMALL_MAX_N)
  bool use_small_ = false;        // decided at bind
  int small_grid_ = 0, small_threads_ = 0;
  int small_cluster_ = 1, small_grid_cap_ = 0;  // thread-block cluster size sharing the state fetch (TMA multicast)
  unsigned small_bar_count_ = 0;  // arrivals the barrier counter has seen so far (host-side mirror)
  size_t small_smem_ = 0;
  void (*small_fn_)(SmallArgs<T>) = nullptr;
  double* warp_part_ = nullptr;   // 2 x (SMs x kSmallMaxWarps) per-row-warp scalar partials
  unsigned* small_bar_ = nullptr; // grid barrier: monotonic arrival counter
  double* h_zc_ = nullptr;        // mapped pinned x | grad | {loss, kinetic, mismatch, divergence word}: the persistent kernel reads and
                                  // writes the host-buffer call's operands in place (no staging copies, no copy launches)

  // row partition (multi-GPU)
  int rank_ = 0, world_ = 1;
  bool comm_active_ = false;
  ncclComm_t comm_ = nullptr;
  LocalGroup* local_ = nullptr;
  // Every buffer a peer may write lives in ONE allocation (traj_, adj_[0..1], d_grad_, h_part_, mm_part_, flags),
  // so a peer's address of any of them is the local address plus one byte distance per peer.
  char* arena_ = nullptr;
  size_t arena_bytes_ = 0;
  unsigned* p2p_flags_ = nullptr;            // [world]: slot r holds the last epoch rank r announced to this rank
  unsigned long long* div_all_ = nullptr;    // [world]: every rank's divergence word of the running evaluation
  bool p2p_active_ = false;
  bool p2p_dirty_ = false;                   // a pair kernel ran since the last flag exchange
  unsigned p2p_epoch_ = 0;
  int n_peers_ = 0;
  int peer_rank_[kMaxPeers] = {};
  long long peer_delta_[kMaxPeers] = {};
  void* peer_mapping_[kMaxPeers] = {};       // cudaIpcOpenMemHandle results (other processes), else nullptr
  int row_tile_begin_(int bm) const;
  int row_tile_end_(int bm) const;
};

// What lms_p2p_export hands to the peers (LMS_P2P_BLOB_BYTES = 128 in the C ABI).
struct P2PBlob {
  unsigned long long magic;
  long long pid;
  int device, rank, world, pad;
  unsigned long long base;   // the exporting process's address of its arena
  unsigned long long bytes;
  cudaIpcMemHandle_t handle; // 64 bytes
};
static_assert(sizeof(P2PBlob) <= 128, "blob must fit the ABI's buffer");

struct RowPartition {
  long long slice = 0;      // rows per rank (multiple of kRowAlign), identical on every rank
  long long stride = 0;     // padded plane length = slice * world
  long long row_begin = 0;  // live rows owned by this rank: [row_begin, row_end)
  long long row_end = 0;
};
RowPartition partition_rows(long long n, int world, int rank);

SystemBase* create_system(const lms_config& cfg, int batch_count = 1);
// device_lbfgs.cu: allocates (once per handle) and warms the workspace of lms_register_device
void prepare_device_lbfgs(SystemBase* sys, int memory);
const char* variant_name(int precision, int variant);

}  // namespace lms
