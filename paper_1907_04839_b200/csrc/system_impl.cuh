// System<T,D>: member definitions.  Included by the four per-instantiation translation units
// (system_f32_d3.cu, system_f64_d3.cu, system_f32_d2.cu, system_f64_d2.cu) so that they compile in parallel.
#pragma once
#include "system.cuh"

#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace lms {

// Phantom-cell period of a thin tile (one cell in `period` sweeps nothing), by kernel mode and split: the cost of a
// thin cell over a full one is the per-staged-tile overhead spread over 1/split of the work, larger for the forward
// kernel (TMA-staged tiles, 8 columns per unrolled iteration) than for the adjoint (measured: DESIGN.md §3).
// Measured at N = 20 000 (ms per launch; full table in DESIGN.md §3): forward, 4 groups, period 9 / 7 / 5 / 4 / 3: 0.2464 /
// 0.2450 / 0.2428 / 0.2429 / 0.2456; adjoint, 4 groups, none / 13 / 9 / 5: 0.5555 / 0.5436 / 0.5439 / 0.5445; adjoint swept
// 8 ways, period 9 / 5 / 3 / 2: 0.5452 / 0.5425 / 0.5437 / 0.5436; forward swept 8 ways, period 2: 0.2429 (no better than 4).
inline int thin_period_default(int mode, int split)
{
  if (mode == kFwd) return split >= 8 ? 2 : 5;
  return split >= 8 ? 5 : 9;
}

// Sweeping a thin tile 8 ways (pair split) pays in the adjoint kernel only (see the table above).
inline bool thin8_enabled(int mode)
{
  static const int knob = [] {
    const char* e = std::getenv("LMS_THIN8");  // experiment knob: 0 = at most 4 ways, 1 = forward and adjoint
    return e ? std::atoi(e) : -1;
  }();
  return knob >= 0 ? knob != 0 : mode == kAdj;
}

inline bool thin_enabled()
{
  static const bool on = [] {
    const char* e = std::getenv("LMS_THIN");  // experiment knob: 0 keeps every row tile a full tile
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}


namespace {

inline long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }
inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

template <typename T>
T* dev_alloc_zero(size_t count)
{
  T* p = nullptr;
  LMS_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  LMS_CUDA(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)));
  return p;
}

template <typename T>
void dev_free(T*& p)
{
  if (p) cudaFree(p);
  p = nullptr;
}

}  // namespace

// ---- construction ------------------------------------------------------------------------------------
#ifdef LMS_TIME_CTOR  // measurement builds: where the handle's construction time goes
inline std::chrono::steady_clock::time_point& ctor_prev() { static std::chrono::steady_clock::time_point t; return t; }
#define LMS_CTOR_T(i) do { auto t_now = std::chrono::steady_clock::now(); if ((i) == 0) ctor_prev() = t_now; std::fprintf(stderr, "ctor %d: +%.3f ms\n", (i), std::chrono::duration<double, std::milli>(t_now - ctor_prev()).count()); ctor_prev() = t_now; } while (0)
#else
#define LMS_CTOR_T(i) do {} while (0)
#endif
template <typename T, int D>
System<T, D>::System(const lms_config& c, int batch_count)
{
  cfg = c;
  batch = std::max(batch_count, 1);
  LMS_CTOR_T(0);
  LMS_CUDA(cudaSetDevice(c.device));
  // (two attribute queries instead of cudaGetDeviceProperties: that call alone took 2.4 ms of a 5.6 ms construction)
  int cc_major = 0;
  LMS_CUDA(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, c.device));
  if (cc_major != 10) throw StatusError{LMS_ERR_CUDA, "device is not sm_100 (B200); no fallback path exists"};
  LMS_CUDA(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, c.device));
  LMS_CTOR_T(1);
  // Programmatic dependent launch between the 2T dependent launches of an evaluation: the next kernel's CTAs are
  // scheduled, and run their prologue up to griddepcontrol.wait, while the previous kernel drains.  Measured on B200
  // (ms per gradient, T = 10, without / with): fp32 N = 4500 0.647 / 0.625, 6000 0.965 / 0.947, 8000 1.509 / 1.506,
  // 20 000 7.93 / 7.95; fp64 N = 3000 0.735 / 0.715, 5000 1.620 / 1.602, 10 000 5.708 / 5.693 -- but a LOSS around
  // N = 1500-2000, where the tiled path is not the default anyway (fp32 2000: 0.244 / 0.285, fp64 2000: 0.429 / 0.637).
  // On for single unpartitioned problems of 2400 to 8000 landmarks (LMS_PDL=0/1 overrides).
  pdl_ = batch == 1 && c.n >= 2400 && c.n < 8000;
  if (const char* e = std::getenv("LMS_PDL")) pdl_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("LMS_CLUSTER")) cluster_combine_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("LMS_SMALL")) small_enabled_ = std::atoi(e) != 0;
  if (c.flags & LMS_FLAG_TILED_ONLY) small_enabled_ = false;
  small_max_n_ = sizeof(T) == 4 ? kSmallMaxN32 : kSmallMaxN64;
  if (const char* e = std::getenv("LMS_SMALL_MAX_N")) small_max_n_ = std::atoi(e);
  LMS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  LMS_CUDA(cudaEventCreate(&ev_begin_));
  LMS_CUDA(cudaEventCreate(&ev_end_));
  LMS_CTOR_T(2);

  // Constants rounded as the reference rounds them (shooting.hpp:63-68,114-115).
  inv_sig2_ = T(1) / (T(c.sigma) * T(c.sigma));
  const T k_scale = T(-0.5) * inv_sig2_;
  if constexpr (sizeof(T) == 4)
    kexp_ = (T)((double)k_scale * 1.4426950408889634074);  // ex2.approx: exp(x) = 2^(x log2 e)
  else
    kexp_ = (T)((long double)k_scale * 1.44269504088896340735992468100189214L * (long double)kExpEntries);  // Math<double>::kernel

  // Variant 0 picks the shapes by problem size: from N = 16 000 on (single problems, fp32, D = 3) four rows per
  // thread with column-major tiles -- 2-3.5 % faster there (N = 20 000: 8.05 vs 8.22 ms, N = 100 000: 190.8 vs
  // 197.6 ms per gradient, same session), but twice the row-tile size, which mid-size and batched problems pay
  // for in parallelism.  Variant 11 pins the two-row shapes for A/B.
  pick_kernels(/*partitioned=*/false);
  LMS_CTOR_T(3);

  max_t_ = std::max(c.max_timesteps, 1);
  const long long N = (long long)c.n;
  stride_ = std::max<long long>(round_up(N, row_align_), row_align_);
  const size_t plane = (size_t)stride_;
  const size_t B = (size_t)batch;
  bs_traj_ = (long long)(max_t_ + 1) * kState * stride_;
  bs_state_ = (long long)kState * stride_;
  bs_vec_ = (long long)D * stride_;
  hp0_ = dev_alloc_zero<T>(B * D * plane);
  target_ = dev_alloc_zero<T>(B * D * plane);
  q0_ = dev_alloc_zero<T>(B * D * plane);
  scratch_in_ = dev_alloc_zero<T>(2 * kState * plane);
  scratch_out_ = dev_alloc_zero<T>(kState * plane);
  d_scalars_ = dev_alloc_zero<double>(4 * B);
  d_diverged_ = reinterpret_cast<unsigned long long*>(d_scalars_ + 3);
  d_metrics_ = dev_alloc_zero<double>(4);
  io_cap_ = (size_t)N * D * B;
  d_io_ = dev_alloc_zero<double>(4 * io_cap_);
  d_x_ = dev_alloc_zero<double>(std::max((size_t)stride_ * D, B * (size_t)N * D));
  d_ids_ = dev_alloc_zero<int>(B);
  LMS_CTOR_T(4);
  // one pinned (mapped) allocation: the scalar records of every problem, and -- single problems -- x | grad | scalars
  // for the persistent kernel's zero-copy host-buffer calls (a pinned allocation costs 1-2.5 ms: one, not two)
  {
    const size_t zc = (B == 1 && small_enabled_ && N <= (long long)small_max_n_) ? 2 * (size_t)N * D + 4 : 0;
    LMS_CUDA(cudaHostAlloc(&h_scalars_, (4 * B + zc) * sizeof(double), cudaHostAllocMapped));
    h_zc_ = zc ? h_scalars_ + 4 * B : nullptr;
  }
  LMS_CTOR_T(5);
  part_tiles_ = (int)(stride_ / kThreads);
  warp_part_ = dev_alloc_zero<double>((size_t)2 * num_sms_ * kSmallMaxWarps);
  small_bar_ = dev_alloc_zero<unsigned>(64);
  alloc_exchange_arena();
  LMS_CTOR_T(6);
  alloc_partials();
  LMS_CTOR_T(7);
}

// Variant 0 picks the shapes by problem size.  From N = 16 000 on (fp32) four rows per thread pay (variant 25;
// variant 9 is the same with the forward tiles staged through registers and the column loop not unrolled: forward
// launch 0.258 -> 0.247 ms at N = 20 000): every staged column tile and every broadcast LDS serves twice the pairs (N = 20 000: 8.22 -> 8.05 ms,
// N = 100 000: 197.6 -> 190.8 ms per gradient, same session).  Larger row tiles cost parallelism at mid size and in
// batches (those keep R = 2, variant 11).  Six or eight rows per thread (variants 12-14) are another 0.8 % faster per
// pair but lose it again to row-tile quantisation -- a mostly padded last tile costs a full tile: 27 tiles of 768
// rows for N = 20 000 waste 3.6 %, 40 tiles of 512 waste 2.3 % -- and do not divide the row partition's slices.
template <typename T, int D>
void System<T, D>::pick_kernels(bool partitioned)
{
  int variant = cfg.variant;
  // (populations: the same shapes once the batch as a whole is that large -- 128 x N = 2000: 10.81 -> 10.49 ms)
  // Single problems: four rows per thread are 1-2 % faster per gradient from N ~ 10 500 on and 3-4 % from 16 000 on, but their
  // 512-row tiles pad more (N = 11 000: 2.4 % against 0.07 % for 256-row tiles).  Padding-aware: take them when the
  // gain exceeds the extra padding (measured on B200, scripts/gpu_thresh.py: R = 4 / R = 2 ratio 0.98-0.99 at
  // N = 8000-15 000 except 1.014 at 11 000; 1.01-1.13 below 8000 -- before the thin last tile; with it see below).
  // Padding of the last row tile, counted as what it costs: a mostly padded tile is swept as a thin tile (plan_for: a
  // quarter or half of a tile's units plus one phantom cell in nine) by the shapes that have that instantiation.
  auto padding = [&](long long bm, bool thin) {
    const long long tiles = ceil_div((long long)cfg.n, bm), live = (long long)cfg.n - (tiles - 1) * bm;
    const double last = !(thin && thin_enabled()) ? (double)bm
                        : (live * 8 <= bm && bm == 4 * kThreads) ? bm * 0.21   /* between the forward's 4 and the adjoint's 8 ways */
                        : live * 4 <= bm ? bm * 0.28125 : (live * 2 <= bm ? bm * 0.5625 : (double)bm);
    return ((double)((tiles - 1) * bm) + last) / (double)std::max(cfg.n, (size_t)1) - 1.0;
  };
  const bool thin2 = pick_kernel<T, D, kFwd>(0).fn_thin != nullptr, thin4 = pick_kernel<T, D, kFwd>(25).fn_thin != nullptr;
  const double gain4 = cfg.n >= 16000 ? 0.035 : 0.015;
  // (scripts/gpu_thin.py, B200: with the thin last tile the four-row shapes win from N ~ 10 800 on -- ratio to the
  // two-row shapes 0.978-0.997 at N = 10 800 ... 15 400 -- and lose below 10 300: 1.005-1.027)
  bool large = batch == 1 ? (cfg.n >= 10500 && padding(4 * kThreads, thin4) - padding(2 * kThreads, thin2) < gain4)
                          : (cfg.n >= 1024 && (long long)batch * (long long)cfg.n >= 32000);
  if (const char* e = std::getenv("LMS_FORCE_ROWS")) large = std::atoi(e) == 4;  // experiment knob: 2 or 4 rows per thread
  if (variant == 0 && sizeof(T) == 4 && large) variant = 25;
  k_fwd_ = pick_kernel<T, D, kFwd>(variant);
  k_adj_ = pick_kernel<T, D, kAdj>(variant);
  k_vel_ = pick_kernel<T, D, kVel>(cfg.variant);
  kernel_names_ = std::string(k_fwd_.name) + " / " + k_adj_.name;
  // planes are padded to a whole number of the largest row tile (and of kRowAlign)
  long long align = kRowAlign;
  const int rows_per_thread[3] = {k_fwd_.rows_per_thread, k_adj_.rows_per_thread, k_vel_.rows_per_thread};
  for (int r : rows_per_thread) {
    const long long bm = (long long)kThreads * r;
    align = align / std::__gcd(align, bm) * bm;
  }
  if (partitioned && align != kRowAlign)
    throw StatusError{LMS_ERR_INVALID, "this kernel variant's row tile does not divide the row partition's slices"};
  row_align_ = align;
}

// traj_, adj_[0..1], d_grad_, h_part_, mm_part_ and the exchange flags in one allocation (see p2p_export).
template <typename T, int D>
void System<T, D>::alloc_exchange_arena()
{
  const size_t B = (size_t)batch;
  const size_t plane = (size_t)stride_;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b_traj = up(B * (size_t)bs_traj_ * sizeof(T));
  const size_t b_adj = up(B * kState * plane * sizeof(T));
  const size_t b_grad = up(std::max(plane * D, B * (size_t)cfg.n * D) * sizeof(double));
  const size_t b_part = up(B * (size_t)part_tiles_ * sizeof(double));
  const size_t b_flags = 256 + kMaxRanks * sizeof(unsigned long long);  // arrival flags, per-rank divergence words
  arena_bytes_ = b_traj + 2 * b_adj + b_grad + 2 * b_part + b_flags;
  arena_ = dev_alloc_zero<char>(arena_bytes_);
  char* p = arena_;
  traj_ = reinterpret_cast<T*>(p);            p += b_traj;
  adj_[0] = reinterpret_cast<T*>(p);          p += b_adj;
  adj_[1] = reinterpret_cast<T*>(p);          p += b_adj;
  d_grad_ = reinterpret_cast<double*>(p);     p += b_grad;
  h_part_ = reinterpret_cast<double*>(p);     p += b_part;
  mm_part_ = reinterpret_cast<double*>(p);    p += b_part;
  p2p_flags_ = reinterpret_cast<unsigned*>(p);
  div_all_ = reinterpret_cast<unsigned long long*>(p + 256);
}

template <typename T, int D>
System<T, D>::~System()
{
  cudaSetDevice(cfg.device);
  if (stream_) cudaStreamSynchronize(stream_);
  destroy_graph();
  if (comm_ && nccl_api().ok) nccl_api().CommDestroy(comm_);
  p2p_disconnect();
  dev_free(arena_);
  dev_free(hp0_);
  dev_free(target_);
  dev_free(q0_);
  dev_free(scratch_in_);
  dev_free(scratch_out_);
  dev_free(points_[0]);
  dev_free(points_[1]);
  dev_free(partials_);
  dev_free(counters_);
  dev_free(warp_part_);
  dev_free(small_bar_);
  dev_free(d_scalars_);
  dev_free(d_metrics_);
  dev_free(d_io_);
  dev_free(d_x_);
  dev_free(d_ids_);
  if (h_scalars_) cudaFreeHost(h_scalars_);  // h_zc_ lives in the same allocation
  for (auto e : events_) cudaEventDestroy(e);
  if (ev_begin_) cudaEventDestroy(ev_begin_);
  if (ev_end_) cudaEventDestroy(ev_end_);
  if (stream_) cudaStreamDestroy(stream_);
}

template <typename T, int D>
void System<T, D>::destroy_graph()
{
  if (graph_) cudaGraphExecDestroy(graph_);
  graph_ = nullptr;
}

// ---- launch planning -----------------------------------------------------------------------------------
template <typename T, int D>
int System<T, D>::row_tile_begin_(int bm) const
{
  const long long slice = stride_ / world_;  // rows per rank, a multiple of kRowAlign
  return (int)(rank_ * slice / bm);
}

template <typename T, int D>
int System<T, D>::row_tile_end_(int bm) const
{
  const long long slice = stride_ / world_;
  const int live_tiles = ceil_div((long long)cfg.n, bm);
  if (world_ == 1) return live_tiles;  // row tiles need not divide the padded plane length when nothing is sliced
  return std::min<int>((int)((rank_ + 1) * slice / bm), live_tiles);
}

template <typename T, int D>
template <int MODE>
LaunchPlan System<T, D>::plan_for(const KernelChoice<T>& k, int n_rows, int row_tile0, int row_tiles,
                                  int batch_count)
{
  LaunchPlan p;
  p.bm = kThreads * k.rows_per_thread;
  p.tiles_per_problem = std::max(row_tiles >= 0 ? row_tiles : ceil_div(n_rows, p.bm), 1);
  p.n_row_tiles = (row_tiles >= 0 ? row_tiles : ceil_div(n_rows, p.bm)) * batch_count;
  p.n_j_tiles = ceil_div((long long)cfg.n, kTileJ);
  const long long units_per_row = (long long)p.n_j_tiles * kUnitsPerTile;  // work units, see pair_kernel
  // Thin last row tile.  A row tile that is mostly padding used to cost a full tile (2.3 % of a launch at N = 20 000
  // with 512-row tiles: 40 tiles for 39.06 tiles' worth of rows).  When its live rows fit the threads of a quarter (or
  // half) of the CTA, those rows are replicated over 4 (2) groups of warps, each group sweeping a quarter (half) of
  // every staged column tile, and the tile counts a quarter (half) of a tile's work units (pair_kernel, `thin`).
  // Every warp stays busy, so -- unlike an earlier attempt that let the dead warps of that tile idle and found a
  // CTA's time set by its busiest warp -- the tile's cost really shrinks.  Single problems on one GPU only.
  const bool thin_on = thin_enabled();
  const bool all_rows = row_tiles < 0 || (row_tile0 == 0 && row_tiles == ceil_div(n_rows, p.bm));
  if (thin_on && k.fn_thin != nullptr && all_rows && batch_count == 1 && !comm_active_ && !cluster_combine_ && p.n_row_tiles >= 1) {
    const long long live_last = (long long)n_rows - (long long)(p.n_row_tiles - 1) * p.bm;
    if (live_last * 8 <= p.bm && k.rows_per_thread == 4 && thin8_enabled(MODE)) p.thin_split = 8;  // pair split (pair_kernel)
    else if (live_last * 4 <= p.bm) p.thin_split = 4;
    else if (live_last * 2 <= p.bm) p.thin_split = 2;
  }
  // A thin tile's units cost a few per cent more than a full tile's (a whole column tile is staged and waited for per
  // 1/thin_split of the work), and stream-K hands every CTA the same number of cells: one cell in `thin_period` of that
  // tile is a phantom, so its CTAs do not finish last (measured).
  static const int thin_period_knob = [] {
    // experiment knobs: LMS_THIN_PERIOD (all modes) or LMS_THIN_PERIOD_FWD / _ADJ; 0 = no phantom cells, -1 = default
    const char* e = std::getenv(MODE == kFwd ? "LMS_THIN_PERIOD_FWD" : (MODE == kAdj ? "LMS_THIN_PERIOD_ADJ" : "LMS_THIN_PERIOD_VEL"));
    if (!e) e = std::getenv("LMS_THIN_PERIOD");
    return e ? std::max(std::atoi(e), 0) : -1;
  }();
  const int thin_period = thin_period_knob >= 0 ? thin_period_knob : thin_period_default(MODE, p.thin_split);
  if (p.thin_split > 1 && thin_period > 1) p.thin_period = thin_period;
  const long long thin_units = units_per_row / p.thin_split;
  const long long thin_cells = thin_units + (p.thin_period > 1 ? thin_units / (p.thin_period - 1) : 0);
  const long long cells = (long long)p.n_row_tiles * units_per_row - (units_per_row - thin_cells);
  if (cells <= 0) return p;
  const auto fn_launched = p.thin_split > 1 ? k.fn_thin : k.fn;  // see launch()
  int per_sm = 0;
  LMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn_launched, kThreads, 0));
  per_sm = std::max(per_sm, 1);
  static const int cap_per_sm = [] {
    const char* e = std::getenv("LMS_CTAS_PER_SM");  // experiment knob: cap on resident CTAs per SM
    return e ? std::max(std::atoi(e), 1) : 1 << 20;
  }();
  per_sm = std::min(per_sm, cap_per_sm);
  const long long full = (long long)num_sms_ * per_sm;
  // Never more CTAs than staged tiles: a CTA sweeps at least one full tile's worth of columns.  (Measured:
  // going finer -- 32 columns per CTA -- makes N = 1000..2000 slower, 0.30 -> 0.43 ms and 0.35 -> 0.88 ms per
  // gradient: the partial-slot write / fence / counter / re-read chain costs more than the extra parallelism.)
  static const int min_units = [] {
    const char* e = std::getenv("LMS_MIN_UNITS");  // experiment knob: work units (8 columns) a CTA sweeps at least
    return e ? std::max(std::atoi(e), 1) : kUnitsPerTile;
  }();
  // ... except when even that leaves half the SMs idle: then half tiles (N = 1000: 0.231 -> 0.194 ms per gradient,
  // N = 1500: 0.241 -> 0.221 ms; from N = 2000 on whole tiles are faster again, 0.248 vs 0.304 ms).
  const long long tiles = cells / kUnitsPerTile;
  const int units = (min_units == kUnitsPerTile && 2 * tiles <= num_sms_) ? kUnitsPerTile / 2 : min_units;
  p.grid = (int)std::min<long long>(full, std::max<long long>(cells / units, 1));
  // The last CTA of a row tile adds that tile's grid / n_row_tiles partial segments one after the other (an L2
  // round trip per few segments).  Measured on B200 (N = 5000: 0.795 -> 0.727 ms, N = 7000: 1.240 -> 1.213 ms per
  // gradient): beyond ~20 segments the serial chain costs more than the occupancy it buys, down to 2 CTAs per SM
  // (N = 20 000 runs only 3.5 % slower at 3 CTAs per SM than at 7).
  static const int seg_cap = [] {
    // experiment knobs: partial segments per row tile at most (LMS_SEG_CAP, or per kernel mode LMS_SEG_CAP_FWD / _ADJ / _VEL)
    const char* mode_knob = MODE == kFwd ? "LMS_SEG_CAP_FWD" : (MODE == kAdj ? "LMS_SEG_CAP_ADJ" : "LMS_SEG_CAP_VEL");
    const char* e = std::getenv(mode_knob);
    if (!e) e = std::getenv("LMS_SEG_CAP");
    return e ? std::max(std::atoi(e), 1) : 20;
  }();
  static const int seg_floor = [] {
    const char* e = std::getenv("LMS_SEG_FLOOR_CTAS_PER_SM");  // experiment knob: never fewer CTAs per SM than this
    return e ? std::max(std::atoi(e), 1) : 2;
  }();
  p.grid = (int)std::min<long long>(p.grid, std::max<long long>((long long)seg_floor * num_sms_, (long long)seg_cap * p.n_row_tiles));
  // mid-size problems: a whole number of CTAs per SM, so no SM carries one CTA more than its neighbours
  static const int round_from = [] {
    const char* e = std::getenv("LMS_ROUND_FROM");  // experiment knob: round only grids of at least this many CTAs per SM
    return e ? std::max(std::atoi(e), 1) : 1;
  }();
  if (p.grid < full && p.grid > (long long)round_from * num_sms_) p.grid -= p.grid % num_sms_;
  // partial slots are indexed by CTA (two per CTA, see the combine in pair_kernel): the buffers allocated by
  // alloc_partials() cover the fullest grid any kernel of this handle can be launched with
  constexpr int NA = Shape<MODE, D>::kAcc;
  p.partial_elems = (size_t)2 * p.grid * NA * p.bm;
  // Small single problems: one cluster of kClusterSize CTAs per row tile, partial sums combined in distributed
  // shared memory (pair_kernel<..., CLUSTER>).  Every CTA sweeps n_j_tiles work units (units_per_row / 16).
  // Measured on B200, fp32, ms per gradient with / without: N = 500 0.151 / 0.172, N = 1000 0.181 / 0.197, N = 1500
  // 0.213 / 0.217; from 8 clusters on they no longer fit the GPCs at once (N = 2000: 0.323 / 0.243), and fp64 gains
  // nothing (0.310 / 0.313), so: fp32, at most 6 row tiles.
  // Not for row-partitioned handles: with several ranks on one GPU a cluster launch of one rank can queue behind
  // another rank's stream-ordered wait for that very launch (observed as a hang of the in-process peer-push test).
  if (cluster_combine_ && !comm_active_ && k.fn_cluster != nullptr && batch_count == 1 && p.n_row_tiles >= 1 &&
      p.n_row_tiles <= 6) {
    p.cluster = true;
    p.grid = p.n_row_tiles * kClusterSize;
  }
  // Mid-size single problems run at most two CTAs per SM (segment cap above), which leaves ~100 KB of shared memory
  // per CTA unused: the last CTA of a row tile lands the tile's partial segments there with bulk-async copies -- a
  // whole batch per L2 round trip instead of four segments per round trip through registers -- and adds them in the
  // same order (bitwise the same sums).  ncu at N = 5000: the serial combine is a 5.6 us tail of a 30 us forward launch.
  // Measured on B200, ms per gradient without / with: fp32 N = 4500 0.622 / 0.610, 5000 0.722 / 0.705, 7000 1.191 / 1.191;
  // fp64 unchanged (3000: 0.717 / 0.717) -- most of that tail is the fence / arrival chain, not the segment loads.
  static const bool combine_smem_on = [] {
    const char* e = std::getenv("LMS_COMBINE_SMEM");  // experiment knob: 0 keeps the register path
    return e ? std::atoi(e) != 0 : true;
  }();
  if (combine_smem_on && !p.cluster && !comm_active_ && batch_count == 1 && p.grid <= 2 * num_sms_ && p.n_row_tiles >= 1) {
    cudaFuncAttributes attr;
    LMS_CUDA(cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(fn_launched)));
    const size_t seg_bytes = (size_t)NA * p.bm * sizeof(T);
    const size_t per_sm = 227 * 1024;
    const long long budget = (long long)(per_sm / 2) - (long long)attr.sharedSizeBytes - 2048;  // two CTAs per SM
    const int max_segs = ceil_div(p.grid, p.n_row_tiles) + 1;
    const int fit = budget > 0 ? (int)(budget / (long long)seg_bytes) : 0;
    const int segs = std::min(max_segs, fit);
    if (segs > kCombineUnroll) {  // otherwise the register path moves as many segments per round trip
      int occ = 0;
      const size_t dyn = (size_t)segs * seg_bytes;
      LMS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn_launched), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)dyn));
      LMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn_launched, kThreads, dyn));
      if ((long long)occ * num_sms_ >= p.grid) {
        p.combine_segments = segs;
        p.dyn_smem = dyn;
      }
    }
  }
  return p;
}

// Stream-K partial slots and arrival counters, sized ONCE for the fullest grid (SMs x resident CTAs) of the
// kernels this handle launches: the captured evaluation graph holds these pointers, and subsets of a batch or
// velocity fields with many more points than landmarks must never force a reallocation or outgrow them.
template <typename T, int D>
void System<T, D>::alloc_partials()
{
  sync();
  dev_free(partials_);
  dev_free(counters_);
  size_t elems = 0;
  int grid_max = 0;
  auto account = [&](const KernelChoice<T>& k, int na) {
    int per_sm = 0;
    LMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, kThreads, 0));
    if (k.fn_thin != nullptr) {
      int per_sm_thin = 0;
      LMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_thin, k.fn_thin, kThreads, 0));
      per_sm = std::max(per_sm, per_sm_thin);
    }
    const int full = num_sms_ * std::max(per_sm, 1);
    grid_max = std::max(grid_max, full);
    elems = std::max(elems, (size_t)2 * full * na * kThreads * k.rows_per_thread);
  };
  account(k_fwd_, Shape<kFwd, D>::kAcc);
  account(k_adj_, Shape<kAdj, D>::kAcc);
  account(k_vel_, Shape<kVel, D>::kAcc);
  partials_ = dev_alloc_zero<T>(elems);
  partials_cap_ = elems;
  counters_ = dev_alloc_zero<int>(grid_max);
  counters_cap_ = grid_max;
}

template <typename T, int D>
PairArgs<T> System<T, D>::base_args() const
{
  PairArgs<T> a{};
  a.jstride = stride_;
  a.istride = stride_;
  a.ostride = stride_;
  a.n_cols = n();
  a.n_rows = n();
  a.row_tile0 = 0;
  a.thin_split = 1;
  a.thin_period = 0;
  a.hp0 = hp0_;
  a.target = target_;
  a.grad_out = d_grad_;
  a.h_part = h_part_;
  a.mm_part = mm_part_;
  a.diverged = d_diverged_;
  a.kexp = kexp_;
  a.inv_sig2 = inv_sig2_;
  a.dt = dt_;
  a.two_lambda = two_lambda_;
  a.epi = kEpiRaw;
  a.step = 0;
  a.tiles_per_problem = 1;
  a.batch_ids = nullptr;
  a.bs_vec = bs_vec_;
  a.bs_grad = (long long)n() * D;
  a.bs_part = part_tiles_;
  a.bs_div = 4;
  a.n_peers = 0;
  return a;
}

template <typename T, int D>
template <int MODE>
void System<T, D>::launch(const KernelChoice<T>& k, PairArgs<T> a, const LaunchPlan& plan)
{
  p2p_dirty_ = true;  // a rank that owns no live rows launches nothing but still has to announce the step
  if (plan.grid <= 0) return;
  a.n_row_tiles = plan.n_row_tiles;
  a.tiles_per_problem = plan.tiles_per_problem;
  a.n_j_tiles = plan.n_j_tiles;
  a.thin_split = plan.thin_split;
  a.thin_period = plan.thin_period;
  if (plan.partial_elems > partials_cap_ || plan.grid > counters_cap_)
    throw StatusError{LMS_ERR_STATE, "launch plan outgrew the stream-K partial buffers"};
  a.partials = partials_;
  a.counters = counters_;
  a.combine_smem_segments = plan.combine_segments;
  // the peer-push stores exist only in the PEERS instantiation of a shape (pair_kernels.cuh, put_all)
  auto fn = plan.thin_split > 1 ? k.fn_thin : k.fn;
  if (a.n_peers > 0) {
    if (k.fn_peers == nullptr)
      throw StatusError{LMS_ERR_STATE, "this kernel variant has no peer-push instantiation (use the default variant)"};
    fn = k.fn_peers;
  }
  if (plan.cluster) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(plan.grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = 0;
    lc.stream = stream_;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kClusterSize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    LMS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k.fn_cluster), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    LMS_CUDA(cudaLaunchKernelEx(&lc, k.fn_cluster, a));
  } else if (pdl_ && !comm_active_) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(plan.grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = plan.dyn_smem;
    lc.stream = stream_;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    LMS_CUDA(cudaLaunchKernelEx(&lc, fn, a));
  } else {
    fn<<<plan.grid, kThreads, plan.dyn_smem, stream_>>>(a);
    LMS_CUDA(cudaGetLastError());
  }
  ++last_eval_launches;
}

// ---- small problems: one persistent cooperative kernel per evaluation (small_kernels.cuh) -----------------------
template <typename T, int D>
void System<T, D>::plan_small()
{
  use_small_ = false;
  if (!small_enabled_ || batch != 1 || comm_active_ || n() <= 0 || n() > small_max_n_) return;
  constexpr int CH = SmallShape<T>::kChunk;
  if (ceil_div(n(), CH) > SmallShape<T>::kMaxChunks) return;  // the whole state is staged at once
  // rows per slot: one packed row pair in fp32, one row in fp64.  (Two packed pairs per slot -- every column load
  // serving both, as in the tiled R = 4 kernels; the kernel template takes RS = 4 -- measured slower on the B200:
  // N = 4000 0.504 vs 0.490 ms, N = 2000 0.188 vs 0.185 ms; it spills at the 128-register cap of a 512-thread CTA.)
  const int rs = SmallShape<T>::kRowsPerSlot;
  const int slots = ceil_div(n(), rs);
  const int grid = std::min(num_sms_, slots);
  // A CTA's slots x 32-column groups are dealt to its sixteen warps in equal contiguous runs (small_kernels.cuh),
  // so any slot count up to kSmallMaxSlots keeps every warp busy.  (Before: one slot per row warp, the spare warps
  // splitting the columns evenly -- N = 3000 left 5 of 16 warps idle.)
  if (ceil_div(slots, grid) > kSmallMaxSlots) return;
  // one adjoint window (N <= 4096 fp32 / 2048 fp64): the instantiation without the window loop
  small_fn_ = n() <= SmallShape<T>::kCols ? small_eval_kernel<T, D, 1> : small_eval_kernel<T, D>;
  small_threads_ = 32 * kSmallWarps;
  int coop = 0;
  LMS_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, cfg.device));
  if (!coop) return;
  // one window: 4D components of kCols columns (adjoint) = 2D components of twice as many (forward)
  small_smem_ = (size_t)(4 * D) * SmallShape<T>::kCols * sizeof(T);
  LMS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(small_fn_), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)small_smem_));
  int per_sm = 0;
  LMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_fn_, small_threads_, small_smem_));
  if (per_sm < 1) return;
  // Thread-block clusters share the state fetch (TMA multicast, small_kernels.cuh): the largest cluster size that
  // still keeps (nearly) every SM busy.  Cluster launches must be whole clusters, so the grid is rounded up to one
  // (CTAs without rows still fetch their share and take part in the barriers).
  static const int force_cs = [] {
    const char* e = std::getenv("LMS_SMALL_CLUSTER");  // experiment knob: cluster size (1 = no clusters)
    return e ? std::atoi(e) : 0;
  }();
  small_cluster_ = 1;
  // Measured on B200 with the state staged in two chunks (ms per gradient, T = 10, clusters of 8 / 4 / 2 / none): fp32
  // N = 500 0.081 / 0.077 / 0.079 / 0.078, 1000 0.101 / 0.093 / 0.096 / 0.094, 2000 0.179 / 0.166 / 0.162 / 0.158, 4000
  // 0.409 / 0.446 / 0.411 / 0.409; fp64 N = 1000 0.156 / 0.144 / 0.145 / 0.141, 2000 0.331 / 0.355 / 0.332 / 0.331.  A shared
  // fetch also couples the CTAs of a cluster (a chunk's barrier completes when the slowest of them has issued its
  // pieces), and with few, large copies L2 serves 148 CTAs as fast as 37 clusters: clusters of four only for the
  // smallest problems, none above.
  const int prefer = n() <= (sizeof(T) == 4 ? 1700 : 700) ? 4 : 1;
  for (int cs : {8, 4, 2}) {
    if (force_cs > 0 ? cs != force_cs : cs > prefer) continue;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(num_sms_ / cs * cs);
    lc.blockDim = dim3(small_threads_);
    lc.dynamicSmemBytes = small_smem_;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, reinterpret_cast<const void*>(small_fn_), &lc) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    const int cap = clusters * cs;
    if (cap >= std::min(grid, num_sms_ * 7 / 8) || force_cs > 0) {
      small_cluster_ = cs;
      small_grid_cap_ = cap;
      break;
    }
  }
  if (small_cluster_ > 1) {
    // cluster launches are whole clusters (CTAs without rows still fetch their share and take part in the barriers)
    const int g = std::min(small_grid_cap_, (int)round_up(grid, small_cluster_));
    if (ceil_div(slots, g) <= kSmallMaxSlots) {
      small_grid_ = g;
    } else {
      small_cluster_ = 1;
      small_grid_ = grid;
    }
  } else {
    small_grid_ = grid;
  }
  use_small_ = true;
}

template <typename T, int D>
void System<T, D>::launch_small(bool host_io)
{
  SmallArgs<T> a{};
  const size_t nd = (size_t)n() * D;
  a.x = host_io ? h_zc_ : d_x_;
  a.traj = traj_;
  a.stride = stride_;
  a.snap_elems = (long long)kState * stride_;
  a.adj0 = adj_[0];
  a.adj1 = adj_[1];
  a.hp0 = hp0_;
  a.target = target_;
  a.grad_out = host_io ? h_zc_ + nd : d_grad_;
  a.warp_part = warp_part_;
  a.scalars = host_io ? h_zc_ + 2 * nd : d_scalars_;
  a.diverged = d_diverged_;
  a.barrier = small_bar_;
  a.bar_base = small_bar_count_;
  // 1 + T + (T-1) barriers per launch; one arrival per CTA, or per cluster with the hierarchical barrier
  small_bar_count_ += (unsigned)(LMS_SMALL_CLUSTER_BARRIER ? small_grid_ / small_cluster_ : small_grid_) * (unsigned)(2 * timesteps);
#ifdef LMS_SMALL_TRACE
  a.trace = reinterpret_cast<unsigned long long*>(d_io_);  // staging scratch: idle during an evaluation
#else
  a.trace = nullptr;
#endif
  a.n = n();
  a.n_chunks = ceil_div(n(), SmallShape<T>::kChunk);
  a.timesteps = timesteps;
  a.kexp = kexp_;
  a.inv_sig2 = inv_sig2_;
  a.dt = dt_;
  a.two_lambda = two_lambda_;
  a.lambda = lambda;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(small_grid_);
  lc.blockDim = dim3(small_threads_);
  lc.dynamicSmemBytes = small_smem_;
  lc.stream = stream_;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the kernel's grid barrier relies on it
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = small_cluster_;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = small_cluster_ > 1 ? 2 : 1;
  LMS_CUDA(cudaLaunchKernelEx(&lc, small_fn_, a));
  last_eval_launches = 1;
  final_adj_ = timesteps & 1;
}

// ---- host <-> planes ---------------------------------------------------------------------------------------
template <typename T, int D>
void System<T, D>::upload(const double* host, T* planes, long long stride, int count, int ncomp, bool check,
                          int step, int batch_count, long long dst_bs)
{
  if (count <= 0) return;
  const size_t elems = (size_t)count * ncomp * batch_count;
  if (elems > io_cap_) {
    sync();
    dev_free(d_io_);
    io_cap_ = elems;
    d_io_ = dev_alloc_zero<double>(4 * io_cap_);
  }
  LMS_CUDA(cudaMemcpyAsync(d_io_, host, elems * sizeof(double), cudaMemcpyHostToDevice, stream_));
  const int blocks = ceil_div((long long)elems, 256);
  aos_to_planes<T><<<blocks, 256, 0, stream_>>>(d_io_, planes, stride, count, ncomp, check ? d_diverged_ : nullptr,
                                                step, batch_count, dst_bs, 4);
  LMS_CUDA(cudaGetLastError());
}

template <typename T, int D>
void System<T, D>::download(const T* planes, long long stride, double* host, int count, int ncomp)
{
  if (count <= 0) return;
  const size_t elems = (size_t)count * ncomp;
  if (elems > io_cap_) {
    sync();
    dev_free(d_io_);
    io_cap_ = elems;
    d_io_ = dev_alloc_zero<double>(4 * io_cap_);
  }
  const int blocks = ceil_div((long long)elems, 256);
  planes_to_aos<T><<<blocks, 256, 0, stream_>>>(planes, stride, d_io_ + io_cap_, count, ncomp);
  LMS_CUDA(cudaGetLastError());
  LMS_CUDA(cudaMemcpyAsync(host, d_io_ + io_cap_, elems * sizeof(double), cudaMemcpyDeviceToHost, stream_));
}

template <typename T, int D>
void System<T, D>::reset_diverged()
{
  LMS_CUDA(cudaMemsetAsync(d_diverged_, 0xff, sizeof(unsigned long long), stream_));
}

template <typename T, int D>
void System<T, D>::read_diverged_or_throw()
{
  LMS_CUDA(cudaMemcpyAsync(h_scalars_, d_scalars_, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  unsigned long long word;
  std::memcpy(&word, h_scalars_ + 3, sizeof(word));
  if (word != kNotDiverged) {
    last_diverged_step = (int)(word >> 32);
    const unsigned low = (unsigned)(word & 0xffffffffull);
    last_diverged_point = low == 0xffffffffu ? -1 : (long long)low;
    throw StatusError{LMS_ERR_DIVERGED, "non-finite state during integration"};
  }
}

template <typename T, int D>
void System<T, D>::require_single(const char* what) const
{
  if (batch != 1) throw StatusError{LMS_ERR_STATE, what};
}

// ---- HamiltonianSystem members ----------------------------------------------------------------------------------
template <typename T, int D>
void System<T, D>::derivatives(const double* q, const double* p, double* hq, double* hp)
{
  require_single("per-function calls need a single-problem handle");
  if (n() == 0) return;
  upload(q, scratch_in_, stride_, n(), D, false, 0);
  upload(p, scratch_in_ + D * stride_, stride_, n(), D, false, 0);
  LaunchPlan plan = plan_for<kFwd>(k_fwd_, n());
  PairArgs<T> a = base_args();
  a.jstate = a.istate = scratch_in_;
  a.out = scratch_out_;
  launch<kFwd>(k_fwd_, a, plan);
  download(scratch_out_, stride_, hq, n(), D);
  sync();
  download(scratch_out_ + D * stride_, stride_, hp, n(), D);
  sync();
}

template <typename T, int D>
void System<T, D>::hamiltonian(const double* q, const double* p, double* out)
{
  require_single("per-function calls need a single-problem handle");
  *out = 0.0;
  if (n() == 0) return;
  upload(q, scratch_in_, stride_, n(), D, false, 0);
  upload(p, scratch_in_ + D * stride_, stride_, n(), D, false, 0);
  LaunchPlan plan = plan_for<kFwd>(k_fwd_, n());
  PairArgs<T> a = base_args();
  a.jstate = a.istate = scratch_in_;
  a.out = scratch_out_;
  a.epi = kEpiRaw | kEpiFirstStep;
  launch<kFwd>(k_fwd_, a, plan);
  // partials are indexed in 128-row units (rt * R), zero where no tile starts
  finalize_scalars<0><<<1, 128, 0, stream_>>>(h_part_, mm_part_, part_tiles_, 0.0, d_scalars_);
  LMS_CUDA(cudaGetLastError());
  LMS_CUDA(cudaMemcpyAsync(h_scalars_, d_scalars_, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  *out = h_scalars_[1];
}

template <typename T, int D>
void System<T, D>::adjoint_step(const double* q, const double* p, const double* alpha, const double* beta,
                                double* da, double* db)
{
  require_single("per-function calls need a single-problem handle");
  if (n() == 0) return;
  upload(q, scratch_in_, stride_, n(), D, false, 0);
  upload(p, scratch_in_ + D * stride_, stride_, n(), D, false, 0);
  upload(alpha, scratch_in_ + 2 * D * stride_, stride_, n(), D, false, 0);
  upload(beta, scratch_in_ + 3 * D * stride_, stride_, n(), D, false, 0);
  LaunchPlan plan = plan_for<kAdj>(k_adj_, n());
  PairArgs<T> a = base_args();
  a.jstate = a.istate = scratch_in_;
  a.jadj = a.iadj = scratch_in_ + kState * stride_;
  a.out = scratch_out_;
  launch<kAdj>(k_adj_, a, plan);
  download(scratch_out_, stride_, da, n(), D);
  sync();
  download(scratch_out_ + D * stride_, stride_, db, n(), D);
  sync();
}

template <typename T, int D>
void System<T, D>::mismatch_sq(const double* a, const double* b, double* out)
{
  require_single("per-function calls need a single-problem handle");
  *out = 0.0;
  if (n() == 0) return;
  upload(a, scratch_in_, stride_, n(), D, false, 0);
  upload(b, scratch_in_ + D * stride_, stride_, n(), D, false, 0);
  mismatch_sequential<T><<<1, 32, 0, stream_>>>(scratch_in_, scratch_in_ + D * stride_, stride_, n(), D,
                                                d_scalars_ + 2);
  LMS_CUDA(cudaGetLastError());
  LMS_CUDA(cudaMemcpyAsync(h_scalars_, d_scalars_, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  *out = h_scalars_[2];
}

template <typename T, int D>
void System<T, D>::integrate_forward(const double* q0, const double* p0, int timesteps, double* tq, double* tp)
{
  require_single("per-function calls need a single-problem handle");
  if (timesteps < 1) throw StatusError{LMS_ERR_INVALID, "timesteps must be >= 1"};
  if (timesteps > max_t_) throw StatusError{LMS_ERR_INVALID, "timesteps exceeds cfg.max_timesteps"};
  if (comm_active_) throw StatusError{LMS_ERR_STATE, "integrate_forward is single-GPU; use the bound objective"};
  stored_t_ = -1;
  traj0_is_q0_ = false;
  if (n() == 0) {
    stored_t_ = timesteps;
    return;
  }
  reset_diverged();
  upload(q0, snapshot(0), stride_, n(), D, true, 0);
  upload(p0, snapshot(0) + D * stride_, stride_, n(), D, true, 0);
  LaunchPlan plan = plan_for<kFwd>(k_fwd_, n());
  const T dt = T(1.0 / timesteps);  // shooting.hpp:190,196
  for (int t = 0; t < timesteps; ++t) {
    PairArgs<T> a = base_args();
    a.jstate = a.istate = snapshot(t);
    a.out = snapshot(t + 1);
    a.dt = dt;
    a.epi = kEpiEuler;
    a.step = t + 1;
    launch<kFwd>(k_fwd_, a, plan);
  }
  read_diverged_or_throw();
  stored_t_ = timesteps;
  for (int t = 0; t <= timesteps; ++t) {
    if (tq) {
      download(snapshot(t), stride_, tq + (size_t)t * n() * D, n(), D);
      sync();
    }
    if (tp) {
      download(snapshot(t) + D * stride_, stride_, tp + (size_t)t * n() * D, n(), D);
      sync();
    }
  }
}

// ---- the bound objective ----------------------------------------------------------------------------------------
// q0 / target: batch x n x D (one registration per problem; batch == 1 for the plain handle).
template <typename T, int D>
void System<T, D>::bind(const double* q0, const double* target, double lambda_in, int timesteps_in)
{
  if (timesteps_in < 1) throw StatusError{LMS_ERR_INVALID, "timesteps must be >= 1"};
  if (timesteps_in > max_t_) throw StatusError{LMS_ERR_INVALID, "timesteps exceeds cfg.max_timesteps"};
  if (!(lambda_in >= 0)) throw StatusError{LMS_ERR_INVALID, "lambda must be >= 0"};
  if (batch > 1 && comm_active_) throw StatusError{LMS_ERR_STATE, "batches are not row-partitioned"};
  sync();
  destroy_graph();
  bound = false;
  lambda = lambda_in;
  timesteps = timesteps_in;
  const size_t per = (size_t)n() * D;
  host_q0.assign(q0, q0 + per * batch);
  host_target.assign(target, target + per * batch);
  dt_ = T(1.0 / timesteps);              // shooting.hpp:190,196,298
  two_lambda_ = T(2) * T(lambda);        // shooting.hpp:293
  q0_bad_ = false;
  q0_bad_problem_.assign(batch, 0);
  for (size_t e = 0; e < host_q0.size(); ++e)
    if (!std::isfinite((double)(T)host_q0[e])) {
      q0_bad_ = true;
      q0_bad_problem_[e / std::max<size_t>(per, 1)] = 1;
    }
  traj0_is_q0_ = false;
  stored_t_ = -1;
  use_small_ = false;
  if (n() > 0) {
    upload(q0, q0_, stride_, n(), D, false, 0, batch, bs_vec_);
    upload(target, target_, stride_, n(), D, false, 0, batch, bs_vec_);
    const int tb_f = row_tile_begin_(kThreads * k_fwd_.rows_per_thread);
    const int te_f = row_tile_end_(kThreads * k_fwd_.rows_per_thread);
    const int tb_a = row_tile_begin_(kThreads * k_adj_.rows_per_thread);
    const int te_a = row_tile_end_(kThreads * k_adj_.rows_per_thread);
    plan_fwd_ = plan_for<kFwd>(k_fwd_, n(), tb_f, std::max(te_f - tb_f, 0), batch);
    plan_adj_ = plan_for<kAdj>(k_adj_, n(), tb_a, std::max(te_a - tb_a, 0), batch);
    sync();
    plan_small();
    if (!comm_active_) {
      // Capture the whole evaluation (2T+2 kernels) into one CUDA graph: at small N the 2T dependent
      // launches are pure latency (SURVEY.md §7 "Small-N latency").
      cudaGraph_t g = nullptr;
      LMS_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_eval(false);
      } catch (...) {
        cudaStreamEndCapture(stream_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      LMS_CUDA(cudaStreamEndCapture(stream_, &g));
      graph_launches_ = last_eval_launches;
      cudaError_t e = cudaGraphInstantiate(&graph_, g, 0);
      cudaGraphDestroy(g);
      LMS_CUDA(e);
    }
  }
  bound = true;
}

// Enqueue one objective evaluation on stream_ for `count` problems (ids on the device, or all): x (double, in
// d_x_) -> scalars in d_scalars_, grad in d_grad_.
template <typename T, int D>
void System<T, D>::enqueue_eval(bool timed, int count, const int* d_ids)
{
  last_eval_launches = 0;
  const int Tn = timesteps;
  if (count < 0) count = batch;
  LaunchPlan pf = plan_fwd_, pa = plan_adj_;
  if (count != batch) {  // a subset of the batch: same kernels, fewer row tiles
    pf = plan_for<kFwd>(k_fwd_, n(), 0, plan_fwd_.tiles_per_problem, count);
    pa = plan_for<kAdj>(k_adj_, n(), 0, plan_adj_.tiles_per_problem, count);
  }
  if (timed && (int)events_.size() < 4 * Tn) {
    while ((int)events_.size() < 4 * Tn) {
      cudaEvent_t e;
      LMS_CUDA(cudaEventCreate(&e));
      events_.push_back(e);
    }
  }
  int ev = 0;
  // reset every problem's divergence word (the 4th double of its scalar record) -- small strided memset
  LMS_CUDA(cudaMemset2DAsync(d_diverged_, 4 * sizeof(double), 0xff, sizeof(unsigned long long), batch, stream_));
  {
    // p0[i][c] = T(x[i*D+c])  (registration.cpp:61-63); non-finite p0 -> DivergedError(0) (shooting.hpp:185-186)
    const long long elems = (long long)n() * D * count;
    aos_to_planes<T><<<ceil_div(elems, 256), 256, 0, stream_>>>(d_x_, snapshot(0) + D * stride_, stride_, n(), D,
                                                                d_diverged_, 0, count, bs_traj_, 4, d_ids);
    LMS_CUDA(cudaGetLastError());
    ++last_eval_launches;
  }
  auto batch_strides = [&](PairArgs<T>& a, long long bs_out, long long bs_adj) {
    if (p2p_active_) {
      a.n_peers = n_peers_;
      for (int k = 0; k < n_peers_; ++k) a.peer_delta[k] = peer_delta_[k];
    }
    a.batch_ids = d_ids;
    a.bs_j = bs_traj_;
    a.bs_adj = bs_adj;
    a.bs_out = bs_out;
    a.bs_seed = bs_state_;
  };
  // forward Euler flow, T+1 snapshots kept for the adjoint (shooting.hpp:199-212)
  for (int t = 0; t < Tn; ++t) {
    PairArgs<T> a = base_args();
    a.jstate = a.istate = snapshot(t);
    a.out = snapshot(t + 1);
    a.adj_seed = adj_[0];
    a.row_tile0 = row_tile_begin_(plan_fwd_.bm);
    a.epi = kEpiEuler | (t == 0 ? kEpiFirstStep : 0u) | (t == Tn - 1 ? kEpiLastStep : 0u);
    a.step = t + 1;
    batch_strides(a, bs_traj_, 0);
    if (timed) LMS_CUDA(cudaEventRecord(events_[ev++], stream_));
    launch<kFwd>(k_fwd_, a, pf);
    if (timed) LMS_CUDA(cudaEventRecord(events_[ev++], stream_));
    if (comm_active_) {
      all_gather_state(snapshot(t + 1));
      if (t == Tn - 1) all_gather_state(adj_[0]);
    }
  }
  if (comm_active_) {
    // Only the rank that owns a non-finite row records the step it appeared at; the others would see it one step
    // later through the gathered state, or not at all when it appears at the last step.  Every rank publishes its
    // word, the words travel with the scalar partials, and every rank keeps the minimum: all ranks then report
    // the same DivergedError(t) (shooting.hpp:210-211) and leave the optimiser together.
    PeerList peers{};
    if (p2p_active_) {
      peers.n = n_peers_;
      for (int k = 0; k < n_peers_; ++k) peers.delta[k] = peer_delta_[k];
    }
    publish_diverged<<<1, 32, 0, stream_>>>(d_diverged_, div_all_ + rank_, peers);
    LMS_CUDA(cudaGetLastError());
    ++last_eval_launches;
    p2p_dirty_ = true;
    gather_inplace({{reinterpret_cast<char*>(h_part_), (size_t)(part_tiles_ / world_) * sizeof(double)},
                    {reinterpret_cast<char*>(mm_part_), (size_t)(part_tiles_ / world_) * sizeof(double)},
                    {reinterpret_cast<char*>(div_all_), sizeof(unsigned long long)}});
    min_diverged<<<1, 32, 0, stream_>>>(div_all_, world_, d_diverged_);
    LMS_CUDA(cudaGetLastError());
    ++last_eval_launches;
  }
  finalize_scalars<0><<<count, 128, 0, stream_>>>(h_part_, mm_part_, part_tiles_, lambda, d_scalars_, d_ids);
  LMS_CUDA(cudaGetLastError());
  ++last_eval_launches;
  // discrete adjoint sweep t = T-1 .. 0 (shooting.hpp:300-307), final gradient fused into the t = 0 launch
  int cur = 0;
  for (int t = Tn - 1; t >= 0; --t) {
    PairArgs<T> a = base_args();
    a.jstate = a.istate = snapshot(t);
    a.jadj = a.iadj = adj_[cur];
    a.out = adj_[cur ^ 1];
    a.row_tile0 = row_tile_begin_(plan_adj_.bm);
    a.epi = kEpiEuler | (t == 0 ? kEpiGradOut : 0u);
    a.step = t;
    batch_strides(a, bs_state_, bs_state_);
    if (timed) LMS_CUDA(cudaEventRecord(events_[ev++], stream_));
    launch<kAdj>(k_adj_, a, pa);
    if (timed) LMS_CUDA(cudaEventRecord(events_[ev++], stream_));
    if (comm_active_ && t > 0) all_gather_state(adj_[cur ^ 1]);
    cur ^= 1;
  }
  if (comm_active_) {
    // every rank ends with the full gradient (row-major double rows are contiguous per rank slice)
    gather_inplace({{reinterpret_cast<char*>(d_grad_), (size_t)(stride_ / world_) * D * sizeof(double)}});
  }
  final_adj_ = cur;
}

// Shared body of eval / eval_batch: copies x in, runs the evaluation, copies grad and the scalar records out.
template <typename T, int D>
void System<T, D>::eval_batch(const double* x, double* grad, double* scalars, int* diverged_step, int count,
                              const int* ids)
{
  if (!bound) throw StatusError{LMS_ERR_STATE, "lms_bind_registration must precede evaluation"};
  if (count < 0 || count > batch) throw StatusError{LMS_ERR_INVALID, "bad problem count"};
  const bool subset = ids != nullptr;
  if (!subset) count = batch;
  for (int b = 0; b < batch; ++b)
    if (!subset && diverged_step) diverged_step[b] = -1;
  if (n() == 0 || count == 0) {
    for (int k = 0; k < count; ++k) {
      const int b = subset ? ids[k] : k;
      scalars[3 * b] = scalars[3 * b + 1] = scalars[3 * b + 2] = 0.0;
      if (diverged_step) diverged_step[b] = -1;
    }
    return;
  }
  const size_t per = (size_t)n() * D;
  if (!traj0_is_q0_) {
    const long long elems = (long long)per * batch;
    copy_planes<T><<<ceil_div(elems, 256), 256, 0, stream_>>>(q0_, stride_, snapshot(0), stride_, n(), D, batch,
                                                              bs_vec_, bs_traj_);
    LMS_CUDA(cudaGetLastError());
    traj0_is_q0_ = true;
  }
  if (subset) {
    for (int k = 0; k < count; ++k)
      if (ids[k] < 0 || ids[k] >= batch) throw StatusError{LMS_ERR_INVALID, "problem id out of range"};
    // runs of neighbouring ids travel as one copy (the rendezvous of lms_batch_register hands sorted lists)
    for (int k = 0; k < count;) {
      int e = k + 1;
      while (e < count && ids[e] == ids[e - 1] + 1) ++e;
      LMS_CUDA(cudaMemcpyAsync(d_x_ + ids[k] * per, x + ids[k] * per, (size_t)(e - k) * per * sizeof(double),
                               cudaMemcpyHostToDevice, stream_));
      k = e;
    }
    LMS_CUDA(cudaMemcpyAsync(d_ids_, ids, count * sizeof(int), cudaMemcpyHostToDevice, stream_));
  } else {
    LMS_CUDA(cudaMemcpyAsync(d_x_, x, per * batch * sizeof(double), cudaMemcpyHostToDevice, stream_));
  }
  LMS_CUDA(cudaEventRecord(ev_begin_, stream_));
  if (graph_ && !subset && !kernel_timing) {
    LMS_CUDA(cudaGraphLaunch(graph_, stream_));
    last_eval_launches = graph_launches_;
  } else {
    enqueue_eval(false, count, subset ? d_ids_ : nullptr);
  }
  LMS_CUDA(cudaEventRecord(ev_end_, stream_));
  if (subset) {
    for (int k = 0; k < count;) {
      int e = k + 1;
      while (e < count && ids[e] == ids[e - 1] + 1) ++e;
      LMS_CUDA(cudaMemcpyAsync(grad + ids[k] * per, d_grad_ + ids[k] * per, (size_t)(e - k) * per * sizeof(double),
                               cudaMemcpyDeviceToHost, stream_));
      k = e;
    }
  } else {
    LMS_CUDA(cudaMemcpyAsync(grad, d_grad_, per * batch * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  }
  LMS_CUDA(cudaMemcpyAsync(h_scalars_, d_scalars_, 4 * sizeof(double) * batch, cudaMemcpyDeviceToHost, stream_));
  sync();
  stored_t_ = timesteps;
  float ms = 0.f;
  LMS_CUDA(cudaEventElapsedTime(&ms, ev_begin_, ev_end_));
  last_eval_ms = ms;
  for (int k = 0; k < count; ++k) {
    const int b = subset ? ids[k] : k;
    unsigned long long word;
    std::memcpy(&word, h_scalars_ + 4 * b + 3, sizeof(word));
    int step = word == kNotDiverged ? -1 : (int)(word >> 32);
    if (q0_bad_problem_[b]) step = 0;  // non-finite template: DivergedError(0), shooting.hpp:185-186
    if (diverged_step) diverged_step[b] = step;
    scalars[3 * b] = h_scalars_[4 * b];
    scalars[3 * b + 1] = h_scalars_[4 * b + 1];
    scalars[3 * b + 2] = h_scalars_[4 * b + 2];
  }
}

template <typename T, int D>
void System<T, D>::eval(const double* x, double* grad, double* scalars, bool device_ptrs)
{
  require_single("this handle holds a batch: use lms_batch_eval");
  if (!bound) throw StatusError{LMS_ERR_STATE, "lms_bind_registration must precede evaluation"};
  if (n() == 0) {
    scalars[0] = scalars[1] = scalars[2] = 0.0;
    return;
  }
  if (q0_bad_) {
    last_diverged_step = 0;
    last_diverged_point = -1;
    throw StatusError{LMS_ERR_DIVERGED, "non-finite template landmarks"};
  }
  const size_t bytes = (size_t)n() * D * sizeof(double);
  if (!traj0_is_q0_) {
    const long long elems = (long long)n() * D;
    copy_planes<T><<<ceil_div(elems, 256), 256, 0, stream_>>>(q0_, stride_, snapshot(0), stride_, n(), D);
    LMS_CUDA(cudaGetLastError());
    traj0_is_q0_ = true;
  }
  const bool timed = kernel_timing;
  // Small problems called with host buffers: the persistent kernel reads x from, and writes the gradient, the
  // scalars and the divergence word to, mapped pinned memory -- no staging copies around the one launch.
  const bool zero_copy = use_small_ && !timed && !device_ptrs && h_zc_ != nullptr;
  if (zero_copy) {
    const size_t nd = (size_t)n() * D;
    std::memcpy(h_zc_, x, bytes);
    d_x_current_ = false;
    LMS_CUDA(cudaEventRecord(ev_begin_, stream_));
    launch_small(/*host_io=*/true);
    LMS_CUDA(cudaEventRecord(ev_end_, stream_));
    stored_t_ = timesteps;
    sync();
    std::memcpy(grad, h_zc_ + nd, bytes);
    std::memcpy(h_scalars_, h_zc_ + 2 * nd, 4 * sizeof(double));
    unsigned long long word;
    std::memcpy(&word, h_scalars_ + 3, sizeof(word));
    if (word != kNotDiverged) {
      last_diverged_step = (int)(word >> 32);
      const unsigned low = (unsigned)(word & 0xffffffffull);
      last_diverged_point = low == 0xffffffffu ? -1 : (long long)low;
      throw StatusError{LMS_ERR_DIVERGED, "non-finite state during integration"};
    }
  } else {
    LMS_CUDA(cudaMemcpyAsync(d_x_, x, bytes, device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             stream_));
    d_x_current_ = true;
    LMS_CUDA(cudaEventRecord(ev_begin_, stream_));
    if (use_small_ && !timed) {
      launch_small();
    } else if (graph_ && !timed) {
      LMS_CUDA(cudaGraphLaunch(graph_, stream_));
      last_eval_launches = graph_launches_;
    } else {
      enqueue_eval(timed);
    }
    LMS_CUDA(cudaEventRecord(ev_end_, stream_));
    LMS_CUDA(cudaMemcpyAsync(grad, d_grad_, bytes, device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             stream_));
    stored_t_ = timesteps;
    read_diverged_or_throw();  // synchronises
  }
  float ms = 0.f;
  LMS_CUDA(cudaEventElapsedTime(&ms, ev_begin_, ev_end_));
  last_eval_ms = ms;
  if (timed) {
    double sum[2] = {0, 0};
    for (int k = 0; k < 2 * timesteps; ++k) {
      float m = 0.f;
      LMS_CUDA(cudaEventElapsedTime(&m, events_[2 * k], events_[2 * k + 1]));
      sum[k < timesteps ? 0 : 1] += m;
    }
    last_kernel_ms[0] = sum[0] / timesteps;
    last_kernel_ms[1] = sum[1] / timesteps;
  }
  scalars[0] = h_scalars_[0];
  scalars[1] = h_scalars_[1];
  scalars[2] = h_scalars_[2];
}

template <typename T, int D>
void System<T, D>::final_q(double* out)
{
  require_single("this handle holds a batch: use lms_batch_final_q");
  if (stored_t_ < 0) throw StatusError{LMS_ERR_STATE, "no stored trajectory"};
  if (n() == 0) return;
  download(snapshot(stored_t_), stride_, out, n(), D);
  sync();
}

// average_dist / max_dist of (template, target) and of (warped = q(1) of the stored trajectory, target), on the
// device (registration.cpp:39-40,95-96; landmarks.cpp:164-179).  The sets are the reference's double landmark sets:
// the bound template / target as given, q(1) widened from the working precision (registration.cpp:88-92).
template <typename T, int D>
void System<T, D>::registration_metrics(double* out)
{
  require_single("registration metrics need a single-problem handle");
  if (!bound) throw StatusError{LMS_ERR_STATE, "lms_bind_registration must precede the metrics"};
  if (stored_t_ < 0) throw StatusError{LMS_ERR_STATE, "no stored trajectory"};
  if (n() == 0) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    return;
  }
  const size_t nd = (size_t)n() * D;  // d_io_ holds 4 * io_cap_ >= 4 nd doubles: a | b | distances
  double* a = d_io_;
  double* b = d_io_ + nd;
  double* dist = d_io_ + 2 * nd;         // n <= nd doubles
  double* res = d_metrics_;
  const int blocks = ceil_div(n(), 256);
  LMS_CUDA(cudaMemcpyAsync(a, host_q0.data(), nd * sizeof(double), cudaMemcpyHostToDevice, stream_));
  LMS_CUDA(cudaMemcpyAsync(b, host_target.data(), nd * sizeof(double), cudaMemcpyHostToDevice, stream_));
  point_distances<><<<blocks, 256, 0, stream_>>>(a, b, n(), D, dist);
  avg_max_sequential<><<<1, 32, 0, stream_>>>(dist, n(), res);
  planes_to_aos<T><<<ceil_div((long long)nd, 256), 256, 0, stream_>>>(snapshot(stored_t_), stride_, a, n(), D);
  point_distances<><<<blocks, 256, 0, stream_>>>(a, b, n(), D, dist);
  avg_max_sequential<><<<1, 32, 0, stream_>>>(dist, n(), res + 2);
  LMS_CUDA(cudaGetLastError());
  LMS_CUDA(cudaMemcpyAsync(h_scalars_, res, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  for (int k = 0; k < 4; ++k) out[k] = h_scalars_[k];
}

// q(1) of every problem of the batch: batch x n x D.
template <typename T, int D>
void System<T, D>::final_q_batch(double* out)
{
  if (stored_t_ < 0) throw StatusError{LMS_ERR_STATE, "no stored trajectory"};
  if (n() == 0) return;
  const size_t elems = (size_t)n() * D * batch;
  if (elems > io_cap_) {
    sync();
    dev_free(d_io_);
    io_cap_ = elems;
    d_io_ = dev_alloc_zero<double>(4 * io_cap_);
  }
  planes_to_aos<T><<<ceil_div((long long)elems, 256), 256, 0, stream_>>>(snapshot(stored_t_), stride_, d_io_ + io_cap_,
                                                                         n(), D, batch, bs_traj_);
  LMS_CUDA(cudaGetLastError());
  LMS_CUDA(cudaMemcpyAsync(out, d_io_ + io_cap_, elems * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
}

// ---- flow --------------------------------------------------------------------------------------------------------
template <typename T, int D>
void System<T, D>::ensure_points(size_t m)
{
  const long long need = std::max<long long>(round_up((long long)m, row_align_), row_align_);
  if ((size_t)need > points_cap_) {
    sync();
    dev_free(points_[0]);
    dev_free(points_[1]);
    points_[0] = dev_alloc_zero<T>((size_t)need * D);
    points_[1] = dev_alloc_zero<T>((size_t)need * D);
    points_cap_ = (size_t)need;
  }
  points_stride_ = (long long)points_cap_;
}

template <typename T, int D>
void System<T, D>::velocities(const double* q, const double* p, size_t m, const double* pts, double* out)
{
  require_single("per-function calls need a single-problem handle");
  if (m == 0) return;
  ensure_points(m);
  if (n() > 0) {
    upload(q, scratch_in_, stride_, n(), D, false, 0);
    upload(p, scratch_in_ + D * stride_, stride_, n(), D, false, 0);
  }
  upload(pts, points_[0], points_stride_, (int)m, D, false, 0);
  if (n() == 0) {  // empty sum
    std::fill(out, out + m * D, 0.0);
    sync();
    return;
  }
  LaunchPlan plan = plan_for<kVel>(k_vel_, (int)m);
  PairArgs<T> a = base_args();
  a.jstate = scratch_in_;
  a.istate = points_[0];
  a.istride = points_stride_;
  a.n_rows = (int)m;
  a.out = points_[1];
  a.ostride = points_stride_;
  launch<kVel>(k_vel_, a, plan);
  download(points_[1], points_stride_, out, (int)m, D);
  sync();
}

template <typename T, int D>
void System<T, D>::warp_stored(size_t m, const double* pts, double* out)
{
  require_single("per-function calls need a single-problem handle");
  if (stored_t_ < 1) throw StatusError{LMS_ERR_STATE, "no stored trajectory: integrate or evaluate first"};
  if (m == 0) return;
  ensure_points(m);
  reset_diverged();
  upload(pts, points_[0], points_stride_, (int)m, D, false, 0);
  int cur = 0;
  if (n() > 0) {
    LaunchPlan plan = plan_for<kVel>(k_vel_, (int)m);
    const T dt = T(1.0 / stored_t_);  // the trajectory's own dt (flow.hpp:70)
    for (int t = 0; t < stored_t_; ++t) {
      PairArgs<T> a = base_args();
      a.jstate = snapshot(t);
      a.istate = points_[cur];
      a.istride = points_stride_;
      a.n_rows = (int)m;
      a.out = points_[cur ^ 1];
      a.ostride = points_stride_;
      a.dt = dt;
      a.epi = kEpiEuler;
      a.step = t + 1;
      launch<kVel>(k_vel_, a, plan);
      cur ^= 1;
    }
  }
  read_diverged_or_throw();
  download(points_[cur], points_stride_, out, (int)m, D);
  sync();
}

// ---- row partition: NCCL over NVLink, or the in-process loopback group -------------------------------------------
// Re-lay the planes so that every rank owns an equal, tile-aligned slice (in-place all-gather).
template <typename T, int D>
void System<T, D>::relayout_for_world(int world, int rank)
{
  if (batch != 1) throw StatusError{LMS_ERR_STATE, "batches are not row-partitioned"};
  sync();
  destroy_graph();
  bound = false;
  if (world > 1) {
    pick_kernels(/*partitioned=*/true);
    alloc_partials();
    // Every kernel a partitioned evaluation launches is loaded now: with lazy module loading a first launch inside
    // an evaluation can synchronise the context while a peer's stream sits in a stream-ordered wait for this
    // rank (ranks that share one process and one GPU would deadlock; see p2p_connect).
    const void* fns[] = {reinterpret_cast<const void*>(k_fwd_.fn), reinterpret_cast<const void*>(k_adj_.fn),
                         reinterpret_cast<const void*>(k_fwd_.fn_peers), reinterpret_cast<const void*>(k_adj_.fn_peers),
                         reinterpret_cast<const void*>(&publish_diverged<0>), reinterpret_cast<const void*>(&min_diverged<0>),
                         reinterpret_cast<const void*>(&finalize_scalars<0>), reinterpret_cast<const void*>(&aos_to_planes<T>),
                         reinterpret_cast<const void*>(&copy_planes<T>)};
    for (const void* fn : fns) {
      if (fn == nullptr) continue;
      cudaFuncAttributes attr;
      LMS_CUDA(cudaFuncGetAttributes(&attr, fn));
    }
  }
  const long long new_stride = world > 1 ? partition_rows((long long)cfg.n, world, rank).stride : stride_;
  if (new_stride != stride_) {
    stride_ = new_stride;
    const size_t plane = (size_t)stride_;
    p2p_disconnect();
    dev_free(arena_); dev_free(hp0_); dev_free(target_); dev_free(q0_);
    dev_free(scratch_in_); dev_free(scratch_out_); dev_free(d_x_);
    bs_traj_ = (long long)(max_t_ + 1) * kState * stride_;
    bs_state_ = (long long)kState * stride_;
    bs_vec_ = (long long)D * stride_;
    hp0_ = dev_alloc_zero<T>(D * plane);
    target_ = dev_alloc_zero<T>(D * plane);
    q0_ = dev_alloc_zero<T>(D * plane);
    scratch_in_ = dev_alloc_zero<T>(2 * kState * plane);
    scratch_out_ = dev_alloc_zero<T>(kState * plane);
    d_x_ = dev_alloc_zero<double>(plane * D);
    part_tiles_ = (int)(stride_ / kThreads);
    alloc_exchange_arena();
  }
  rank_ = rank;
  world_ = world;
}

template <typename T, int D>
void System<T, D>::comm_init(const unsigned char* id, int rank, int world)
{
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world) throw StatusError{LMS_ERR_INVALID, "bad rank/world"};
  // world == 1 normally needs no communicator; LMS_FORCE_NCCL=1 keeps the NCCL path on so that a single-GPU
  // box can exercise it (tests/test_gpu_parity.py::test_nccl_path_single_rank).
  const char* force = std::getenv("LMS_FORCE_NCCL");
  if (world == 1 && !(force && force[0] == '1')) return;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) throw StatusError{LMS_ERR_COMM, "libnccl.so.2 could not be loaded"};
  relayout_for_world(world, rank);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  if (nc.CommInitRank(&comm_, world, uid, rank) != 0) throw StatusError{LMS_ERR_COMM, "ncclCommInitRank failed"};
  local_ = nullptr;
  comm_active_ = true;
}

template <typename T, int D>
void System<T, D>::join_local_group(LocalGroup* group, int rank)
{
  if (!group || group->world > kMaxRanks || rank < 0 || rank >= group->world)
    throw StatusError{LMS_ERR_INVALID, "bad rank/world"};
  relayout_for_world(group->world, rank);
  local_ = group;
  comm_active_ = true;
}

// The one exchange primitive: every buffer is `world` slices of `bytes`; rank r's slice r is final on this rank
// and the other slices are filled from the peers.
template <typename T, int D>
void System<T, D>::gather_inplace(const std::vector<std::pair<char*, size_t>>& buffers)
{
  if (p2p_active_) {  // the epilogues already pushed every slice: only the arrival flags are exchanged
    p2p_exchange();
    return;
  }
  if (local_ == nullptr) {
    const NcclApi& nc = nccl_api();
    bool ok = nc.GroupStart() == 0;
    for (const auto& b : buffers)
      ok = ok && nc.AllGather(b.first + rank_ * b.second, b.first, b.second, kNcclInt8, comm_, stream_) == 0;
    ok = (nc.GroupEnd() == 0) && ok;
    if (!ok) throw StatusError{LMS_ERR_COMM, "ncclAllGather failed"};
    return;
  }
  // loopback: my slices are final once my stream drains; publish, meet, pull the peers' slices, meet again so
  // that nobody overwrites a buffer a peer is still reading
  cudaError_t e = cudaStreamSynchronize(stream_);
  {
    std::lock_guard<std::mutex> lock(local_->m);
    local_->lists[rank_] = buffers;
    if (e != cudaSuccess) local_->failed = true;
  }
  local_->barrier();
  if (!local_->failed) {
    for (int p = 0; p < world_ && e == cudaSuccess; ++p) {
      if (p == rank_) continue;
      const auto& theirs = local_->lists[p];
      for (size_t k = 0; k < buffers.size() && k < theirs.size() && e == cudaSuccess; ++k)
        e = cudaMemcpyAsync(buffers[k].first + p * buffers[k].second, theirs[k].first + p * theirs[k].second,
                            buffers[k].second, cudaMemcpyDeviceToDevice, stream_);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream_);
    if (e != cudaSuccess) {
      std::lock_guard<std::mutex> lock(local_->m);
      local_->failed = true;
    }
  }
  local_->barrier();
  if (local_->failed) throw StatusError{LMS_ERR_COMM, "loopback exchange failed"};
}

// In-place all-gather of every plane of a (q,p) or (alpha,beta) state: rank r contributes rows
// [r*slice, (r+1)*slice) of each plane.
template <typename T, int D>
void System<T, D>::all_gather_state(T* planes)
{
  const size_t slice_bytes = (size_t)(stride_ / world_) * sizeof(T);
  std::vector<std::pair<char*, size_t>> buffers;
  for (int k = 0; k < kState; ++k)
    buffers.emplace_back(reinterpret_cast<char*>(planes + (long long)k * stride_), slice_bytes);
  gather_inplace(buffers);
}

// Per-row-tile double partials: tiles are indexed globally, each rank filled its own contiguous range.
template <typename T, int D>
void System<T, D>::all_gather_doubles(double* buf)
{
  gather_inplace({{reinterpret_cast<char*>(buf), (size_t)(part_tiles_ / world_) * sizeof(double)}});
}

// ---- peer-push exchange ------------------------------------------------------------------------------------------
// The third transport of the row partition (after NCCL and the in-process loopback).  Every rank maps every
// peer's exchange arena -- cudaIpcOpenMemHandle across processes, the plain pointer inside one process (peer
// access enabled when the devices differ) -- and the Euler epilogues of the pair kernels store each updated
// row into all arenas (put_all, pair_kernels.cuh): the exchange of step t rides on the NVLink stores issued
// while the remaining row tiles of step t are still being computed.  What is left of the all-gather is one
// 4-byte flag per peer: after its launch a rank writes its epoch into every peer's flag slot in stream order
// (cuStreamWriteValue32: fenced after the kernel's stores) and its stream waits until every peer's slot has
// reached the epoch (cuStreamWaitValue32), so no SM ever spins.  Buffers cannot be overwritten early: a rank
// only starts step s+1 after every peer has finished step s, and the two adjoint states / T+1 snapshots are
// written in alternation.
namespace {
using StreamValueFn = int (*)(cudaStream_t, unsigned long long, unsigned, unsigned);
struct StreamMemOps {
  StreamValueFn write = nullptr, wait = nullptr;
  bool ok = false;
};
const StreamMemOps& stream_mem_ops()
{
  static const StreamMemOps ops = [] {
    StreamMemOps o;
    void* w = nullptr;
    void* q = nullptr;
    cudaDriverEntryPointQueryResult rw, rq;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &rw) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &q, cudaEnableDefault, &rq) == cudaSuccess &&
        rw == cudaDriverEntryPointSuccess && rq == cudaDriverEntryPointSuccess && w && q) {
      o.write = reinterpret_cast<StreamValueFn>(w);
      o.wait = reinterpret_cast<StreamValueFn>(q);
      o.ok = true;
    }
    cudaGetLastError();
    return o;
  }();
  return ops;
}
constexpr unsigned long long kBlobMagic = 0x4c4d53503250ull;  // "LMSP2P"
}  // namespace

template <typename T, int D>
void System<T, D>::p2p_export(int rank, int world, unsigned char* blob)
{
  if (world < 1 || world > kMaxPeers + 1 || rank < 0 || rank >= world)
    throw StatusError{LMS_ERR_INVALID, "bad rank/world (the peer-push exchange serves up to 8 ranks)"};
  if (!stream_mem_ops().ok) throw StatusError{LMS_ERR_COMM, "stream memory operations are not available"};
  relayout_for_world(world, rank);
  p2p_disconnect();
  LMS_CUDA(cudaMemsetAsync(p2p_flags_, 0, 256, stream_));
  sync();
  P2PBlob b{};
  b.magic = kBlobMagic;
  b.pid = (long long)getpid();
  b.device = cfg.device;
  b.rank = rank;
  b.world = world;
  b.base = (unsigned long long)reinterpret_cast<uintptr_t>(arena_);
  b.bytes = arena_bytes_;
  if (world > 1) LMS_CUDA(cudaIpcGetMemHandle(&b.handle, arena_));
  std::memset(blob, 0, 128);
  std::memcpy(blob, &b, sizeof(b));
}

template <typename T, int D>
void System<T, D>::p2p_connect(const unsigned char* blobs)
{
  P2PBlob mine{};
  std::memcpy(&mine, blobs + (size_t)rank_ * 128, sizeof(mine));
  if (mine.magic != kBlobMagic || mine.rank != rank_ || mine.world != world_ ||
      mine.base != (unsigned long long)reinterpret_cast<uintptr_t>(arena_))
    throw StatusError{LMS_ERR_STATE, "lms_p2p_connect: this rank's blob is not the one lms_p2p_export produced"};
  p2p_disconnect();
  n_peers_ = 0;
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) continue;
    P2PBlob b{};
    std::memcpy(&b, blobs + (size_t)r * 128, sizeof(b));
    if (b.magic != kBlobMagic || b.rank != r || b.world != world_ || b.bytes != arena_bytes_)
      throw StatusError{LMS_ERR_INVALID, "lms_p2p_connect: inconsistent peer blob (same n, T, precision on every rank?)"};
    char* theirs = nullptr;
    if (b.pid == (long long)getpid()) {
      theirs = reinterpret_cast<char*>((uintptr_t)b.base);
      if (b.device != cfg.device) {
        int can = 0;
        LMS_CUDA(cudaDeviceCanAccessPeer(&can, cfg.device, b.device));
        if (!can) throw StatusError{LMS_ERR_COMM, "peer access between the devices is not possible"};
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) LMS_CUDA(e);
        cudaGetLastError();
      }
    } else {
      void* mapped = nullptr;
      LMS_CUDA(cudaIpcOpenMemHandle(&mapped, b.handle, cudaIpcMemLazyEnablePeerAccess));
      peer_mapping_[n_peers_] = mapped;
      theirs = static_cast<char*>(mapped);
    }
    peer_rank_[n_peers_] = r;
    peer_delta_[n_peers_] = (long long)(theirs - arena_);
    ++n_peers_;
  }
  p2p_epoch_ = 0;
  p2p_dirty_ = false;
  local_ = nullptr;
  p2p_active_ = world_ > 1;
  comm_active_ = world_ > 1;
  // The peer-push instantiations are launched for the first time inside a partitioned evaluation, when a peer's
  // stream may already sit in a stream-ordered wait for this rank's flag: lazy module loading at that point
  // synchronises the context and would deadlock ranks that share one.  Load them now.
  void (*const peer_fns[2])(PairArgs<T>) = {k_fwd_.fn_peers, k_adj_.fn_peers};
  for (auto fn : peer_fns) {
    if (fn == nullptr) throw StatusError{LMS_ERR_STATE, "this kernel variant has no peer-push instantiation (use the default variant)"};
    cudaFuncAttributes attr;
    LMS_CUDA(cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(fn)));
    PairArgs<T> none{};  // no row tiles, no columns: the kernel starts and returns without touching memory
    fn<<<1, kThreads, 0, stream_>>>(none);
    LMS_CUDA(cudaGetLastError());
  }
  sync();
}

template <typename T, int D>
void System<T, D>::p2p_disconnect()
{
  if (stream_) cudaStreamSynchronize(stream_);
  for (int k = 0; k < kMaxPeers; ++k) {
    if (peer_mapping_[k]) cudaIpcCloseMemHandle(peer_mapping_[k]);
    peer_mapping_[k] = nullptr;
  }
  n_peers_ = 0;
  if (p2p_active_) comm_active_ = false;
  p2p_active_ = false;
}

// Announce "everything up to my last launch is in your arena" to every peer, then hold the stream until every
// peer has announced the same.  Consecutive gathers with no launch in between share one exchange.
template <typename T, int D>
void System<T, D>::p2p_exchange()
{
  if (!p2p_dirty_) return;
  p2p_dirty_ = false;
  const StreamMemOps& ops = stream_mem_ops();
  ++p2p_epoch_;
  bool ok = true;
  for (int k = 0; k < n_peers_; ++k) {
    unsigned* slot = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(p2p_flags_ + rank_) + peer_delta_[k]);
    ok = ok && ops.write(stream_, (unsigned long long)reinterpret_cast<uintptr_t>(slot), p2p_epoch_, 0u) == 0;
  }
  for (int k = 0; k < n_peers_; ++k)  // CU_STREAM_WAIT_VALUE_GEQ = 0: (int)(*slot - epoch) >= 0, wrap-safe
    ok = ok && ops.wait(stream_, (unsigned long long)reinterpret_cast<uintptr_t>(p2p_flags_ + peer_rank_[k]),
                        p2p_epoch_, 0u) == 0;
  if (!ok) throw StatusError{LMS_ERR_COMM, "stream memory operation failed"};
}

}  // namespace lms
