// Fused pairwise-interaction kernels for landmark geodesic shooting on sm_100a.
//
// One kernel template covers the three O(N^2) row reductions of the reference:
//   kFwd  derivatives            shooting.hpp:147-176 (term :158-169)
//   kAdj  adjoint_step           shooting.hpp:233-271 (term :249-264)
//   kVel  velocities_at_step     flow.hpp:26-48
// K_ij is never materialised: each thread owns R rows, keeps their 2D (or D) running sums in
// registers and sweeps j-tiles of the landmark state staged in shared memory.  The Euler update
// (shooting.hpp:205-211 / :302-306), the finite check, the loss scalars (:286-288), the adjoint seed
// (:290-296) and the final gradient (:309-313) run as epilogues of the same kernels.
//
// Data layout in HBM: component planes.  A "state" is 2*D planes (q_0..q_{D-1}, p_0..p_{D-1}) of
// `stride` elements each; an "adjoint state" is 2*D planes (alpha, beta).  Planes are zero-padded
// past n: a padded column has p = alpha = 0 and finite q, beta, so it contributes exact zeros to
// every sum (SURVEY.md §7 "Padding").
//
// Work decomposition: the (row tile) x (j tile) cell grid is laid out row-major and cut into
// gridDim.x equal contiguous ranges (stream-K), so every CTA does the same number of cells +-1
// whatever N is.  A CTA whose range ends inside a row tile writes its partial sums to a slot; the
// last CTA to arrive for that row tile (threadfence + counter) adds the slots in ascending j order
// and runs the epilogue.  The combine order depends only on (n, grid), never on timing, so results
// are bitwise reproducible run to run (reduction.hpp:38-40 promises the same of the CPU backends).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

// segments of partial sums whose loads are in flight together in the last CTA's combine loop
#ifndef LMS_COMBINE_UNROLL
#define LMS_COMBINE_UNROLL 4
#endif

namespace lms {

// -DLMS_TAIL_TRACE: thread 0 of every CTA that finishes a shared row tile prints the cycle counts of its hand-over
// chain (measurement build only: scripts/gpu_tail_trace.py)
#ifdef LMS_TAIL_TRACE
#define LMS_TT(i) do { if (threadIdx.x == 0) tt[i] = clock64(); } while (0)
#else
#define LMS_TT(i) do { } while (0)
#endif

constexpr int kCombineUnroll = LMS_COMBINE_UNROLL;
constexpr int kThreads = 128;  // threads per CTA
constexpr int kTileJ = 128;    // columns staged per shared-memory tile
constexpr int kUnitJ = 8;      // stream-K work unit: kUnitJ columns of one row tile
constexpr int kUnitsPerTile = kTileJ / kUnitJ;
constexpr int kClusterSize = 16;  // CTAs per row tile in the cluster-combine kernels (non-portable cluster size)
constexpr int kMaxPeers = 7;   // row partition, peer-push transport: up to 8 GPUs of one NVSwitch domain
constexpr int kMaxRanks = 64;  // row partition, any transport (the in-process loopback group takes up to 64)

enum Mode : int { kFwd = 0, kAdj = 1, kVel = 2 };
template <bool B>
struct ThinTag { static constexpr bool value = B; };

// Epilogue selector / flags.
enum : unsigned {
  kEpiRaw = 0u,        // write the row sums themselves (hq,hp | d_alpha,d_beta | v)
  kEpiEuler = 1u,      // apply the explicit-Euler (or Euler-adjoint) update and store the new state
  kEpiFirstStep = 2u,  // fwd: also store hp(q0,p0) and the per-tile partial of H = 1/2 sum p.hp
  kEpiLastStep = 4u,   // fwd: also per-tile mismatch partial and the adjoint seed (alpha_T, beta_T)
  kEpiGradOut = 8u,    // adj: also grad = beta_0 + hp(q0,p0) as row-major double
};

template <typename T>
struct PairArgs {
  // columns j: landmark state (and adjoint state for kAdj)
  const T* jstate;
  const T* jadj;
  long long jstride;
  int n_cols;
  int n_j_tiles;
  // rows i: for kFwd/kAdj the same arrays as the columns; for kVel the D planes of query points
  const T* istate;
  const T* iadj;
  long long istride;
  int n_rows;       // rows are valid for row < n_rows
  int row_tile0;    // first row tile owned by this launch (row partition across GPUs)
  int n_row_tiles;  // row tiles owned by this launch
  // Thin last row tile: when the launch's last row tile holds at most 1/thin_split of a tile's rows (the rest is
  // padding), its live rows are replicated over thin_split groups of warps and each group sweeps 1/thin_split of
  // every staged column tile; the groups' sums meet in shared memory before the stream-K combine.  The tile then
  // counts 1/thin_split of a tile's work units.  1: every tile is a full tile.  (2 or 4; single problem only.)
  int thin_split;
  // A thin tile stages a whole column tile for 1/thin_split of the work, so its units cost a few per cent more than a
  // full tile's, and the CTAs sweeping it would finish last.  To keep the stream-K shares equal in time, every
  // thin_period-th cell of the thin tile is a phantom (no columns): the tile counts P + P / (thin_period - 1) cells
  // for its P units.  0: no phantoms.
  int thin_period;
  // outputs
  T* out;           // raw: sums planes; euler: next state / next adjoint state / moved points
  long long ostride;
  T* adj_seed;      // kEpiLastStep: adjoint state planes receiving (alpha_T, beta_T = 0)
  T* hp0;           // kEpiFirstStep: D planes written; kEpiGradOut: D planes read
  const T* target;  // kEpiLastStep: D planes
  double* grad_out; // kEpiGradOut: row-major double n x D
  double* h_part;   // per-row-tile partials of sum_i p_i . hp_i
  double* mm_part;  // per-row-tile partials of sum_i |q_i(1) - target_i|^2
  unsigned long long* diverged;  // atomicMin of (step << 32 | point)
  // stream-K bookkeeping
  T* partials;   // 2 * gridDim.x slots of kAcc * (kThreads * R) sums (see the combine in pair_kernel)
  int combine_smem_segments;  // partial segments the launch's dynamic shared memory holds at once (0: none)
  int* counters; // gridDim.x arrival counters, zero between launches
  // constants, rounded on the host exactly as the reference rounds them (shooting.hpp:63-68,114-115,
  // 196,293): kexp = k_scale * log2(e) for float (ex2.approx), k_scale * log2(e) * 2^kExpBits for double (Math<double>).
  T kexp;
  T inv_sig2;
  T dt;
  T two_lambda;
  unsigned epi;
  int step;  // time step whose state this launch produces (for the divergence record)
  // batch of independent problems (population studies): row tile t of this launch belongs to problem
  // batch_ids[t / tiles_per_problem] (identity when null); every pointer above is problem 0's and the
  // strides below (in elements of the pointed-to type) step to the next problem.  Single problem: all zero.
  int tiles_per_problem;
  const int* batch_ids;
  long long bs_j, bs_adj, bs_out, bs_seed, bs_vec, bs_grad, bs_part, bs_div;
  // Row partition with the peer-push exchange (system.cu, p2p_*): every store of the Euler epilogues (new state,
  // adjoint seed, gradient, scalar partials) also goes to the same offset of each peer's exchange arena -- over
  // NVLink when the peer is another GPU -- so the updated slice travels while the other row tiles are still
  // being computed and no gather kernel follows.  n_peers == 0: single GPU, or the NCCL / loopback transports.
  int n_peers;
  long long peer_delta[kMaxPeers];  // byte distance from this rank's arena to each peer's mapping of its arena
};

// One value to the local buffer and -- PEERS kernels only -- to the same place in every peer's arena.  (The peer loop
// is compiled only into the kernels a row-partitioned handle launches with the peer-push transport: unrolled into
// every epilogue store it made the kernels 4-5 x larger -- 11 584 instead of 2 200 instructions for the fp32 adjoint --
// and the cold, bloated epilogue cost every launch of a single-GPU evaluation 0.3 % at N = 20 000 up to 6 % at N = 1000.)
template <bool PEERS, typename T, typename V>
__device__ __forceinline__ void put_all(const PairArgs<T>& a, V* p, V v)
{
  *p = v;
  if constexpr (PEERS) {
    for (int k = 0; k < a.n_peers; ++k) *reinterpret_cast<V*>(reinterpret_cast<char*>(p) + a.peer_delta[k]) = v;
  }
}

// ---------------------------------------------------------------------------------------------
// scalar math per working precision
// ---------------------------------------------------------------------------------------------
template <typename T>
struct Math;

template <>
struct Math<float> {
  static __device__ __forceinline__ float kernel(float r2, float kexp, const double* = nullptr)
  {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(r2 * kexp));
    return y;
  }
  static __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ bool finite(float a) { return isfinite(a); }
};

// fp64 exp: table of 2^(j/2^B) and a near-minimax polynomial for 2^(g/2^B) on g in [-1/2, 1/2] (mpmath chebyfit,
// 50 digits, coefficients rounded to double; constant term exactly 1 so that K(r = 0) = 1).  LMS_EXP_BITS selects
//   4: 16 entries (128 B: every bank once, conflict-free for any index pattern), degree 6, |rel err| < 7.9e-18
//   5: 32 entries, degree 5, < 1.5e-16        6: 64 entries, degree 4, < 2.5e-15
// A larger table trades DP-pipe work (one DFMA per step) for shared-memory bank conflicts on the table load.
// Measured on B200 (N = 20 000, T = 10 gradient; side-by-side builds with LMS_NVCC_EXTRA=-DLMS_EXP_BITS=..): 22.33 / 21.90 / 21.64 ms for B = 4 / 5 / 6
// (degree 7 with 16 entries, the first version: 22.85 ms).  Default 5: the last setting below half an ulp.
#ifndef LMS_EXP_BITS
#define LMS_EXP_BITS 5
#endif
constexpr int kExpBits = LMS_EXP_BITS;
constexpr int kExpEntries = 1 << kExpBits;
// 2^(j/64), j = 0..63, correctly rounded; the smaller tables take every 2nd / 4th entry.
__device__ __constant__ double kExp2Table64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};

// The shared-memory table of Math<double>::kernel (see the layout note there).
#ifndef LMS_EXP_TABLE_PER_LANE
#define LMS_EXP_TABLE_PER_LANE 0
#endif
constexpr int kExpTableCopies = LMS_EXP_TABLE_PER_LANE ? 32 : 1;
constexpr int kExpTableDoubles = kExpEntries * kExpTableCopies;
__device__ __forceinline__ void fill_exp_table(double* tbl, int tid, int threads)
{
  for (int e = tid; e < kExpTableDoubles; e += threads)
    tbl[e] = kExp2Table64[(e / kExpTableCopies) * (64 / kExpEntries)];
}
// this thread's view of the table
__device__ __forceinline__ const double* exp_table_of_lane(const double* tbl, int tid)
{
  return LMS_EXP_TABLE_PER_LANE ? tbl + (tid & 31) : tbl;
}

template <>
struct Math<double> {
  // exp(r2 * k_scale) for r2 * k_scale <= 0, branch-free.  kexp = k_scale * log2(e) * 2^B (host, one rounding),
  // s = r2 * kexp; 2^(s/2^B) = 2^n * 2^(j/2^B) * 2^(g/2^B) with 2^B n + j = rint(s), g = s - rint(s) in
  // [-1/2, 1/2].  With B = 5: 11 DP-pipe operations against the 18 of CUDA's exp(), and no slow path: with
  // landmarks many sigma apart most pairs underflow, which is exactly where the library routine branches.
  // Results below the normal range flush to zero.
  static __device__ __forceinline__ double kernel(double r2, double kexp, const double* __restrict__ tbl)
  {
    double s = r2 * kexp;
    constexpr double floor_s = -1080.0 * kExpEntries;  // 2^-1080; a NaN argument falls through and propagates
    s = s < floor_s ? floor_s : s;
    const double magic = 6755399441055744.0;  // 1.5 * 2^52: the low word of (s + magic) is rint(s)
    const double km = __dadd_rn(s, magic);
    const int ki = __double2loint(km);
    const double g = s - __dadd_rn(km, -magic);
    double p;
    if constexpr (kExpBits == 4) {
      p = 0x1.430a49610efc6p-37;
      p = fma(p, g, 0x1.5d89be4c12513p-30);
      p = fma(p, g, 0x1.3b2ab6fb09b31p-23);
      p = fma(p, g, 0x1.c6b08d6e8a384p-17);
      p = fma(p, g, 0x1.ebfbdff82c594p-11);
      p = fma(p, g, 0x1.62e42fefa39fdp-5);
    } else if constexpr (kExpBits == 5) {
      // (Estrin's grouping of the same polynomial -- one more multiply, a chain of 4 instead of 6 -- measured slower:
      // 22.73 vs 22.38 ms per gradient; the DP pipe, not the chain, is what is short.)
      p = 0x1.5d885e6ef14a6p-35;
      p = fma(p, g, 0x1.3b2b301f1eb9cp-27);
      p = fma(p, g, 0x1.c6b08d70380ddp-20);
      p = fma(p, g, 0x1.ebfbdff7feebap-13);
      p = fma(p, g, 0x1.62e42fefa39efp-6);
    } else {
      p = 0x1.3b2ad0385b409p-31;
      p = fma(p, g, 0x1.c6b0c40d8c4e9p-23);
      p = fma(p, g, 0x1.ebfbdff82ac52p-15);
      p = fma(p, g, 0x1.62e42fefa0352p-7);
    }
    p = fma(p, g, 1.0);
    // One shared copy of the table (LMS_EXP_TABLE_PER_LANE=0, the default): entries j and j + 16 sit on the same bank
    // pair, and ncu counts 5.6 M shared-memory conflict replays per launch at N = 20 000 -- but landmarks many sigma
    // apart clamp to the same entry, which is a broadcast, and the two conflict-free layouts measured SLOWER on the
    // B200 (fp64 gradient, N = 20 000, T = 10): one copy 21.85 ms | low/high words in two 32-entry arrays (every
    // entry its own bank, two LDS.32) 22.42 ms | one copy per lane (tbl[j * 32 + lane], one LDS.64, always two full
    // wavefronts) 22.38 ms; conflicts 5.63 M -> 0 / 7 in both.  The per-lane layout stays selectable for A/B.
#if LMS_EXP_TABLE_PER_LANE
    const double r = tbl[(ki & (kExpEntries - 1)) * 32] * p;  // `tbl` already points at this lane's copy
#else
    const double r = tbl[ki & (kExpEntries - 1)] * p;
#endif
    const int n = ki >> kExpBits;
    const double scaled = __hiloint2double(__double2hiint(r) + n * 1048576, __double2loint(r));
    return n < -1021 ? 0.0 : scaled;
  }
  static __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ bool finite(double a) { return isfinite(a); }
};

template <int MODE, int D>
struct Shape {
  static constexpr int kColComps = MODE == kAdj ? 4 * D : 2 * D;              // staged per column
  static constexpr int kRowComps = MODE == kAdj ? 4 * D : (MODE == kFwd ? 2 * D : D);
  static constexpr int kAcc = MODE == kVel ? D : 2 * D;                        // sums per row
};

// One pair (i, j).  ri: row operands [q, p, (alpha, beta)] or [x]; cj: column operands.
// Forward accumulates  acc[0..D) += (p_i.p_j) K dx,  acc[D..2D) += K p_j   (hq = -inv_sig2 * acc[0..D)).
// Adjoint accumulates  acc[0..D) += K (dx (c t - pa) - c db),  acc[D..2D) += K a_j - K t p_j
//   with t = inv_sig2 (dx.db);  d_alpha = inv_sig2 * acc[0..D),  d_beta = acc[D..2D).
template <typename T, int D, int MODE>
__device__ __forceinline__ void pair_term(const T* __restrict__ ri, const T* __restrict__ cj,
                                          T* __restrict__ acc, T kexp, T inv_sig2, const double* __restrict__ tbl)
{
  T dx[D];
#pragma unroll
  for (int c = 0; c < D; ++c) dx[c] = ri[c] - cj[c];
  T r2 = dx[0] * dx[0];
#pragma unroll
  for (int c = 1; c < D; ++c) r2 = fma(dx[c], dx[c], r2);
  const T k = Math<T>::kernel(r2, kexp, tbl);
  if constexpr (MODE == kVel) {
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] = fma(k, cj[D + c], acc[c]);
  } else if constexpr (MODE == kFwd) {
    T cc = ri[D] * cj[D];
#pragma unroll
    for (int c = 1; c < D; ++c) cc = fma(ri[D + c], cj[D + c], cc);
    const T s = cc * k;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      acc[c] = fma(s, dx[c], acc[c]);
      acc[D + c] = fma(k, cj[D + c], acc[D + c]);
    }
  } else {
    const T* pi = ri + D;
    const T* ai = ri + 2 * D;
    const T* bi = ri + 3 * D;
    const T* pj = cj + D;
    const T* aj = cj + 2 * D;
    const T* bj = cj + 3 * D;
    T cc = pi[0] * pj[0];
    T pa = pi[0] * aj[0];
#pragma unroll
    for (int c = 1; c < D; ++c) {
      cc = fma(pi[c], pj[c], cc);
      pa = fma(pi[c], aj[c], pa);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) pa = fma(pj[c], ai[c], pa);
    T db[D];
#pragma unroll
    for (int c = 0; c < D; ++c) db[c] = bj[c] - bi[c];
    T rb = dx[0] * db[0];
#pragma unroll
    for (int c = 1; c < D; ++c) rb = fma(dx[c], db[c], rb);
    const T t = rb * inv_sig2;
    const T u = fma(cc, t, -pa);
    const T ka = k * u;
    const T kc = k * cc;
    const T kt = k * t;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      acc[c] = fma(ka, dx[c], acc[c]);
      acc[c] = fma(-kc, db[c], acc[c]);
      acc[D + c] = fma(k, aj[c], acc[D + c]);
      acc[D + c] = fma(-kt, pj[c], acc[D + c]);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// fp32 packed path: sm_100a's two-wide FP32 instructions (FFMA2 / FADD2 / FMUL2).
// A thread packs two of its rows into the halves of a 64-bit register pair; the column operand is
// the same for both rows and enters as FFMA2's scalar-broadcast (.F32) operand.  Measured on B200 (profiles/ubench): FFMA2 sustains 128 lanes/SM/clk from HALF the issue
// slots of scalar FFMA, and its 64-bit operand reads do not hit the register-bank dispatch stalls
// that hold the scalar kernels at ~77 % issue utilisation (profiles/r1_ncu_v0_scalar.md).
// Packed operands cannot take a free negation, so the terms are arranged with plus signs only:
//   ndx = q_j - q_i (= -dx), nbv = b_i - b_j (= -db), nt = -inv_sig2 (ndx.nbv) (= -t)
//   forward : acc[0..D) += (p_i.p_j) K ndx   (= -(p_i.p_j) K dx: negated once after the sweep)
//   adjoint : acc[0..D) += K (pa - c t) ndx + K c nbv,   acc[D..2D) += K a_j + K nt p_j
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ float2 splat2(float v) { return make_float2(v, v); }

__device__ __forceinline__ float2 ex2_pair(float2 x)
{
  float2 y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(x.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(x.y));
  return y;
}

// ri2: packed row operands [nq (= -q_i), p, (alpha, beta)] or [nx]; cj2: duplicated column operands.
template <int D, int MODE>
__device__ __forceinline__ void pair_term_packed(const float2* __restrict__ ri2, const float2* __restrict__ cj2,
                                                 float2* __restrict__ acc, float2 kexp2, float2 ns2, float2 neg1)
{
  float2 ndx[D];
#pragma unroll
  for (int c = 0; c < D; ++c) ndx[c] = __fadd2_rn(cj2[c], ri2[c]);
  float2 r2 = __fmul2_rn(ndx[0], ndx[0]);
#pragma unroll
  for (int c = 1; c < D; ++c) r2 = __ffma2_rn(ndx[c], ndx[c], r2);
  const float2 k = ex2_pair(__fmul2_rn(r2, kexp2));
  if constexpr (MODE == kVel) {
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] = __ffma2_rn(k, cj2[D + c], acc[c]);
  } else if constexpr (MODE == kFwd) {
    float2 cc = __fmul2_rn(ri2[D], cj2[D]);
#pragma unroll
    for (int c = 1; c < D; ++c) cc = __ffma2_rn(ri2[D + c], cj2[D + c], cc);
    const float2 s = __fmul2_rn(cc, k);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      acc[c] = __ffma2_rn(s, ndx[c], acc[c]);
      acc[D + c] = __ffma2_rn(k, cj2[D + c], acc[D + c]);
    }
  } else {
    const float2* pi = ri2 + D;
    const float2* ai = ri2 + 2 * D;
    const float2* bi = ri2 + 3 * D;
    const float2* pj = cj2 + D;
    const float2* aj = cj2 + 2 * D;
    const float2* bj = cj2 + 3 * D;
    float2 cc = __fmul2_rn(pi[0], pj[0]);
    float2 pa = __fmul2_rn(pi[0], aj[0]);
#pragma unroll
    for (int c = 1; c < D; ++c) {
      cc = __ffma2_rn(pi[c], pj[c], cc);
      pa = __ffma2_rn(pi[c], aj[c], pa);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) pa = __ffma2_rn(pj[c], ai[c], pa);
    float2 nbv[D];
#pragma unroll
    for (int c = 0; c < D; ++c) nbv[c] = __ffma2_rn(bj[c], neg1, bi[c]);
    float2 rb = __fmul2_rn(ndx[0], nbv[0]);
#pragma unroll
    for (int c = 1; c < D; ++c) rb = __ffma2_rn(ndx[c], nbv[c], rb);
    const float2 nt = __fmul2_rn(rb, ns2);
    const float2 w = __ffma2_rn(cc, nt, pa);
    const float2 kw = __fmul2_rn(k, w);
    const float2 kc = __fmul2_rn(k, cc);
    const float2 knt = __fmul2_rn(k, nt);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      acc[c] = __ffma2_rn(kw, ndx[c], acc[c]);
      acc[c] = __ffma2_rn(kc, nbv[c], acc[c]);
      acc[D + c] = __ffma2_rn(k, aj[c], acc[D + c]);
      acc[D + c] = __ffma2_rn(knt, pj[c], acc[D + c]);
    }
  }
}

// Row owned by (r, tid) in row tile rt.  Packed kernels pair rows (2*tid, 2*tid+1) of each 256-row group.
template <int R, bool PACKED>
__device__ __forceinline__ long long row_of(int rt, int r, int tid, int threads = kThreads)
{
  // `threads` < kThreads: a thin tile (PairArgs::thin_split), whose rows are laid over the first `threads`
  // threads only (tid is then the index within that group)
  if constexpr (PACKED)
    return (long long)rt * (kThreads * R) + (r >> 1) * (2 * threads) + 2 * tid + (r & 1);
  else
    return (long long)rt * (kThreads * R) + r * threads + tid;
}

// ---------------------------------------------------------------------------------------------
// Bulk-async (TMA) staging of column tiles: one elected thread issues cp.async.bulk copies of the
// contiguous 128-column chunk of every component plane straight into shared memory; completion is
// tracked by an mbarrier (complete_tx), so no thread spends registers or LDG/STS slots on staging.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity)
{
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LMS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra LMS_DONE_%=;\n"
      "bra LMS_WAIT_%=;\n"
      "LMS_DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Vector load of JU consecutive columns of one staged component.
template <typename T, int JU>
struct ColVec;
template <>
struct ColVec<float, 4> {
  static __device__ __forceinline__ void load(const float* p, float* v)
  {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
};
template <>
struct ColVec<float, 2> {
  static __device__ __forceinline__ void load(const float* p, float* v)
  {
    const float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  }
};
template <>
struct ColVec<double, 2> {
  static __device__ __forceinline__ void load(const double* p, double* v)
  {
    const double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x; v[1] = t.y;
  }
};
template <>
struct ColVec<double, 1> {
  static __device__ __forceinline__ void load(const double* p, double* v) { v[0] = *p; }
};
template <>
struct ColVec<float, 1> {
  static __device__ __forceinline__ void load(const float* p, float* v) { v[0] = *p; }
};

// Fixed-order block sum of one double per thread (tree over shared memory; deterministic).
__device__ __forceinline__ double block_sum(double v, double* scratch)
{
  const int tid = threadIdx.x;
  scratch[tid] = v;
  __syncthreads();
#pragma unroll
  for (int h = kThreads / 2; h >= 1; h >>= 1) {
    if (tid < h) scratch[tid] += scratch[tid + h];
    __syncthreads();
  }
  const double r = scratch[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
// AOS: the shared-memory tile holds each column's NC components contiguously (column-major), filled by
// the register-staged path (every thread transposes its own column with 16-byte stores), so one column
// costs NC/4 LDS.128 with only NC registers of column data live (the plane layout needs JU = 4 columns,
// 4 NC registers, for the same load count).
// CLUSTER: small problems.  The launch is kClusterSize CTAs per row tile, each with an equal share of the columns,
// started as one thread-block cluster; the tile's partial sums meet in distributed shared memory (every CTA parks
// its sums in its own tile buffers, rank 0 adds the kClusterSize copies in ascending column order and runs the
// epilogue) instead of going through global slots, a fence, an arrival counter and L2 round trips.
template <typename T, int D, int MODE, int R, int JU, int MINB, bool PACKED = false, int UNR = 1, bool BULK = false,
          bool AOS = false, bool CLUSTER = false, bool PEERS = false, bool THINOK = false>
__global__ void __launch_bounds__(kThreads, MINB) pair_kernel(const PairArgs<T> a)
{
  static_assert(!CLUSTER || 2 * Shape<MODE, D>::kColComps * kTileJ >= Shape<MODE, D>::kAcc * kThreads * R,
                "the tile buffers must hold one set of partial sums");
  static_assert(!PACKED || (sizeof(T) == 4 && R % 2 == 0), "the packed path is fp32 with an even row count");
  static_assert(!AOS || (sizeof(T) == 4 && JU == 1 && !BULK && Shape<MODE, D>::kColComps % 4 == 0),
                "column-major tiles: fp32, one column per step, register-staged, 16-byte multiples");
  using S = Shape<MODE, D>;
  constexpr int NC = S::kColComps;
  constexpr int NR = S::kRowComps;
  constexpr int NA = S::kAcc;
  constexpr int BM = kThreads * R;

  __shared__ __align__(16) T tile[2][AOS ? kTileJ : NC][AOS ? NC : kTileJ];
  __shared__ double red_scratch[kThreads];
  __shared__ double exp_tbl_all[sizeof(T) == 8 ? kExpTableDoubles : 1];  // fp64 only: 2^(j/2^B)
  __shared__ int s_last;
  __shared__ __align__(8) unsigned long long tile_bar[2];  // BULK only: one mbarrier per tile buffer
  __shared__ __align__(8) unsigned long long combine_bar;  // the combine's bulk copies (see below)
  extern __shared__ __align__(128) unsigned char combine_smem[];  // landing zone for partial segments, if any
  unsigned combine_parity = 0;
  // Programmatic dependent launch: the next launch of the evaluation may start scheduling its CTAs as soon as
  // every CTA of this one is running, so they take over SM slots as ours retire and the launch latency
  // between the 2T dependent steps disappears.  A no-op when the launch carries no PDL attribute.
  asm volatile("griddepcontrol.launch_dependents;");
  int buf = 0;                // tile buffer in use; kept across row tiles so the mbarrier phases stay in step
  unsigned wait_parity = 0;   // bit b: parity the next wait on buffer b must observe
  if constexpr (BULK) {
    if (threadIdx.x == 0) {
      mbar_init(&tile_bar[0], 1);
      mbar_init(&tile_bar[1], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  if (a.combine_smem_segments > 0) {
    if (threadIdx.x == 0) {
      mbar_init(&combine_bar, 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  if constexpr (sizeof(T) == 8) {
    fill_exp_table(exp_tbl_all, threadIdx.x, kThreads);
    __syncthreads();
  }

  // everything above touched no global memory; everything below reads what the previous launch wrote
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int tid = threadIdx.x;
  const double* exp_tbl = exp_table_of_lane(exp_tbl_all, tid);
  // Work is counted in units of kUnitJ columns of one row tile, so every CTA's share differs by at most
  // one unit (1/16 of a staged tile); `cells` and `nJ` below are in those units.
  const long long nJ = (long long)a.n_j_tiles * kUnitsPerTile;
  // (THINOK: only the shapes instantiated with the thin-tile code take it; the others compile as if it did not exist)
  const int split = THINOK && a.thin_split > 1 ? a.thin_split : 1;  // > 1: the last row tile is thin and holds fewer units
  // split == 8 (four-row packed shapes): 4 groups of warps, and inside a group the thread's two packed row pairs hold
  // the SAME two rows and sweep the two halves of the group's column window (`pair split`)
  constexpr bool kPairSplit = THINOK && PACKED && R == 4;
  const bool pair_split = kPairSplit && split == 8;
  const int groups = pair_split ? 4 : split;
  const int period = split > 1 && a.thin_period > 1 ? a.thin_period : 0;
  const long long nJ_thin = nJ / split + (period ? (nJ / split) / (period - 1) : 0);  // cells of the thin tile
  const long long cells = (long long)a.n_row_tiles * nJ - (nJ - nJ_thin);
  const long long G = gridDim.x;
  long long c = cells * blockIdx.x / G;
  const long long c_end = cells * (blockIdx.x + 1) / G;

  while (c < c_end) {
    const long long rt_local = c / nJ;  // (the thin tile is the last one, so this holds for it too)
    const bool thin = THINOK && split > 1 && rt_local == a.n_row_tiles - 1;
    const long long nJ_this = thin ? nJ_thin : nJ;
    const int tc0 = (int)(c - rt_local * nJ);  // cell range [tc0, tc1) of this row tile
    const long long span = c_end - c;
    const int tc1 = (int)((long long)tc0 + span < nJ_this ? (long long)tc0 + span : nJ_this);
    // Unit range of the cells [tc0, tc1): the cells themselves, minus the phantoms before them in a thin tile.  A
    // unit is kUnitJ columns per sweeping group of warps.  Full tile: one group (the CTA), kUnitsPerTile units per
    // staged tile.  Thin tile: `split` groups side by side, group g sweeping columns [g, g + 1) * kTileJ / split of
    // every staged tile, so a staged tile holds kUnitsPerTile / split units.  (Everything thin-specific is derived
    // from tc0 / tc1 where it is used, so that full tiles carry nothing extra through their sweep.)
    auto units_of = [&](int tc) { return period ? tc - tc / period : tc; };
    const int jt_first = thin ? units_of(tc0) / (kUnitsPerTile / split) : tc0 * kUnitJ / kTileJ;  // first staged tile
    // problem this row tile belongs to (uniform per CTA iteration: lives in uniform registers)
    const long long bc = rt_local / a.tiles_per_problem;
    const long long prob = a.batch_ids != nullptr ? (long long)a.batch_ids[bc] : bc;
    const int rt = a.row_tile0 + (int)(rt_local - bc * a.tiles_per_problem);
    const T* jstate_b = a.jstate + prob * a.bs_j;
    const T* jadj_b = a.jadj + prob * a.bs_adj;
    const T* istate_b = MODE == kVel ? a.istate : a.istate + prob * a.bs_j;
    const T* iadj_b = a.iadj + prob * a.bs_adj;
    T* out_b = a.out + prob * a.bs_out;
    T* adj_seed_b = a.adj_seed + prob * a.bs_seed;
    T* hp0_b = a.hp0 + prob * a.bs_vec;
    const T* target_b = a.target + prob * a.bs_vec;
    double* grad_out_b = a.grad_out + prob * a.bs_grad;
    double* h_part_b = a.h_part + prob * a.bs_part;
    double* mm_part_b = a.mm_part + prob * a.bs_part;
    unsigned long long* diverged_b = a.diverged + prob * a.bs_div;
    // Column plane c of a tile: kAdj stages state planes [0,2D) then adjoint planes [0,2D).
    auto col_plane = [&](int comp) -> const T* {
      if constexpr (MODE == kAdj) {
        return comp < 2 * D ? jstate_b + (long long)comp * a.jstride : jadj_b + (long long)(comp - 2 * D) * a.jstride;
      } else {
        return jstate_b + (long long)comp * a.jstride;
      }
    };

    // ---- row operands --------------------------------------------------------------------
    T ri[R][NR];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int grp_threads = thin ? kThreads / groups : kThreads;  // threads that hold distinct rows
      const long long row = thin ? row_of<R, PACKED>(rt, pair_split ? (r & 1) : r, tid % grp_threads, grp_threads)
                                 : row_of<R, PACKED>(rt, r, tid);
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        if constexpr (MODE == kAdj) {
          ri[r][k] = k < 2 * D ? istate_b[(long long)k * a.istride + row]
                               : iadj_b[(long long)(k - 2 * D) * a.istride + row];
        } else {
          ri[r][k] = istate_b[(long long)k * a.istride + row];
        }
      }
    }
    T acc[R][NA];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NA; ++k) acc[r][k] = T(0);

    // ---- sweep the j tiles [jt0, jt1) with register-prefetched double buffering ---------------
    // (only the units [u0, u1) of the first and last tile are accumulated)
    T stage[BULK ? 1 : NC];
    auto issue_tile = [&](int jt, int b) {  // BULK: called by thread 0 only
      mbar_expect_tx(&tile_bar[b], (unsigned)(NC * kTileJ * sizeof(T)));
#pragma unroll
      for (int k = 0; k < NC; ++k)
        bulk_g2s(&tile[b][k][0], col_plane(k) + (long long)jt * kTileJ, (unsigned)(kTileJ * sizeof(T)), &tile_bar[b]);
    };
    if constexpr (BULK) {
      // (a thin range that is a single phantom cell sweeps nothing: tc1 - tc0 > 1 or the cell is a real one)
      if (tid == 0 && (!thin || units_of(tc1) > units_of(tc0))) issue_tile(jt_first, buf);  // `buf` was last read before the previous __syncthreads
    } else {
#pragma unroll
      for (int k = 0; k < NC; ++k) stage[k] = col_plane(k)[(long long)jt_first * kTileJ + tid];
      buf = 0;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        if constexpr (AOS) tile[0][tid][k] = stage[k];
        else tile[0][k][tid] = stage[k];
      }
      __syncthreads();
    }

    // packed path only: two rows per 64-bit register pair; -q_i (or -x_i) first, the rest as they are
    constexpr int RP = PACKED ? R / 2 : 1;
    float2 ri2[RP][NR];
    float2 acc2[RP][NA];
    float2 kexp2, ns2, neg1;
    if constexpr (PACKED) {
#pragma unroll
      for (int rp = 0; rp < RP; ++rp) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          const float lo = (float)ri[2 * rp][k], hi = (float)ri[2 * rp + 1][k];
          ri2[rp][k] = k < D ? make_float2(-lo, -hi) : make_float2(lo, hi);
        }
#pragma unroll
        for (int k = 0; k < NA; ++k) acc2[rp][k] = make_float2(0.f, 0.f);
      }
      kexp2 = splat2((float)a.kexp);
      ns2 = splat2(-(float)a.inv_sig2);
      neg1 = splat2(-1.f);
    }

    // The sweep is instantiated twice: the full-tile copy has its column bounds in compile-time multiples of the
    // tile (the hot loop of every launch, code-generated exactly as before the thin tile existed), the thin copy
    // takes the group's column window and units-per-tile from registers.
    auto sweep = [&](auto thin_tag) {
    constexpr bool THIN = decltype(thin_tag)::value;
    // full tile: the column range [col0, col1) in multiples of kUnitJ, as compile-time-scaled integers
    const int col0 = tc0 * kUnitJ, col1 = tc1 * kUnitJ;
    const int upt_s = kUnitsPerTile / split;
    const int u0 = THIN ? units_of(tc0) : 0;
    const int u1 = THIN ? units_of(tc1) : 0;
    const int jt0 = THIN ? u0 / upt_s : col0 / kTileJ;
    const int jt1 = THIN ? (u1 > u0 ? (u1 + upt_s - 1) / upt_s : jt0) : (col1 + kTileJ - 1) / kTileJ;
    const int jj_base = THIN ? (tid / (kThreads / groups)) * (kTileJ / groups) : 0;  // this group's window of a tile
    const int pair_off = THIN && pair_split ? kTileJ / 8 : 0;  // second row pair: the other half of the window
    for (int jt = jt0; jt < jt1; ++jt) {
      const bool more = jt + 1 < jt1;
      if constexpr (BULK) {
        if (more && tid == 0) issue_tile(jt + 1, buf ^ 1);
        mbar_wait(&tile_bar[buf], (wait_parity >> buf) & 1u);
        wait_parity ^= 1u << buf;
      } else {
        if (more) {
#pragma unroll
          for (int k = 0; k < NC; ++k) stage[k] = col_plane(k)[(long long)(jt + 1) * kTileJ + tid];
        }
      }
      int jj_lo, jj_hi;
      if constexpr (THIN) {
        const int k_lo = u0 > jt * upt_s ? u0 - jt * upt_s : 0;
        const int k_hi = u1 < (jt + 1) * upt_s ? u1 - jt * upt_s : upt_s;
        jj_lo = jj_base + k_lo * kUnitJ;
        jj_hi = jj_base + k_hi * kUnitJ;
      } else {
        jj_lo = col0 > jt * kTileJ ? col0 - jt * kTileJ : 0;
        jj_hi = col1 < (jt + 1) * kTileJ ? col1 - jt * kTileJ : kTileJ;
      }
#pragma unroll UNR
      for (int jj = jj_lo; jj < jj_hi; jj += JU) {
        T cj[JU][NC];
        if constexpr (AOS) {
#pragma unroll
          for (int k = 0; k < NC; k += 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(&tile[buf][jj][k]);
            cj[0][k] = t4.x; cj[0][k + 1] = t4.y; cj[0][k + 2] = t4.z; cj[0][k + 3] = t4.w;
          }
        } else {
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            T v[JU];
            ColVec<T, JU>::load(&tile[buf][k][jj], v);
#pragma unroll
            for (int u = 0; u < JU; ++u) cj[u][k] = v[u];
          }
        }
        // thin tile of the four-row packed shapes: the second row pair reads its own columns (pair_off further on; the
        // same ones when the tile is not pair-split)
        constexpr bool kSecond = THIN && kPairSplit;
        T cjb[kSecond ? JU : 1][kSecond ? NC : 1];
        if constexpr (kSecond) {
          if constexpr (AOS) {
#pragma unroll
            for (int k = 0; k < NC; k += 4) {
              const float4 t4 = *reinterpret_cast<const float4*>(&tile[buf][jj + pair_off][k]);
              cjb[0][k] = t4.x; cjb[0][k + 1] = t4.y; cjb[0][k + 2] = t4.z; cjb[0][k + 3] = t4.w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < NC; ++k) {
              T v[JU];
              ColVec<T, JU>::load(&tile[buf][k][jj + pair_off], v);
#pragma unroll
              for (int u = 0; u < JU; ++u) cjb[u][k] = v[u];
            }
          }
        }
        if constexpr (!PACKED) {
#pragma unroll
          for (int u = 0; u < JU; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) pair_term<T, D, MODE>(ri[r], cj[u], acc[r], a.kexp, a.inv_sig2, exp_tbl);
        } else {
#pragma unroll
          for (int u = 0; u < JU; ++u) {
            // the column operand is the same for both packed rows: ptxas folds splat2() into FFMA2's
            // scalar-broadcast (.F32) operand form, so no register or shared-memory duplication is needed
            float2 cj2[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) cj2[k] = splat2((float)cj[u][k]);
            if constexpr (kSecond) {
              float2 cjb2[NC];
#pragma unroll
              for (int k = 0; k < NC; ++k) cjb2[k] = splat2((float)cjb[u][k]);
              pair_term_packed<D, MODE>(ri2[0], cj2, acc2[0], kexp2, ns2, neg1);
              pair_term_packed<D, MODE>(ri2[1], cjb2, acc2[1], kexp2, ns2, neg1);
            } else {
#pragma unroll
              for (int rp = 0; rp < RP; ++rp) pair_term_packed<D, MODE>(ri2[rp], cj2, acc2[rp], kexp2, ns2, neg1);
            }
          }
        }
      }
      if constexpr (!BULK) {
        if (more) {
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            if constexpr (AOS) tile[buf ^ 1][tid][k] = stage[k];
            else tile[buf ^ 1][k][tid] = stage[k];
          }
        }
      }
      __syncthreads();
      buf ^= 1;
    }
    };
    if constexpr (THINOK) {
      if (thin) sweep(ThinTag<true>{});
      else sweep(ThinTag<false>{});
    } else {
      sweep(ThinTag<false>{});
    }
    if constexpr (PACKED) {
      // back to the scalar convention of pair_term: forward acc[0..D) holds +(p_i.p_j) K dx.  The scalar
      // row operands are rebuilt from the packed ones so that only one copy stays live across the sweep.
#pragma unroll
      for (int rp = 0; rp < RP; ++rp) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          ri[2 * rp][k] = (T)(k < D ? -ri2[rp][k].x : ri2[rp][k].x);
          ri[2 * rp + 1][k] = (T)(k < D ? -ri2[rp][k].y : ri2[rp][k].y);
        }
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          const bool flip = MODE == kFwd && k < D;
          acc[2 * rp][k] = (T)(flip ? -acc2[rp][k].x : acc2[rp][k].x);
          acc[2 * rp + 1][k] = (T)(flip ? -acc2[rp][k].y : acc2[rp][k].y);
        }
      }
    }

#ifdef LMS_TAIL_TRACE
    long long tt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    LMS_TT(0);  // sweep done
    // ---- combine partial sums across the CTAs that share this row tile ----------------------------
    // (recomputed here rather than kept in registers across the sweep)
    const int grp_threads = thin ? kThreads / groups : kThreads;  // threads that hold distinct rows
    const int grp = thin ? tid / grp_threads : 0;                 // column group of this thread (warp-uniform)
    const int gtid = tid - grp * grp_threads;                     // its index within the group
    if constexpr (kPairSplit) {
      if (thin && pair_split) {
        // both row pairs hold sums of the same two rows over the two halves of the window: first half + second half
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          acc[0][k] += acc[2][k];
          acc[1][k] += acc[3][k];
          acc[2][k] = T(0);
          acc[3][k] = T(0);
        }
      }
    }
    if (thin) {
      // the `split` column groups hold partial sums of the same rows: group 0 adds them in ascending group
      // (= ascending column-within-tile) order, one accumulator at a time through the reduction scratch
      T* red = reinterpret_cast<T*>(red_scratch);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          red[tid] = acc[r][k];
          __syncthreads();
          if (grp == 0) {
            T v = acc[r][k];
            for (int g = 1; g < groups; ++g) v += red[g * grp_threads + gtid];
            acc[r][k] = v;
          }
          __syncthreads();
        }
    }
    const long long cell_lo = rt_local * nJ;
    const long long cell_hi = cell_lo + nJ_this - 1;
    const long long cta_first = ((cell_lo + 1) * G - 1) / cells;
    const long long cta_last = ((cell_hi + 1) * G - 1) / cells;
    bool do_epilogue = true;
    if constexpr (CLUSTER) {
      namespace cg = cooperative_groups;
      cg::cluster_group cluster = cg::this_cluster();
      // every sweep of this CTA is over (one range per CTA in this mode): the tile buffers are free
      T* mine = reinterpret_cast<T*>(&tile[0][0][0]);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < NA; ++k) mine[k * BM + r * kThreads + tid] = acc[r][k];
      cluster.sync();
      do_epilogue = cluster.block_rank() == 0;
      if (do_epilogue) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < NA; ++k) acc[r][k] = T(0);
        // cluster rank = column segment: ascending ranks = ascending columns
#pragma unroll 4
        for (int ord = 0; ord < kClusterSize; ++ord) {
          const T* theirs = cluster.map_shared_rank(mine, ord);
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int k = 0; k < NA; ++k) acc[r][k] += theirs[k * BM + r * kThreads + tid];
        }
      }
      cluster.sync();  // nobody's shared memory goes away before rank 0 has read it
    } else if (cta_first != cta_last) {
      // Partial slots are indexed by the writing CTA, not by the row tile: a CTA leaves at most two partial
      // segments per launch -- the tile its range starts in (slot 2b) and, when that is a different one, the tile
      // it ends in (slot 2b + 1); whole tiles in between are finished alone.  2 * gridDim.x slots always suffice,
      // whatever the row-tile count (velocity fields with many more points than landmarks, subsets of a batch).
      const long long my_start = cells * blockIdx.x / G;
      const long long slot = 2LL * blockIdx.x + (my_start < cell_lo ? 1 : 0);
      T* mine = a.partials + slot * (NA * BM);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < NA; ++k) __stcg(mine + k * BM + r * kThreads + tid, acc[r][k]);
      LMS_TT(1);  // partial stores issued
      __threadfence();
      LMS_TT(2);  // fence done
      __syncthreads();
      const int nseg = (int)(cta_last - cta_first + 1);
      // one arrival counter per shared row tile, indexed by its first CTA (unique: a CTA that covers the first
      // cell of two row tiles covers the earlier one entirely, which is then not shared)
      int* counter = a.counters + cta_first;
      if (tid == 0) {
        const int prev = atomicAdd(counter, 1);
        const int last = prev == nseg - 1;
        if (last) *counter = 0;  // everyone has arrived: re-arm for the next launch
        s_last = last;
      }
      __syncthreads();
      do_epilogue = s_last != 0;
      LMS_TT(3);  // arrival known
      if (do_epilogue) {
        __threadfence();
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < NA; ++k) acc[r][k] = T(0);
        // ascending segment order = ascending columns; loads of several segments are in flight together.
        // Segment 0 is the first CTA's "ends here" slot unless that CTA's range starts exactly at this tile;
        // every later CTA starts inside this tile: its slot 2b.
        const long long first_start = cells * cta_first / G;
        const T* seg0 = a.partials + (2LL * cta_first) * (long long)(NA * BM);
        const long long first_off = first_start < cell_lo ? (long long)(NA * BM) : 0;
        if (a.combine_smem_segments > 0 && !CLUSTER) {
          // The launch has dynamic shared memory to spare (mid-size problems run two CTAs per SM): the segments land
          // there by bulk-async copies, a batch per round trip instead of four segments per round trip through
          // registers, and are added from shared memory in the same ascending order (bitwise the same sums).  The
          // partial sums were written through the generic proxy: fence before the async proxy reads them.
          T* land = reinterpret_cast<T*>(combine_smem);
          const int per_batch = a.combine_smem_segments;
          for (int base = 0; base < nseg; base += per_batch) {
            const int cnt = nseg - base < per_batch ? nseg - base : per_batch;
            if (tid == 0) {
              asm volatile("fence.proxy.async.global;" ::: "memory");
              mbar_expect_tx(&combine_bar, (unsigned)(cnt * NA * BM * sizeof(T)));
              for (int s2 = 0; s2 < cnt; ++s2) {
                const int ord = base + s2;
                const T* theirs = seg0 + (long long)ord * (2 * NA * BM) + (ord == 0 ? first_off : 0);
                bulk_g2s(land + (long long)s2 * (NA * BM), theirs, (unsigned)(NA * BM * sizeof(T)), &combine_bar);
              }
            }
            mbar_wait(&combine_bar, combine_parity);
            combine_parity ^= 1u;
            for (int s2 = 0; s2 < cnt; ++s2) {
              const T* theirs = land + (long long)s2 * (NA * BM);
#pragma unroll
              for (int r = 0; r < R; ++r)
#pragma unroll
                for (int k = 0; k < NA; ++k) acc[r][k] += theirs[k * BM + r * kThreads + tid];
            }
            __syncthreads();  // the landing zone is reused by the next batch (and by this CTA's next shared tile)
          }
        } else {
#pragma unroll kCombineUnroll
          for (int ord = 0; ord < nseg; ++ord) {
            const T* theirs = seg0 + (long long)ord * (2 * NA * BM) + (ord == 0 ? first_off : 0);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
              for (int k = 0; k < NA; ++k) acc[r][k] += __ldcg(theirs + k * BM + r * kThreads + tid);
          }
        }
      }
    }

    LMS_TT(4);  // segments added
    // ---- epilogue ----------------------------------------------------------------------------
    if (do_epilogue) {
      double hsum = 0.0, msum = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool second_pair = thin && pair_split && r >= 2;  // pair-split thin tile: rows live in the first pair only
        const long long row = row_of<R, PACKED>(rt, second_pair ? (r & 1) : r, gtid, grp_threads);
        const bool live = row < a.n_rows && grp == 0 && !second_pair;  // thin tile: group 0 holds the sums
        if constexpr (MODE == kVel) {
          if (live) {
            if (a.epi & kEpiEuler) {
              bool ok = true;
#pragma unroll
              for (int k = 0; k < D; ++k) {
                const T xn = Math<T>::add_rn(ri[r][k], Math<T>::mul_rn(a.dt, acc[r][k]));
                ok = ok && Math<T>::finite(xn);
                out_b[(long long)k * a.ostride + row] = xn;
              }
              if (!ok)
                atomicMin(diverged_b, ((unsigned long long)(unsigned)a.step << 32) | (unsigned long long)row);
            } else {
#pragma unroll
              for (int k = 0; k < D; ++k) out_b[(long long)k * a.ostride + row] = acc[r][k];
            }
          }
        } else if constexpr (MODE == kFwd) {
          T hq[D], hp[D];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            hq[k] = -a.inv_sig2 * acc[r][k];
            hp[k] = acc[r][D + k];
          }
          if (live) {
            if (a.epi & kEpiEuler) {
              bool ok = true;
              T qn[D];
#pragma unroll
              for (int k = 0; k < D; ++k) {
                // q_{t+1} = q_t + dt*hp ; p_{t+1} = p_t - dt*hq   (shooting.hpp:205-209)
                qn[k] = Math<T>::add_rn(ri[r][k], Math<T>::mul_rn(a.dt, hp[k]));
                const T pn = Math<T>::add_rn(ri[r][D + k], -Math<T>::mul_rn(a.dt, hq[k]));
                ok = ok && Math<T>::finite(qn[k]) && Math<T>::finite(pn);
                put_all<PEERS>(a, &out_b[(long long)k * a.ostride + row], qn[k]);
                put_all<PEERS>(a, &out_b[(long long)(D + k) * a.ostride + row], pn);
              }
              if (!ok) atomicMin(diverged_b, ((unsigned long long)(unsigned)a.step << 32) | 0xffffffffull);
              if (a.epi & kEpiFirstStep) {
#pragma unroll
                for (int k = 0; k < D; ++k) {
                  hp0_b[(long long)k * a.ostride + row] = hp[k];
                  hsum += (double)ri[r][D + k] * (double)hp[k];
                }
              }
              if (a.epi & kEpiLastStep) {
#pragma unroll
                for (int k = 0; k < D; ++k) {
                  const T tg = target_b[(long long)k * a.ostride + row];
                  const double df = (double)qn[k] - (double)tg;  // shooting.hpp:324-325
                  msum += df * df;
                  // alpha_T = 2*lambda*(q(1) - target), beta_T = 0   (shooting.hpp:290-296)
                  put_all<PEERS>(a, &adj_seed_b[(long long)k * a.ostride + row], Math<T>::mul_rn(a.two_lambda, qn[k] - tg));
                  put_all<PEERS>(a, &adj_seed_b[(long long)(D + k) * a.ostride + row], T(0));
                }
              }
            } else {
#pragma unroll
              for (int k = 0; k < D; ++k) {
                out_b[(long long)k * a.ostride + row] = hq[k];
                out_b[(long long)(D + k) * a.ostride + row] = hp[k];
                if (a.epi & kEpiFirstStep) hsum += (double)ri[r][D + k] * (double)hp[k];
              }
            }
          }
        } else {
          if (live) {
#pragma unroll
            for (int k = 0; k < D; ++k) {
              const T da = a.inv_sig2 * acc[r][k];
              const T dbeta = acc[r][D + k];
              if (a.epi & kEpiEuler) {
                // alpha += dt*d_alpha ; beta += dt*d_beta   (shooting.hpp:302-306)
                const T an = Math<T>::add_rn(ri[r][2 * D + k], Math<T>::mul_rn(a.dt, da));
                const T bn = Math<T>::add_rn(ri[r][3 * D + k], Math<T>::mul_rn(a.dt, dbeta));
                put_all<PEERS>(a, &out_b[(long long)k * a.ostride + row], an);
                put_all<PEERS>(a, &out_b[(long long)(D + k) * a.ostride + row], bn);
                if (a.epi & kEpiGradOut)  // grad = beta_0 + hp(q0,p0)   (shooting.hpp:311-313)
                  put_all<PEERS>(a, &grad_out_b[row * D + k],
                          (double)Math<T>::add_rn(bn, hp0_b[(long long)k * a.ostride + row]));
              } else {
                out_b[(long long)k * a.ostride + row] = da;
                out_b[(long long)(D + k) * a.ostride + row] = dbeta;
              }
            }
          }
        }
      }
      if constexpr (MODE == kFwd) {
        // block-uniform flags: every thread takes the same branch around the barriers in block_sum
        if (a.epi & kEpiFirstStep) {
          const double h = block_sum(hsum, red_scratch);
          if (tid == 0) put_all<PEERS>(a, &h_part_b[(long long)rt * R], h);  // indexed in 128-row units
        }
        if (a.epi & kEpiLastStep) {
          const double m = block_sum(msum, red_scratch);
          if (tid == 0) put_all<PEERS>(a, &mm_part_b[(long long)rt * R], m);
        }
      }
    }
#ifdef LMS_TAIL_TRACE
    __syncthreads();
    LMS_TT(5);  // epilogue done
    if (threadIdx.x == 0 && do_epilogue && cta_first != cta_last)
      printf("TT mode %d step %d cta %d rt %d nseg %d : stores %lld fence %lld arrive %lld combine %lld epilogue %lld\n", MODE, a.step,
             (int)blockIdx.x, (int)rt_local, (int)(cta_last - cta_first + 1), tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4]);
#endif
    c += tc1 - tc0;
  }
}

// ---------------------------------------------------------------------------------------------
// O(N) helpers
// ---------------------------------------------------------------------------------------------

// Row-major double (n x ncomp) -> ncomp planes of T, cast T(x) as registration.cpp:63 does, for `batch`
// problems (source stride n*ncomp doubles, destination stride dst_bs elements, divergence word stride div_bs).
// Non-finite inputs record divergence at `step` (integrate_forward's entry check, shooting.hpp:185-186).
template <typename T>
__global__ void aos_to_planes(const double* __restrict__ src, T* __restrict__ dst, long long stride, int n, int ncomp,
                              unsigned long long* diverged, int step, int batch = 1, long long dst_bs = 0,
                              long long div_bs = 0, const int* batch_ids = nullptr)
{
  const long long per = (long long)n * ncomp;
  const long long e_all = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e_all >= per * batch) return;
  const long long bc = e_all / per;
  const long long b = batch_ids != nullptr ? (long long)batch_ids[bc] : bc;
  const long long e = e_all - bc * per;
  const int i = (int)(e / ncomp);
  const int c = (int)(e - (long long)i * ncomp);
  const T v = (T)src[b * per + e];
  dst[b * dst_bs + (long long)c * stride + i] = v;
  if (diverged != nullptr && !isfinite(v))
    atomicMin(diverged + b * div_bs, ((unsigned long long)(unsigned)step << 32) | 0xffffffffull);
}

template <typename T>
__global__ void planes_to_aos(const T* __restrict__ src, long long stride, double* __restrict__ dst, int n,
                              int ncomp, int batch = 1, long long src_bs = 0)
{
  const long long per = (long long)n * ncomp;
  const long long e_all = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e_all >= per * batch) return;
  const long long b = e_all / per;
  const long long e = e_all - b * per;
  const int i = (int)(e / ncomp);
  const int c = (int)(e - (long long)i * ncomp);
  dst[e_all] = (double)src[b * src_bs + (long long)c * stride + i];
}

// Plane-to-plane copy of the live rows (device-resident snapshot 0 <- bound q0), per problem.
template <typename T>
__global__ void copy_planes(const T* __restrict__ src, long long sstride, T* __restrict__ dst, long long dstride,
                            int n, int ncomp, int batch = 1, long long src_bs = 0, long long dst_bs = 0)
{
  const long long per = (long long)n * ncomp;
  const long long e_all = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e_all >= per * batch) return;
  const long long b = e_all / per;
  const long long e = e_all - b * per;
  const int c = (int)(e / n);
  const int i = (int)(e - (long long)c * n);
  dst[b * dst_bs + (long long)c * dstride + i] = src[b * src_bs + (long long)c * sstride + i];
}

// Finite check of state planes (q0/p0 entry check, shooting.hpp:185-186).
template <typename T>
__global__ void check_finite_planes(const T* __restrict__ src, long long stride, int n, int ncomp,
                                    unsigned long long* diverged, int step)
{
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * ncomp) return;
  const int c = (int)(e / n);
  const int i = (int)(e - (long long)c * n);
  if (!isfinite(src[(long long)c * stride + i]))
    atomicMin(diverged, ((unsigned long long)(unsigned)step << 32) | 0xffffffffull);
}

// Row partition: this rank's divergence word into slot `rank` of every rank's word array ...
struct PeerList {
  int n;
  long long delta[kMaxPeers];  // byte distance to each peer's mapping of the exchange arena
};
template <int kUnused = 0>
__global__ void publish_diverged(const unsigned long long* __restrict__ mine, unsigned long long* slot, PeerList peers)
{
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const unsigned long long w = *mine;
  *slot = w;
  for (int k = 0; k < peers.n; ++k)
    *reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(slot) + peers.delta[k]) = w;
}
// ... and, after the exchange, the earliest record of all ranks back into the local word (first non-finite
// time step wins, as in the reference's sequential loop: shooting.hpp:210-211).
template <int kUnused = 0>
__global__ void min_diverged(const unsigned long long* __restrict__ words, int world, unsigned long long* out)
{
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned long long w = ~0ull;
  for (int r = 0; r < world; ++r) w = words[r] < w ? words[r] : w;
  *out = w;
}

// scalars[0..2] = {loss, kinetic, mismatch}: fixed ascending sum of the per-row-tile partials
// (loss = H + lambda*mismatch, shooting.hpp:286-288; H = 1/2 sum_i p_i . hp_i).  One block per problem;
// problem b's partials start at b * n_tiles, its scalars at b * 4 (the 4th word is the divergence record).
template <int kUnused = 0>
__global__ void finalize_scalars(const double* __restrict__ h_part, const double* __restrict__ mm_part,
                                 int n_tiles, double lambda, double* __restrict__ scalars,
                                 const int* batch_ids = nullptr)
{
  // the block's threads fetch the partials together (a single thread walking them pays an L2 round trip per
  // entry: 10 us at N = 20 000); thread 0 then adds them in ascending order, chunk by chunk
  constexpr int kChunk = 256;
  __shared__ double sh[kChunk], sm[kChunk];
  const long long b = batch_ids != nullptr ? (long long)batch_ids[blockIdx.x] : (long long)blockIdx.x;
  double h = 0.0, m = 0.0;
  for (int base = 0; base < n_tiles; base += kChunk) {
    const int cnt = n_tiles - base < kChunk ? n_tiles - base : kChunk;
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      sh[t] = h_part[b * n_tiles + base + t];
      sm[t] = mm_part[b * n_tiles + base + t];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int t = 0; t < cnt; ++t) {
        h += sh[t];
        m += sm[t];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  h *= 0.5;
  scalars[b * 4 + 1] = h;
  scalars[b * 4 + 2] = m;
  scalars[b * 4 + 0] = h + lambda * m;
}

// Strictly sequential double sum of squared differences over row-major-equivalent order
// (mismatch_sq, shooting.hpp:318-329): one thread, element order i-major then c, as the reference.
template <typename T>
__global__ void mismatch_sequential(const T* __restrict__ a, const T* __restrict__ b, long long stride, int n,
                                    int ncomp, double* __restrict__ out)
{
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < ncomp; ++c) {
      // explicit _rn ops: no FMA contraction, so the sum is bit-identical to the reference's loop
      const double d = __dadd_rn((double)a[(long long)c * stride + i], -(double)b[(long long)c * stride + i]);
      s = __dadd_rn(s, __dmul_rn(d, d));
    }
  *out = s;
}

// Registration metrics (landmarks.cpp:148-179): per-point Euclidean distance between two row-major double sets, in
// double with explicit _rn operations (no contraction), then average_dist's strictly sequential sum and max_dist's
// running maximum by one thread -- bit-identical to the reference's loops.
template <int kUnused = 0>
__global__ void point_distances(const double* __restrict__ a, const double* __restrict__ b, int n, int ncomp,
                                double* __restrict__ dist)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int c = 0; c < ncomp; ++c) {
    const double d = __dadd_rn(a[(long long)i * ncomp + c], -b[(long long)i * ncomp + c]);
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  dist[i] = __dsqrt_rn(s);
}
template <int kUnused = 0>
__global__ void avg_max_sequential(const double* __restrict__ dist, int n, double* __restrict__ out)
{
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double sum = 0.0, best = 0.0;
  for (int i = 0; i < n; ++i) {
    sum = __dadd_rn(sum, dist[i]);
    best = best > dist[i] ? best : dist[i];
  }
  out[0] = n > 0 ? __ddiv_rn(sum, (double)n) : 0.0;
  out[1] = best;
}

}  // namespace lms
