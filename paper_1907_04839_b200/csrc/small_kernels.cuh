// Small problems (N up to a few thousand landmarks): the whole objective evaluation -- p0 conversion, T forward
// Euler steps with the loss scalars, T adjoint steps, the final gradient (shooting.hpp:277-315) -- as ONE
// persistent cooperative kernel.
//
// At N = 1000 a time step is 1e6 pair evaluations, half a microsecond of B200 math; the 2T+2 dependent launches
// of the tiled path (pair_kernels.cuh) then cost ~10 us each whatever they compute: launch, row-operand and tile
// load latency, and the cross-CTA combine of the stream-K partial sums (slot write, fence, counter, re-read by
// the last CTA).  Here the mapping is transposed: a WARP owns a few rows and its 32 lanes split the columns, so
// a row's sums meet in a shuffle tree inside the warp -- no partial sums ever leave the SM, no combine pass, and
// the only global synchronisation is one grid barrier per time step.
//
//   rows      "slots" of RS rows (fp32: the 2 rows of a packed FFMA2 operand; fp64: 1 row) are dealt round-robin
//             to gridDim.x * WR "row warps"; a row warp keeps up to RP slots (row operands + 2D running sums per
//             row) in registers.  Row operands are warp-uniform.
//   columns   every CTA pulls the whole landmark state into shared memory in chunks of 512 (fp64: 256) columns with
//             bulk-async copies (cp.async.bulk + one mbarrier per chunk: reads L2, so the state other CTAs wrote
//             before the barrier is seen without any L1 concern).  All chunks of a step are in flight at once (up
//             to 8: N <= 4096 fp32 / 2048 fp64) and a warp waits only for the chunk it is about to read, so there
//             is no CTA-wide synchronisation inside a sweep.  When a CTA has fewer slots
//             than warps, WC warps share a slot: warp wc takes the 32-column groups wc, wc + WC, ... of every
//             chunk and lane l column l of a group (consecutive lanes, consecutive words: conflict-free LDS.32).
//   sums      per lane ascending columns, the WC column warps in ascending order through shared memory, then a
//             fixed xor-butterfly over the lanes: bitwise reproducible.
//   epilogue  lane r of the warp finishes the warp's row r with exactly the arithmetic of the tiled kernels'
//             epilogues (explicit _rn operations in the reference's expression order).
//   barrier   one monotonic arrival counter in global memory (the launch is cooperative: all CTAs are resident):
//             red.release to arrive, ld.acquire to poll; the host hands every launch the count it starts from.
#pragma once

#include "pair_kernels.cuh"

namespace lms {

constexpr int kSmallMaxWarps = 16;  // warps per CTA: 16 with one slot per row warp, 8 with several
// Largest n the persistent kernel is chosen for (LMS_SMALL_MAX_N overrides): the measured crossover with the tiled
// path in fp32 (ms per gradient, T = 10, persistent / tiled: N = 1000 0.107 / 0.217, 2000 0.195 / 0.265, 3000 0.364 /
// 0.414, 4000 0.564 / 0.550), and the shared-memory capacity for the staged state in fp64 (N = 2000 0.427 / 0.443).
constexpr int kSmallMaxN32 = 3500;
constexpr int kSmallMaxN64 = 2048;

// LMS_SMALL_TRACE: phase timestamps (globaltimer, ns) of CTA 0 into SmallArgs::trace -- a measurement build only
// (scripts/small_trace.py); the shipped library compiles the macro to nothing.
#ifdef LMS_SMALL_TRACE
#define LMS_TRACE_POINT(a, idx)                                                  \
  do {                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (a).trace != nullptr) {           \
      unsigned long long t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                      \
      (a).trace[(idx)] = t_;                                                     \
    }                                                                            \
  } while (0)
#else
#define LMS_TRACE_POINT(a, idx) \
  do {                          \
  } while (0)
#endif

template <typename T>
struct SmallShape {
  static constexpr int kChunk = sizeof(T) == 4 ? 512 : 256;  // columns per staged chunk
  static constexpr int kMaxChunks = 8;                        // chunk buffers (all resident during a step)
  static constexpr int kRowsPerSlot = sizeof(T) == 4 ? 2 : 1;
};

template <typename T>
struct SmallArgs {
  const double* x;        // p0, row-major double n x D (registration.cpp:61-63)
  T* traj;                // T+1 snapshots of 2D planes; snapshot 0's q planes already hold q0
  long long stride;       // plane length (zero-padded past n to a multiple of the chunk)
  long long snap_elems;   // elements between consecutive snapshots
  T* adj0;                // adjoint states (alpha, beta), ping-pong; the seed goes to adj0
  T* adj1;
  T* hp0;                 // H_p(q0, p0): D planes
  const T* target;        // D planes
  double* grad_out;       // row-major double n x D
  double* warp_part;      // 2 x (gridDim.x * wr): per-row-warp partials of sum p.hp and of the mismatch
  double* scalars;        // {loss, kinetic, mismatch}
  unsigned long long* diverged;
  unsigned* barrier;      // monotonic arrival counter
  unsigned bar_base;      // its value when this launch starts (the host counts gridDim.x * barriers per launch)
  int wr, wc;             // row warps per CTA x column warps per slot (wr * wc <= warps per CTA)
  unsigned long long* trace;  // LMS_SMALL_TRACE builds: 8 timestamps per step; else null
  int n;
  int n_chunks;
  int timesteps;
  T kexp, inv_sig2, dt, two_lambda;
  double lambda;
};

// Bulk copy global -> the same shared-memory offset of every CTA in cta_mask, completing on the mbarrier at the
// same offset in each of them.
__device__ __forceinline__ void bulk_g2s_multicast(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                                   unsigned short cta_mask)
{
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}

// All CTAs of the (cooperative) launch meet here.  Everything written before it -- by the generic proxy -- is
// visible after it to generic loads that bypass L1 (__ldcg) and to bulk-async copies (async proxy).  `target` is
// the counter value that means "everybody has arrived" (advanced by gridDim.x per barrier; wrap-safe compare).
__device__ __forceinline__ void small_grid_barrier(unsigned* bar, unsigned& target)
{
  target += gridDim.x;
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while ((int)(seen - target) < 0);
  }
  __syncthreads();
  asm volatile("fence.proxy.async.global;" ::: "memory");  // before this thread's bulk-async reads of that data
}

// One time step for the rows this warp owns.  MODE kFwd: state -> out = next snapshot (Euler, shooting.hpp:205-211)
// with the first / last step extras; MODE kAdj: (state, adj_in) -> out = next adjoint state (:302-306).
template <typename T, int D, int MODE, int RP>
__device__ __forceinline__ void small_step(const SmallArgs<T>& a, const T* __restrict__ state,
                                           const T* __restrict__ adj_in, T* __restrict__ out, unsigned epi, int step_no,
                                           T* tile, T* part, unsigned long long* bars, unsigned& phase,
                                           double& hsum, double& msum, const double* exp_tbl, int trace_base)
{
  LMS_TRACE_POINT(a, trace_base + 0);
  using S = Shape<MODE, D>;
  constexpr int NC = S::kColComps, NR = S::kRowComps, NA = S::kAcc;
  constexpr bool F32 = sizeof(T) == 4;
  constexpr int RS = SmallShape<T>::kRowsPerSlot;
  constexpr int CH = SmallShape<T>::kChunk;
  constexpr int NCMAX = 4 * D;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wc = warp / a.wr;            // column part of this warp (>= a.wc: a spare warp, no work)
  const int GW = gridDim.x * a.wr;       // row warps of the launch
  const int gw = blockIdx.x * a.wr + (warp - wc * a.wr);
  const int slots = (a.n + RS - 1) / RS;
  int my = 0;  // slots this warp works on: gw, gw + GW, ...
  if (wc < a.wc) {
#pragma unroll
    for (int i = 0; i < RP; ++i)
      if (gw + i * GW < slots) my = i + 1;
  }

  auto plane = [&](int k) -> const T* {
    if constexpr (MODE == kAdj)
      return k < 2 * D ? state + (long long)k * a.stride : adj_in + (long long)(k - 2 * D) * a.stride;
    else
      return state + (long long)k * a.stride;
  };
  // Every chunk of this step's state goes into its own buffer, all in flight together: one bulk copy per
  // (chunk, component plane), issued by lanes 0..NC-1 of warp 0 side by side; lane 0's arrive.expect_tx is a
  // chunk barrier's one arrival, so its phase cannot complete before every byte has been expected and delivered.
  // (All warps passed the grid barrier's __syncthreads since they last read these buffers.)
  // All 148 CTAs pull the same bytes at the same moment, and the L2 -> SM fabric (not latency) is what the first
  // chunk then waits for (measured: 96 KB per CTA take 3 us at N = 2000).  Launched as thread-block clusters, the
  // CTAs of a cluster share the fetch: piece (chunk, plane) is requested by ONE of them and multicast into the
  // same buffer offset of all (and completes on the same mbarrier offset of all), so L2 serves 1/cluster-size of
  // the traffic.
  unsigned cl_rank, cl_size;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(cl_rank));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(cl_size));
  if (warp == 0) {
    for (int c = 0; c < a.n_chunks; ++c) {
      if (lane == 0) mbar_expect_tx(&bars[c], (unsigned)(NC * CH * sizeof(T)));
      if (lane < NC) {
        T* dst = tile + ((long long)c * NCMAX + lane) * CH;
        const T* src = plane(lane) + (long long)c * CH;
        if (cl_size == 1)
          bulk_g2s(dst, src, (unsigned)(CH * sizeof(T)), &bars[c]);
        else if ((unsigned)(c * NC + lane) % cl_size == cl_rank)
          bulk_g2s_multicast(dst, src, (unsigned)(CH * sizeof(T)), &bars[c], (unsigned short)((1u << cl_size) - 1u));
      }
    }
  }

  // ---- row operands (warp-uniform; read past L1: other CTAs wrote them before the grid barrier) ----
  T rv[RP][RS][NR];
#pragma unroll
  for (int i = 0; i < RP; ++i)
#pragma unroll
    for (int h = 0; h < RS; ++h) {
      const long long row = (long long)(gw + i * GW) * RS + h;
      const bool ok = i < my && row < a.n;
#pragma unroll
      for (int k = 0; k < NR; ++k) rv[i][h][k] = ok ? __ldcg(plane(k) + row) : T(0);
    }
  T acc[RP][RS][NA];
  float2 ri2[F32 ? RP : 1][NR];
  float2 acc2[F32 ? RP : 1][NA];
  float2 kexp2, ns2, neg1;
  if constexpr (F32) {
#pragma unroll
    for (int i = 0; i < RP; ++i) {
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        const float lo = (float)rv[i][0][k], hi = (float)rv[i][RS - 1][k];
        ri2[i][k] = k < D ? make_float2(-lo, -hi) : make_float2(lo, hi);  // pair_term_packed takes -q_i
      }
#pragma unroll
      for (int k = 0; k < NA; ++k) acc2[i][k] = make_float2(0.f, 0.f);
    }
    kexp2 = splat2((float)a.kexp);
    ns2 = splat2(-(float)a.inv_sig2);
    neg1 = splat2(-1.f);
  } else {
#pragma unroll
    for (int i = 0; i < RP; ++i)
#pragma unroll
      for (int k = 0; k < NA; ++k) acc[i][0][k] = T(0);
  }

  // ---- sweep the columns: this warp's 32-column groups wc, wc + WC, ... of the whole staged state ----
  // U groups are loaded and evaluated together -- U independent dependency chains (LDS -> r^2 -> ex2 -> sums) in
  // one basic block, which is what lets the few warps of a CTA keep the FMA pipe busy.  A chunk is waited for the
  // first time one of its groups comes up.
  constexpr int GPC = CH / 32;  // groups per chunk
  constexpr int U = F32 ? (MODE == kAdj ? 2 : 4) : (MODE == kAdj ? 1 : 2);
  if (my > 0) {
    const int G = a.n_chunks * GPC;
    int waited = 0;  // chunks [0, waited) have landed
    auto need = [&](int g_last) {
      const int c = g_last / GPC;
      while (waited <= c) {
        mbar_wait(&bars[waited], phase);
        ++waited;
      }
    };
    auto col_ptr = [&](int g) -> const T* {
      const int c = g / GPC;
      return tile + (long long)c * NCMAX * CH + (g - c * GPC) * 32 + lane;
    };
    auto evaluate = [&](const T(&cj)[NC]) {
      if constexpr (F32) {
        float2 cj2[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) cj2[k] = splat2((float)cj[k]);
#pragma unroll
        for (int i = 0; i < RP; ++i)
          if (RP == 1 || i < my) pair_term_packed<D, MODE>(ri2[i], cj2, acc2[i], kexp2, ns2, neg1);
      } else {
#pragma unroll
        for (int i = 0; i < RP; ++i)
          if (RP == 1 || i < my) pair_term<T, D, MODE>(rv[i][0], cj, acc[i][0], a.kexp, a.inv_sig2, exp_tbl);
      }
    };
    int g = wc;
#ifdef LMS_SMALL_TRACE
    if (g < G) need(g);
    LMS_TRACE_POINT(a, trace_base + 1);
#endif
    for (; g + (U - 1) * a.wc < G; g += U * a.wc) {
      need(g + (U - 1) * a.wc);
      T cj[U][NC];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const T* cp = col_ptr(g + u * a.wc);
#pragma unroll
        for (int k = 0; k < NC; ++k) cj[u][k] = cp[k * CH];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) evaluate(cj[u]);
    }
    for (; g < G; g += a.wc) {
      need(g);
      T cj[NC];
      const T* cp = col_ptr(g);
#pragma unroll
      for (int k = 0; k < NC; ++k) cj[k] = cp[k * CH];
      evaluate(cj);
    }
  }
  phase ^= 1u;  // every chunk barrier completed one phase

  // ---- row sums: fixed butterfly over the lanes ----
  if constexpr (F32) {
#pragma unroll
    for (int i = 0; i < RP; ++i)
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        const bool flip = MODE == kFwd && k < D;  // the packed forward term accumulates -(p_i.p_j) K dx
        acc[i][0][k] = (T)(flip ? -acc2[i][k].x : acc2[i][k].x);
        acc[i][RS - 1][k] = (T)(flip ? -acc2[i][k].y : acc2[i][k].y);
      }
  }
  LMS_TRACE_POINT(a, trace_base + 2);
  if (a.wc > 1) {
    // the column warps of a slot meet in shared memory: ascending column part, lane by lane
    constexpr int PER = RP * RS * NA * 32;  // one warp's partial sums
    if (wc > 0 && my > 0) {
      T* mine = part + ((long long)(wc - 1) * a.wr + (warp - wc * a.wr)) * PER;
#pragma unroll
      for (int i = 0; i < RP; ++i)
#pragma unroll
        for (int h = 0; h < RS; ++h)
#pragma unroll
          for (int k = 0; k < NA; ++k) mine[((i * RS + h) * NA + k) * 32 + lane] = acc[i][h][k];
    }
    __syncthreads();
    if (wc == 0 && my > 0) {
      for (int c = 1; c < a.wc; ++c) {
        const T* theirs = part + ((long long)(c - 1) * a.wr + warp) * PER;
#pragma unroll
        for (int i = 0; i < RP; ++i)
#pragma unroll
          for (int h = 0; h < RS; ++h)
#pragma unroll
            for (int k = 0; k < NA; ++k) acc[i][h][k] += theirs[((i * RS + h) * NA + k) * 32 + lane];
      }
    }
    if (wc > 0) my = 0;  // only the first column warp of a slot finishes its rows
  }
#pragma unroll
  for (int i = 0; i < RP; ++i) {
    if (i < my) {
#pragma unroll
      for (int h = 0; h < RS; ++h)
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          T v = acc[i][h][k];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
          acc[i][h][k] = v;
        }
    }
  }

  LMS_TRACE_POINT(a, trace_base + 3);
  // ---- epilogue: lane i*RS+h finishes row (i, h) ----
#pragma unroll
  for (int i = 0; i < RP; ++i) {
#pragma unroll
    for (int h = 0; h < RS; ++h) {
      const long long row = (long long)(gw + i * GW) * RS + h;
      if (lane == i * RS + h && i < my && row < a.n) {
        const T* ri = rv[i][h];
        const T* sum = acc[i][h];
        if constexpr (MODE == kFwd) {
          bool ok = true;
          T qn[D];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const T hq = -a.inv_sig2 * sum[k];
            const T hp = sum[D + k];
            // q_{t+1} = q_t + dt*hp ; p_{t+1} = p_t - dt*hq   (shooting.hpp:205-209)
            qn[k] = Math<T>::add_rn(ri[k], Math<T>::mul_rn(a.dt, hp));
            const T pn = Math<T>::add_rn(ri[D + k], -Math<T>::mul_rn(a.dt, hq));
            ok = ok && Math<T>::finite(qn[k]) && Math<T>::finite(pn);
            out[(long long)k * a.stride + row] = qn[k];
            out[(long long)(D + k) * a.stride + row] = pn;
            if (epi & kEpiFirstStep) {
              a.hp0[(long long)k * a.stride + row] = hp;
              hsum += (double)ri[D + k] * (double)hp;
            }
          }
          if (!ok) atomicMin(a.diverged, ((unsigned long long)(unsigned)step_no << 32) | 0xffffffffull);
          if (epi & kEpiLastStep) {
#pragma unroll
            for (int k = 0; k < D; ++k) {
              const T tg = a.target[(long long)k * a.stride + row];
              const double df = (double)qn[k] - (double)tg;  // shooting.hpp:324-325
              msum += df * df;
              // alpha_T = 2*lambda*(q(1) - target), beta_T = 0   (shooting.hpp:290-296)
              a.adj0[(long long)k * a.stride + row] = Math<T>::mul_rn(a.two_lambda, qn[k] - tg);
              a.adj0[(long long)(D + k) * a.stride + row] = T(0);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const T da = a.inv_sig2 * sum[k];
            const T dbeta = sum[D + k];
            // alpha += dt*d_alpha ; beta += dt*d_beta   (shooting.hpp:302-306)
            const T an = Math<T>::add_rn(ri[2 * D + k], Math<T>::mul_rn(a.dt, da));
            const T bn = Math<T>::add_rn(ri[3 * D + k], Math<T>::mul_rn(a.dt, dbeta));
            out[(long long)k * a.stride + row] = an;
            out[(long long)(D + k) * a.stride + row] = bn;
            if (epi & kEpiGradOut)  // grad = beta_0 + hp(q0,p0)   (shooting.hpp:311-313)
              a.grad_out[row * D + k] = (double)Math<T>::add_rn(bn, __ldcg(a.hp0 + (long long)k * a.stride + row));
          }
        }
      }
    }
  }
}

template <typename T, int D, int RP, int W>
__global__ void __launch_bounds__(32 * W, 1) small_eval_kernel(const SmallArgs<T> a)
{
  constexpr int kThreadsHere = 32 * W;
  constexpr int RS = SmallShape<T>::kRowsPerSlot;
  extern __shared__ __align__(128) unsigned char small_smem[];
  T* tile = reinterpret_cast<T*>(small_smem);
  __shared__ __align__(16) T part[(W - 1) * RP * RS * Shape<kFwd, D>::kAcc * 32];  // column-warp partial sums
  __shared__ __align__(8) unsigned long long bars[SmallShape<T>::kMaxChunks];
  __shared__ double exp_tbl_all[sizeof(T) == 8 ? kExpTableDoubles : 1];  // fp64 only
  if (threadIdx.x == 0) {
    for (int c = 0; c < SmallShape<T>::kMaxChunks; ++c) mbar_init(&bars[c], 1);
    mbar_fence_init();
  }
  if constexpr (sizeof(T) == 8) {
    fill_exp_table(exp_tbl_all, threadIdx.x, kThreadsHere);
  }
  const double* exp_tbl = exp_table_of_lane(exp_tbl_all, threadIdx.x);
  // p0[i][c] = T(x[i*D+c])  (registration.cpp:61-63); non-finite p0 -> DivergedError(0) (shooting.hpp:185-186).
  // The divergence word is re-armed here (CTA 0, before the first barrier) and non-finite inputs are recorded
  // after it, so no separate memset launch precedes the kernel.
  bool bad_input = false;
  {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.diverged = ~0ull;
    T* p_planes = a.traj + (long long)D * a.stride;
    const long long total = (long long)a.n * D;
    for (long long e = (long long)blockIdx.x * kThreadsHere + threadIdx.x; e < total;
         e += (long long)gridDim.x * kThreadsHere) {
      const int i = (int)(e / D);
      const int c = (int)(e - (long long)i * D);
      const T v = (T)a.x[e];
      p_planes[(long long)c * a.stride + i] = v;
      bad_input = bad_input || !Math<T>::finite(v);
    }
  }
  unsigned bar_target = a.bar_base;
  small_grid_barrier(a.barrier, bar_target);
  if (bad_input) atomicMin(a.diverged, 0xffffffffull);  // step 0

  unsigned phase = 0;  // parity the chunk barriers complete next
  double hsum = 0.0, msum = 0.0;
  const int Tn = a.timesteps;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int GW = gridDim.x * a.wr;
  // forward Euler flow, T+1 snapshots kept for the adjoint (shooting.hpp:199-212)
  for (int t = 0; t < Tn; ++t) {
    const unsigned epi = kEpiEuler | (t == 0 ? kEpiFirstStep : 0u) | (t == Tn - 1 ? kEpiLastStep : 0u);
    small_step<T, D, kFwd, RP>(a, a.traj + (long long)t * a.snap_elems, nullptr,
                               a.traj + (long long)(t + 1) * a.snap_elems, epi, t + 1, tile, part, bars, phase, hsum,
                               msum, exp_tbl, 8 * t);
    LMS_TRACE_POINT(a, 8 * t + 4);
    if (t == Tn - 1) {
      // per-row-warp partials of the two double sums: lanes hold their rows' terms; fixed butterfly
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
        msum += __shfl_xor_sync(0xffffffffu, msum, off);
      }
      if (lane == 0 && warp < a.wr) {
        a.warp_part[blockIdx.x * a.wr + warp] = hsum;
        a.warp_part[GW + blockIdx.x * a.wr + warp] = msum;
      }
    }
    small_grid_barrier(a.barrier, bar_target);
    LMS_TRACE_POINT(a, 8 * t + 5);
  }
  // loss = H + lambda*mismatch, H = 1/2 sum_i p_i . hp_i  (shooting.hpp:286-288): warp 0 of CTA 0 adds the per-warp
  // partials (lane-strided ascending, then the fixed butterfly)
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double h = 0.0, m = 0.0;
    for (int w = lane; w < GW; w += 32) {
      h += __ldcg(a.warp_part + w);
      m += __ldcg(a.warp_part + GW + w);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      h += __shfl_xor_sync(0xffffffffu, h, off);
      m += __shfl_xor_sync(0xffffffffu, m, off);
    }
    if (lane == 0) {
      h *= 0.5;
      a.scalars[1] = h;
      a.scalars[2] = m;
      a.scalars[0] = h + a.lambda * m;
    }
  }
  // discrete adjoint sweep t = T-1 .. 0 (shooting.hpp:300-307), final gradient fused into the t = 0 step
  T* adj_in = a.adj0;
  T* adj_out = a.adj1;
  for (int t = Tn - 1; t >= 0; --t) {
    small_step<T, D, kAdj, RP>(a, a.traj + (long long)t * a.snap_elems, adj_in, adj_out,
                               kEpiEuler | (t == 0 ? kEpiGradOut : 0u), t, tile, part, bars, phase, hsum, msum, exp_tbl,
                               8 * (2 * Tn - 1 - t));
    LMS_TRACE_POINT(a, 8 * (2 * Tn - 1 - t) + 4);
    T* tmp = adj_in;
    adj_in = adj_out;
    adj_out = tmp;
    if (t > 0) small_grid_barrier(a.barrier, bar_target);
    LMS_TRACE_POINT(a, 8 * (2 * Tn - 1 - t) + 5);
  }
  // nobody leaves while a multicast of a cluster peer may still be landing in its shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace lms
