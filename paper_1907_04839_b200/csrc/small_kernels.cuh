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
//   columns   every CTA streams the whole landmark state through shared memory in chunks of 512 (fp64: 256)
//             columns, double buffered with bulk-async copies (cp.async.bulk + mbarrier: reads L2, so the state
//             other CTAs wrote before the barrier is seen without any L1 concern).  When a CTA has fewer slots
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
// largest n the persistent kernel is chosen for (measured crossover with the tiled path; LMS_SMALL_MAX_N overrides)
constexpr int kSmallMaxN32 = 4000;
constexpr int kSmallMaxN64 = 3000;

template <typename T>
struct SmallShape {
  static constexpr int kChunk = sizeof(T) == 4 ? 512 : 256;  // columns per staged chunk
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
  int n;
  int n_chunks;
  int timesteps;
  T kexp, inv_sig2, dt, two_lambda;
  double lambda;
};

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
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
}

// One time step for the rows this warp owns.  MODE kFwd: state -> out = next snapshot (Euler, shooting.hpp:205-211)
// with the first / last step extras; MODE kAdj: (state, adj_in) -> out = next adjoint state (:302-306).
template <typename T, int D, int MODE, int RP>
__device__ __forceinline__ void small_step(const SmallArgs<T>& a, const T* __restrict__ state,
                                           const T* __restrict__ adj_in, T* __restrict__ out, unsigned epi, int step_no,
                                           T* tile, T* part, unsigned long long* bars, unsigned& buf,
                                           unsigned& wait_parity, double& hsum, double& msum, const double* exp_tbl)
{
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
  auto issue = [&](int c, unsigned b) {  // thread 0 only
    mbar_expect_tx(&bars[b], (unsigned)(NC * CH * sizeof(T)));
#pragma unroll
    for (int k = 0; k < NC; ++k)
      bulk_g2s(tile + ((long long)b * NCMAX + k) * CH, plane(k) + (long long)c * CH, (unsigned)(CH * sizeof(T)), &bars[b]);
  };
  if (threadIdx.x == 0) issue(0, buf);  // buffer `buf` was last read before the previous __syncthreads

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

  // ---- sweep the columns, chunk by chunk ----
  for (int c = 0; c < a.n_chunks; ++c) {
    if (c + 1 < a.n_chunks && threadIdx.x == 0) issue(c + 1, buf ^ 1u);
    mbar_wait(&bars[buf], (wait_parity >> buf) & 1u);
    wait_parity ^= 1u << buf;
    const T* tb = tile + (long long)buf * NCMAX * CH;
    const int jstep = 32 * a.wc;
#pragma unroll 2
    for (int jj = wc * 32 + lane; jj < CH; jj += jstep) {
      T cj[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) cj[k] = tb[k * CH + jj];
      if constexpr (F32) {
        float2 cj2[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) cj2[k] = splat2((float)cj[k]);
#pragma unroll
        for (int i = 0; i < RP; ++i)
          if (i < my) pair_term_packed<D, MODE>(ri2[i], cj2, acc2[i], kexp2, ns2, neg1);
      } else {
#pragma unroll
        for (int i = 0; i < RP; ++i)
          if (i < my) pair_term<T, D, MODE>(rv[i][0], cj, acc[i][0], a.kexp, a.inv_sig2, exp_tbl);
      }
    }
    __syncthreads();
    buf ^= 1u;
  }

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
  if (a.wc > 1) {
    // the column warps of a slot meet in shared memory: ascending column part, lane by lane (RP == 1 here)
    if (wc > 0 && my > 0) {
      T* mine = part + ((long long)(wc - 1) * a.wr + (warp - wc * a.wr)) * (RS * NA * 32);
#pragma unroll
      for (int h = 0; h < RS; ++h)
#pragma unroll
        for (int k = 0; k < NA; ++k) mine[(h * NA + k) * 32 + lane] = acc[0][h][k];
    }
    __syncthreads();
    if (wc == 0 && my > 0) {
      for (int c = 1; c < a.wc; ++c) {
        const T* theirs = part + ((long long)(c - 1) * a.wr + warp) * (RS * NA * 32);
#pragma unroll
        for (int h = 0; h < RS; ++h)
#pragma unroll
          for (int k = 0; k < NA; ++k) acc[0][h][k] += theirs[(h * NA + k) * 32 + lane];
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
  __shared__ __align__(16) T part[(W - 1) * RS * Shape<kFwd, D>::kAcc * 32];  // column-warp partial sums
  __shared__ __align__(8) unsigned long long bars[2];
  __shared__ double exp_tbl[kExpEntries];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  if constexpr (sizeof(T) == 8) {
    if (threadIdx.x < kExpEntries) exp_tbl[threadIdx.x] = kExp2Table64[threadIdx.x * (64 / kExpEntries)];
  }
  // p0[i][c] = T(x[i*D+c])  (registration.cpp:61-63); non-finite p0 -> DivergedError(0) (shooting.hpp:185-186)
  {
    T* p_planes = a.traj + (long long)D * a.stride;
    const long long total = (long long)a.n * D;
    for (long long e = (long long)blockIdx.x * kThreadsHere + threadIdx.x; e < total;
         e += (long long)gridDim.x * kThreadsHere) {
      const int i = (int)(e / D);
      const int c = (int)(e - (long long)i * D);
      const T v = (T)a.x[e];
      p_planes[(long long)c * a.stride + i] = v;
      if (!Math<T>::finite(v)) atomicMin(a.diverged, 0xffffffffull);  // step 0
    }
  }
  unsigned bar_target = a.bar_base;
  small_grid_barrier(a.barrier, bar_target);

  unsigned buf = 0, wait_parity = 0;
  double hsum = 0.0, msum = 0.0;
  const int Tn = a.timesteps;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int GW = gridDim.x * a.wr;
  // forward Euler flow, T+1 snapshots kept for the adjoint (shooting.hpp:199-212)
  for (int t = 0; t < Tn; ++t) {
    const unsigned epi = kEpiEuler | (t == 0 ? kEpiFirstStep : 0u) | (t == Tn - 1 ? kEpiLastStep : 0u);
    small_step<T, D, kFwd, RP>(a, a.traj + (long long)t * a.snap_elems, nullptr,
                               a.traj + (long long)(t + 1) * a.snap_elems, epi, t + 1, tile, part, bars, buf,
                               wait_parity, hsum, msum, exp_tbl);
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
                               kEpiEuler | (t == 0 ? kEpiGradOut : 0u), t, tile, part, bars, buf, wait_parity, hsum, msum,
                               exp_tbl);
    T* tmp = adj_in;
    adj_in = adj_out;
    adj_out = tmp;
    if (t > 0) small_grid_barrier(a.barrier, bar_target);
  }
}

}  // namespace lms
