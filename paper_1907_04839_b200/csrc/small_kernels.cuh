// Small problems (N up to a few thousand landmarks): the whole objective evaluation -- p0 conversion, T forward
// Euler steps with the loss scalars, T adjoint steps, the final gradient (shooting.hpp:277-315) -- as ONE
// persistent cooperative kernel.
//
// At N = 1000 a time step is 1e6 pair evaluations, half a microsecond of B200 math; the 2T+2 dependent launches
// of the tiled path (pair_kernels.cuh) then cost ~10 us each whatever they compute: launch, row-operand and tile
// load latency, and the cross-CTA combine of the stream-K partial sums (slot write, fence, counter, re-read by
// the last CTA).  Here the mapping is transposed: a WARP works on one "slot" of rows at a time and its 32 lanes
// split the columns, so a row's sums meet in a shuffle tree inside the warp -- no partial sums ever leave the SM,
// no combine pass, and the only global synchronisation is one grid barrier per time step.
//
//   rows      "slots" of RS rows (fp32: the 2 rows of a packed FFMA2 operand; fp64: 1 row) are dealt to the CTAs
//             in contiguous, equal (+-1) runs.  Row operands are warp-uniform registers.
//   columns   every CTA pulls the whole landmark state into shared memory, one contiguous array per component,
//             in chunks of 2048 (fp64: 1024) columns with bulk-async copies (cp.async.bulk + one mbarrier per chunk:
//             reads L2, so the state other CTAs wrote before the barrier is seen without any L1 concern).  All
//             chunks of a window are in flight at once and a warp waits only for the chunks it is about to read,
//             so there is no CTA-wide synchronisation inside a window.  A window is what fits 192 KB: 8192 columns
//             (fp64: 4096) of the forward sweep's 2D components, half as many of the adjoint's 4D; wider problems
//             sweep two adjoint windows per step, their pieces parked separately and added in column order.
//   work      a CTA with s slots has s x G work items (slot, group of 32 columns), slot-major; its 16 warps take
//             equal contiguous runs of that list (stream-K inside the CTA), so every warp is busy for the same
//             time whatever s is.  A run touches at most three slots: up to three "pieces" (slot, group range) per
//             warp and window.
//             Inside a piece lane l takes U consecutive columns of each block of 32 U (one LDS.128 / LDS.64 per
//             component serves U pairs per row: U independent dependency chains in one basic block).
//   sums      per lane ascending columns; a fixed transposing shuffle tree over the lanes of the piece; the
//             pieces of a slot in ascending column order (one thread per row adds them): bitwise reproducible.
//   epilogue  thread r of the CTA finishes the CTA's row r with exactly the arithmetic of the tiled kernels'
//             epilogues (explicit _rn operations in the reference's expression order); rows are contiguous per
//             CTA, so the stores coalesce.
//   barrier   one monotonic arrival counter in global memory (the launch is cooperative: all CTAs are resident):
//             red.release to arrive, ld.acquire to poll; the host hands every launch the count it starts from.
#pragma once

#include "pair_kernels.cuh"

namespace lms {

#ifndef LMS_SMALL_WARPS
#define LMS_SMALL_WARPS 16  // measured: 12 warps (168 registers) are 1-3 % faster in fp32 and 1-2 % slower in fp64; 8 lose
#endif
constexpr int kSmallWarps = LMS_SMALL_WARPS;  // warps per CTA
constexpr int kSmallMaxWarps = kSmallWarps;
constexpr int kSmallMaxSlots = 32;  // slots per CTA (a warp's run of work then spans at most three slots)
constexpr int kSmallMaxPieces = 3;  // ... pieces per warp and window
constexpr int kSmallMaxWindows = 2; // adjoint windows (the forward sweep has one)
// Largest n the persistent kernel is chosen for (LMS_SMALL_MAX_N overrides): fp32 the capacity (measured on B200,
// persistent / tiled ms per gradient: N = 5000 0.635 / 0.704, 6000 0.879 / 0.941, 7000 1.129 / 1.192, 8192 1.490 / 1.509);
// fp64 the crossover with the tiled path (N = 2049 0.380 / 0.507, 3000 0.685 / 0.715, 4096 1.144 / 1.110).
constexpr int kSmallMaxN32 = 8192;
constexpr int kSmallMaxN64 = 3400;
// hard limit: one forward window = two adjoint windows (SmallShape)
constexpr int kSmallCapacity32 = 8192;
constexpr int kSmallCapacity64 = 4096;

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
  // The staged state: 192 KB of shared memory hold every component of 4096 (fp64: 2048) columns in the adjoint sweep
  // (4D components) and of twice as many in the forward sweep (2D components).  A sweep stages one such WINDOW at a
  // time, in chunks with one mbarrier each; problems wider than a window sweep several, one after the other.
#ifndef LMS_SMALL_CHUNKS
#define LMS_SMALL_CHUNKS 2  // chunks per adjoint window.  Measured on B200 (ms per gradient, 16 / 8 / 4 / 2 / 1 chunks): fp32 N = 2000 0.206 /
                            // 0.179 / 0.163 / 0.162 / 0.161, N = 4000 0.520 / 0.462 / 0.427 / 0.411 / 0.415; fp64 N = 2000 0.447 / 0.384 / 0.347 / 0.332 / 0.334
#endif
  static constexpr int kCols = sizeof(T) == 4 ? 4096 : 2048;   // columns per component in an adjoint window
  static constexpr int kColsFwd = 2 * kCols;                   // ... in a forward window
  static constexpr int kChunk = kCols / LMS_SMALL_CHUNKS;      // columns per staged chunk
  static constexpr int kMaxChunks = kColsFwd / kChunk;         // chunk barriers
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
  double* warp_part;      // 2 x (gridDim.x * kSmallWarps): per-warp partials of sum p.hp and of the mismatch
  double* scalars;        // {loss, kinetic, mismatch}
  unsigned long long* diverged;
  unsigned* barrier;      // monotonic arrival counter
  unsigned bar_base;      // its value when this launch starts (the host counts gridDim.x * barriers per launch)
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

// mbar_wait on a precomputed shared-window address (keeps the generic -> shared conversion out of the sweep)
__device__ __forceinline__ void mbar_wait_u32(unsigned bar, unsigned parity)
{
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LMS_WAITU_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra LMS_DONEU_%=;\n"
      "bra LMS_WAITU_%=;\n"
      "LMS_DONEU_%=:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// All CTAs of the (cooperative) launch meet here.  Everything written before it -- by the generic proxy -- is
// visible after it to generic loads that bypass L1 (__ldcg) and to bulk-async copies (async proxy).  `target` is
// the counter value that means "everybody has arrived" (wrap-safe compare).
// Hierarchical when LMS_SMALL_CLUSTER_BARRIER is set: the CTAs of a cluster meet in the hardware cluster barrier,
// ONE of them arrives at / polls the global counter (an eighth of the same-address atomics and pollers), and a
// second cluster barrier releases the rest; release / acquire are cumulative, so the chain CTA -> cluster barrier ->
// red.release.gpu -> ld.acquire.gpu -> cluster barrier -> CTA orders every CTA's writes before every CTA's reads.
#ifndef LMS_SMALL_CLUSTER_BARRIER
#define LMS_SMALL_CLUSTER_BARRIER 0
#endif
__device__ __forceinline__ void small_grid_barrier(unsigned* bar, unsigned& target)
{
  asm volatile("fence.proxy.async.global;" ::: "memory");
#if LMS_SMALL_CLUSTER_BARRIER
  unsigned cl_rank, cl_size;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(cl_rank));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(cl_size));
  target += gridDim.x / cl_size;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (cl_rank == 0 && threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while ((int)(seen - target) < 0);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#else
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while ((int)(seen - target) < 0);
  }
  __syncthreads();
#endif
  asm volatile("fence.proxy.async.global;" ::: "memory");  // before this thread's bulk-async reads of that data
}

// Sum NV per-lane values over the 32 lanes with a fixed "transposing" shuffle tree: while the count is even, lanes
// l and l ^ off split the values between them (each keeps one half and adds the partner's copy of it), then plain
// butterflies finish.  On return v[0 .. count) hold complete sums of the values [first, first + count) on every
// lane; the lanes with (lane & live_mask) == 0 between them hold every value exactly once.
template <typename T, int NV>
struct LaneTree {
  static constexpr int count_after(int c, int stages) { return stages == 0 ? c : count_after(c % 2 == 0 ? c / 2 : c, stages - 1); }
  static constexpr int kCount = count_after(NV, 5);
  static __device__ __forceinline__ void run(T (&v)[NV], int lane, int& first, unsigned& live_mask)
  {
    first = 0;
    live_mask = 0;
    int count = NV;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      if (count % 2 == 0) {
        const int half = count / 2;
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < NV / 2; ++j) {
          if (j < half) {
            const T send = up ? v[j] : v[j + half];
            const T keep = up ? v[j + half] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        if (up) first += half;
        count = half;
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (j < count) v[j] += __shfl_xor_sync(0xffffffffu, v[j], off);
        live_mask |= (unsigned)off;
      }
    }
  }
};

// Vector loads of U consecutive columns of one staged component (16 bytes per load at most).
template <typename T, int U>
__device__ __forceinline__ void load_cols(const T* p, T (&v)[U])
{
  constexpr int VW = (int)(16 / sizeof(T)) < U ? (int)(16 / sizeof(T)) : U;  // elements per load
  if constexpr (VW == 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = p[u];
  } else {
#pragma unroll
    for (int b = 0; b < U / VW; ++b) {
      T w[VW];
      ColVec<T, VW>::load(p + b * VW, w);
#pragma unroll
      for (int u = 0; u < VW; ++u) v[b * VW + u] = w[u];
    }
  }
}

// columns a lane evaluates together in the forward / adjoint sweep (independent dependency chains per basic block)
#ifndef LMS_SMALL_UF
#define LMS_SMALL_UF 4
#endif
#ifndef LMS_SMALL_UA
#define LMS_SMALL_UA 2
#endif
#ifndef LMS_SMALL_UF64
#define LMS_SMALL_UF64 2
#endif
#ifndef LMS_SMALL_UA64
#define LMS_SMALL_UA64 1
#endif

// What a thread needs to know about the CTA's work list; the same for every time step, so it is worked out once
// per launch (the per-step code between two sweeps is latency-critical and mostly cold in the instruction cache:
// it is kept as short as possible).
struct SmallWarpPlan {  // a warp's run of one window's work list: up to three pieces (slot, groups [g0, g1))
  int n_pieces;
  int pid0;  // index of the warp's first piece among the CTA's pieces of that window (ascending work-list order)
  int sl[kSmallMaxPieces], g0[kSmallMaxPieces], g1[kSmallMaxPieces];
};
struct SmallEpiPlan {  // epilogue thread: its slot's pieces of that window are [first, first + count)
  int first, count;
};

// The work list of one window (s_b slots x Gw groups, slot-major) cut into sixteen equal contiguous runs.  Two
// phases around one __syncthreads, so that the integer divisions are done once per run and not by every thread (the
// plan is worked out once per launch, but on a 0.1 ms evaluation a few microseconds count): thread w < 16 describes
// run w; then lane 0 of every warp records its warp's pieces and epilogue thread t (component t % D of the CTA's
// row t / D) finds where its slot's pieces lie.
struct SmallRun {
  int r0, r1;  // items [r0, r1) of the window's work list
  int s0, s1;  // first and last slot touched (s1 <= s0 + 2); r1 == r0: an empty run (fewer items than warps)
};
template <int RS, int D>
__device__ __forceinline__ void small_plan_window(int Gw, const SmallRun* runs, SmallWarpPlan* wplan, SmallEpiPlan* eplan)
{
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  if (lane == 0) {
    SmallWarpPlan mine;
    const SmallRun r = runs[warp];
    mine.n_pieces = r.s1 - r.s0 + 1;  // 0 for an empty run
    mine.pid0 = 0;
    for (int w = 0; w < warp; ++w) mine.pid0 += runs[w].s1 - runs[w].s0 + 1;
#pragma unroll
    for (int j = 0; j < kSmallMaxPieces; ++j) {
      const int sl = r.s0 + j;
      const bool on = sl <= r.s1;
      mine.sl[j] = on ? sl : 0;
      mine.g0[j] = on && j == 0 ? r.r0 - r.s0 * Gw : 0;
      mine.g1[j] = on ? (sl == r.s1 ? r.r1 - r.s1 * Gw : Gw) : 0;
    }
    wplan[warp] = mine;
  }
  if ((int)threadIdx.x < kSmallMaxSlots * RS * D) {
    const int my_slot = (int)threadIdx.x / (RS * D);
    int first = 0, count = 0;
    for (int w = 0; w < kSmallWarps; ++w) {
      const int s0 = runs[w].s0, s1 = runs[w].s1;
      for (int sl = s0; sl <= s1; ++sl) {
        if (sl < my_slot) ++first;
        if (sl == my_slot) ++count;
      }
    }
    eplan[threadIdx.x].first = first;
    eplan[threadIdx.x].count = count;
  }
}

// What a step needs to know about the CTA's share of the problem; worked out once per launch (the per-step code
// between two sweeps is latency-critical and mostly cold in the instruction cache: it is kept as short as possible).
struct SmallCtx {
  int slot0, s_b;                      // the CTA's slots [slot0, slot0 + s_b)
  int adj_windows;                     // windows of the adjoint sweep (1 or 2); the forward sweep has one
  const SmallWarpPlan* wplan;          // [1 + kSmallMaxWindows][kSmallWarps]: forward, adjoint window 0, adjoint window 1
  const SmallEpiPlan* eplan;           // [1 + kSmallMaxWindows][epilogue threads]
  int epi_stride;                      // epilogue threads per plan
};

// One time step for this CTA's rows.  MODE kFwd: state -> out = next snapshot (Euler, shooting.hpp:205-211) with
// the first / last step extras; MODE kAdj: (state, adj_in) -> out = next adjoint state (:302-306).
template <typename T, int D, int MODE, int RS, int MAXW>
__device__ __forceinline__ void small_step(const SmallArgs<T>& a, const SmallCtx& cx, const T* __restrict__ state,
                                           const T* __restrict__ adj_in, T* __restrict__ out, unsigned epi, int step_no,
                                           T* tile, T* part, T* rowbuf, unsigned long long* bars, unsigned& phase_bits,
                                           double& hsum, double& msum, const double* exp_tbl, int trace_base)
{
  LMS_TRACE_POINT(a, trace_base + 0);
  using S = Shape<MODE, D>;
  constexpr int NC = S::kColComps, NR = S::kRowComps, NA = S::kAcc;
  constexpr bool F32 = sizeof(T) == 4;
  constexpr int CH = SmallShape<T>::kChunk;
  constexpr int NTOT = MODE == kAdj ? SmallShape<T>::kCols : SmallShape<T>::kColsFwd;  // columns per window
  constexpr int WCH = NTOT / CH;  // chunks per window
  constexpr int GPC = CH / 32;    // 32-column groups per chunk
  constexpr int GPW = NTOT / 32;  // ... per window
  constexpr int NV = RS * NA;     // sums per slot
  constexpr int NRMAX = 4 * D;    // row operands per row in the adjoint sweep (rowbuf is sized for it)
  constexpr int PMAX = kSmallWarps * kSmallMaxPieces;  // pieces per window
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // MAXW == 1: the whole state fits one adjoint window (N <= 4096 fp32 / 2048 fp64): no window loop, and the forward
  // and adjoint sweeps share one work plan
  const int n_windows = (MODE == kAdj && MAXW > 1) ? cx.adj_windows : 1;
  const int plan0 = (MODE == kAdj && MAXW > 1) ? 1 : 0;
  const int G = (a.n + 31) / 32;  // live groups

  auto plane = [&](int k) -> const T* {
    if constexpr (MODE == kAdj)
      return k < 2 * D ? state + (long long)k * a.stride : adj_in + (long long)(k - 2 * D) * a.stride;
    else
      return state + (long long)k * a.stride;
  };
  const unsigned bars_u32 = smem_u32(bars);

#pragma unroll 1
  for (int win = 0; win < n_windows; ++win) {
    // everyone is done reading the previous window (the first window of a step: the grid barrier's __syncthreads)
    if (win > 0) __syncthreads();
    // Every chunk of the window is fetched at once: one bulk copy per (chunk, component plane), issued by lanes
    // 0..NC-1 of the last warp side by side; lane 0's arrive.expect_tx is a chunk barrier's one arrival, so its phase
    // cannot complete before every byte has been expected and delivered.  Launched as thread-block clusters, the CTAs
    // of a cluster share the fetch: piece (chunk, plane) is requested by ONE of them and multicast into the same
    // buffer offset of all (and completes on the same mbarrier offset of all).
    const int chunk0 = win * WCH;
    const int n_ch = a.n_chunks - chunk0 < WCH ? a.n_chunks - chunk0 : WCH;
    if (warp == kSmallWarps - 1) {
      unsigned cl_rank, cl_size;
      asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(cl_rank));
      asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(cl_size));
#pragma unroll 1
      for (int c = 0; c < n_ch; ++c) {
        // the last chunk ends with the plane (planes are padded to 512 columns, chunks may be longer)
        const long long col = (long long)(chunk0 + c) * CH;
        const long long left = a.stride - col;
        const unsigned cols = (unsigned)(left < CH ? left : CH);
        if (lane == 0) mbar_expect_tx(&bars[c], (unsigned)(NC * cols * sizeof(T)));
        if (lane < NC) {
          T* dst = tile + (long long)lane * NTOT + (long long)c * CH;
          const T* src = plane(lane) + col;
          if (cl_size == 1)
            bulk_g2s(dst, src, (unsigned)(cols * sizeof(T)), &bars[c]);
          else if ((unsigned)(c * NC + lane) % cl_size == cl_rank)
            bulk_g2s_multicast(dst, src, (unsigned)(cols * sizeof(T)), &bars[c], (unsigned short)((1u << cl_size) - 1u));
        }
      }
    } else if (win == 0) {
      // ---- row operands of the CTA's rows: one value per thread (of the other warps), read past L1 (other CTAs
      // wrote them before the grid barrier) and parked in shared memory for the sweeps and the epilogue; the fetch
      // overlaps the chunk copies ----
      for (int t = threadIdx.x; t < cx.s_b * RS * NR; t += 32 * (kSmallWarps - 1)) {
        const int rl = t / NR, k = t - rl * NR;  // row of the CTA, component
        const long long row = (long long)cx.slot0 * RS + rl;
        // [slot][component][row of the slot]: a slot's packed (row 0, row 1) operand is one 8-byte word
        rowbuf[((rl / RS) * NRMAX + k) * RS + (rl % RS)] = row < a.n ? __ldcg(plane(k) + row) : T(0);
      }
    }
    if (win == 0) {
      __syncthreads();
      LMS_TRACE_POINT(a, trace_base + 1);
    }

    // ---- the warp's pieces of this window: (slot, groups [g0, g1)), groups counted from the window's first ----
    const SmallWarpPlan wp = cx.wplan[(plan0 + win) * kSmallWarps + warp];
    constexpr int U = F32 ? (MODE == kAdj ? (RS == 4 ? 1 : LMS_SMALL_UA) : (RS == 4 ? 2 : LMS_SMALL_UF))
                          : (MODE == kAdj ? LMS_SMALL_UA64 : LMS_SMALL_UF64);
    int waited = 0;  // chunks [0, waited) of this window have landed
    // A run that wraps from the tail of one slot into the head of the next is swept head first: the head starts at
    // the window's first column, whose chunk lands first, while the tail's chunks are the last to arrive (a warp
    // waits only for the chunks it reads).  The epilogue adds a slot's pieces in ascending column order whatever
    // order they were swept in.
#pragma unroll 1
    for (int pc = wp.n_pieces - 1; pc >= 0; --pc) {
      const int sl = pc == 0 ? wp.sl[0] : (pc == 1 ? wp.sl[1] : wp.sl[2]);
      const int g0 = pc == 0 ? wp.g0[0] : (pc == 1 ? wp.g0[1] : wp.g0[2]);
      const int g1 = pc == 0 ? wp.g1[0] : (pc == 1 ? wp.g1[1] : wp.g1[2]);
      T rv[RS][NR];  // warp-uniform
      if constexpr (RS > 1) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          T v[RS];
          load_cols<T, RS>(rowbuf + (sl * NRMAX + k) * RS, v);
#pragma unroll
          for (int h = 0; h < RS; ++h) rv[h][k] = v[h];
        }
      } else {
#pragma unroll
        for (int k = 0; k < NR; ++k) rv[0][k] = rowbuf[sl * NRMAX + k];
      }

      constexpr int RPK = F32 ? RS / 2 : 1;  // packed row pairs per slot (fp32)
      T acc[NV];
      float2 ri2[RPK][NR], acc2[RPK][NA];
      float2 kexp2, ns2, neg1;
      if constexpr (F32) {
#pragma unroll
        for (int rp = 0; rp < RPK; ++rp) {
#pragma unroll
          for (int k = 0; k < NR; ++k) {
            const float lo = (float)rv[2 * rp][k], hi = (float)rv[2 * rp + 1][k];
            ri2[rp][k] = k < D ? make_float2(-lo, -hi) : make_float2(lo, hi);  // pair_term_packed takes -q_i
          }
#pragma unroll
          for (int k = 0; k < NA; ++k) acc2[rp][k] = make_float2(0.f, 0.f);
        }
        kexp2 = splat2((float)a.kexp);
        ns2 = splat2(-(float)a.inv_sig2);
        neg1 = splat2(-1.f);
      } else {
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] = T(0);
      }
      auto evaluate = [&](const T(&cj)[NC]) {
        if constexpr (F32) {
          float2 cj2[NC];
#pragma unroll
          for (int k = 0; k < NC; ++k) cj2[k] = splat2((float)cj[k]);
#pragma unroll
          for (int rp = 0; rp < RPK; ++rp) pair_term_packed<D, MODE>(ri2[rp], cj2, acc2[rp], kexp2, ns2, neg1);
        } else {
          pair_term<T, D, MODE>(rv[0], cj, acc, a.kexp, a.inv_sig2, exp_tbl);
        }
      };
      // The piece chunk by chunk: a chunk is waited for once (they land roughly in order, so everything up to it is
      // waited for), then its groups are swept without further checks -- blocks of U groups (lane l takes the U
      // consecutive columns 32 U b + U l ..: one vector load per component), then single groups up to the chunk's
      // end.  Chunks start at multiples of GPC groups, so only a piece's first chunk can have such a remainder.
      // Counters and offsets are warp-uniform (uniform datapath: no vector-register reads in the loop control).
      const T* lane_blk = tile + lane * U;
      const T* lane_one = tile + lane;
      int g = g0;
#pragma unroll 1
      while (g < g1) {
        const int c = (int)((unsigned)g / (unsigned)GPC);
        if (c >= waited) {
#pragma unroll 1
          do {
            mbar_wait_u32(bars_u32 + 8u * (unsigned)waited, (phase_bits >> waited) & 1u);
            ++waited;
          } while (waited <= c);
        }
        const int gend = (c + 1) * GPC < g1 ? (c + 1) * GPC : g1;
#pragma unroll 1
        for (; g + U <= gend; g += U) {
          const T* cp = lane_blk + g * 32;
          T cj[U][NC];
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            T v[U];
            load_cols<T, U>(cp + k * NTOT, v);
#pragma unroll
            for (int u = 0; u < U; ++u) cj[u][k] = v[u];
          }
#pragma unroll
          for (int u = 0; u < U; ++u) evaluate(cj[u]);
        }
        if constexpr (U > 1) {
#pragma unroll 1
          for (; g < gend; ++g) {
            const T* cs = lane_one + g * 32;
            T cj[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) cj[k] = cs[k * NTOT];
            evaluate(cj);
          }
        }
      }

      // ---- the piece's sums over the lanes (fixed tree), parked for the slot's epilogue threads ----
      if constexpr (F32) {
#pragma unroll
        for (int rp = 0; rp < RPK; ++rp)
#pragma unroll
          for (int k = 0; k < NA; ++k) {
            const bool flip = MODE == kFwd && k < D;  // the packed forward term accumulates -(p_i.p_j) K dx
            acc[(2 * rp) * NA + k] = (T)(flip ? -acc2[rp][k].x : acc2[rp][k].x);
            acc[(2 * rp + 1) * NA + k] = (T)(flip ? -acc2[rp][k].y : acc2[rp][k].y);
          }
      }
      int first;
      unsigned live_mask;
      LaneTree<T, NV>::run(acc, lane, first, live_mask);
      if ((lane & live_mask) == 0) {
        T* mine = part + (win * PMAX + wp.pid0 + pc) * NV;
#pragma unroll
        for (int j = 0; j < LaneTree<T, NV>::kCount; ++j) mine[first + j] = acc[j];
      }
    }
    // every chunk barrier of this window completed one phase (whether or not this warp waited for it)
    phase_bits ^= (1u << n_ch) - 1u;
  }
  (void)G;
  (void)GPW;
  LMS_TRACE_POINT(a, trace_base + 2);
  __syncthreads();
  LMS_TRACE_POINT(a, trace_base + 3);

  // ---- epilogue: thread t finishes component t % D of the CTA's row t / D ----
  const int t = threadIdx.x;
  if (t < cx.s_b * RS * D) {
    const int rl = t / D, k = t - rl * D;
    const int sl = rl / RS, h = rl - sl * RS;
    const long long row = (long long)cx.slot0 * RS + rl;
    if (row < a.n) {
      // the slot's pieces in ascending column order: window by window
      T s0 = T(0), s1 = T(0);
#pragma unroll 1
      for (int win = 0; win < n_windows; ++win) {
        const SmallEpiPlan ep = cx.eplan[(plan0 + win) * cx.epi_stride + t];
        const T* theirs = part + (win * PMAX + ep.first) * NV + h * NA + k;
#pragma unroll 1
        for (int i = 0; i < ep.count; ++i, theirs += NV) {
          s0 += theirs[0];
          s1 += theirs[D];
        }
      }
      const T* ri = rowbuf + sl * NRMAX * RS + h;  // component c of this row: ri[c * RS]
      if constexpr (MODE == kFwd) {
        const T hq = -a.inv_sig2 * s0;
        const T hp = s1;
        // q_{t+1} = q_t + dt*hp ; p_{t+1} = p_t - dt*hq   (shooting.hpp:205-209)
        const T pk = ri[(D + k) * RS];
        const T qn = Math<T>::add_rn(ri[k * RS], Math<T>::mul_rn(a.dt, hp));
        const T pn = Math<T>::add_rn(pk, -Math<T>::mul_rn(a.dt, hq));
        out[(long long)k * a.stride + row] = qn;
        out[(long long)(D + k) * a.stride + row] = pn;
        if (!(Math<T>::finite(qn) && Math<T>::finite(pn)))
          atomicMin(a.diverged, ((unsigned long long)(unsigned)step_no << 32) | 0xffffffffull);
        if (epi & kEpiFirstStep) {
          a.hp0[(long long)k * a.stride + row] = hp;
          hsum += (double)pk * (double)hp;
        }
        if (epi & kEpiLastStep) {
          const T tg = a.target[(long long)k * a.stride + row];
          const double df = (double)qn - (double)tg;  // shooting.hpp:324-325
          msum += df * df;
          // alpha_T = 2*lambda*(q(1) - target), beta_T = 0   (shooting.hpp:290-296)
          a.adj0[(long long)k * a.stride + row] = Math<T>::mul_rn(a.two_lambda, qn - tg);
          a.adj0[(long long)(D + k) * a.stride + row] = T(0);
        }
      } else {
        const T da = a.inv_sig2 * s0;
        const T dbeta = s1;
        // alpha += dt*d_alpha ; beta += dt*d_beta   (shooting.hpp:302-306)
        const T an = Math<T>::add_rn(ri[(2 * D + k) * RS], Math<T>::mul_rn(a.dt, da));
        const T bn = Math<T>::add_rn(ri[(3 * D + k) * RS], Math<T>::mul_rn(a.dt, dbeta));
        out[(long long)k * a.stride + row] = an;
        out[(long long)(D + k) * a.stride + row] = bn;
        if (epi & kEpiGradOut)  // grad = beta_0 + hp(q0,p0)   (shooting.hpp:311-313)
          a.grad_out[row * D + k] = (double)Math<T>::add_rn(bn, __ldcg(a.hp0 + (long long)k * a.stride + row));
      }
    }
  }
}

template <typename T, int D, int MAXW = kSmallMaxWindows, int RS = SmallShape<T>::kRowsPerSlot>
__global__ void __launch_bounds__(32 * kSmallWarps, 1) small_eval_kernel(const SmallArgs<T> a)
{
  constexpr int kThreadsHere = 32 * kSmallWarps;
  constexpr int NV = RS * 2 * D;
  extern __shared__ __align__(128) unsigned char small_smem[];
  T* tile = reinterpret_cast<T*>(small_smem);
  __shared__ __align__(16) T part[MAXW * kSmallWarps * kSmallMaxPieces * NV];  // the pieces' sums
  constexpr int kEpiThreads = kSmallMaxSlots * RS * D;
  constexpr int kPlans = MAXW > 1 ? 1 + MAXW : 1;  // forward + adjoint windows, or one shared plan
  __shared__ SmallWarpPlan wplans[kPlans * kSmallWarps];
  __shared__ SmallRun runs[kPlans * kSmallWarps];
  __shared__ SmallEpiPlan eplans[(MAXW > 1 ? 1 + MAXW : 1) * kEpiThreads];
  __shared__ __align__(16) T rowbuf[kSmallMaxSlots * RS * 4 * D];      // row operands for the epilogue threads
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

  // the work plan of the launch: the forward window, then the one or two adjoint windows (read after the next
  // __syncthreads: the row staging's)
  SmallCtx cx;
  {
    const int slots = (a.n + RS - 1) / RS;
    cx.slot0 = (int)((long long)blockIdx.x * slots / gridDim.x);
    cx.s_b = (int)((long long)(blockIdx.x + 1) * slots / gridDim.x) - cx.slot0;
    const int G = (a.n + 31) / 32;                    // live 32-column groups
    constexpr int GPW = SmallShape<T>::kCols / 32;    // ... per adjoint window
    cx.adj_windows = (MAXW > 1 && G > GPW) ? 2 : 1;
    cx.wplan = wplans;
    cx.eplan = eplans;
    cx.epi_stride = kEpiThreads;
    // plan 0: the forward window (all G groups); with MAXW > 1 plans 1, 2: the adjoint windows (the first GPW groups, the
    // rest); with MAXW == 1 the host guarantees G <= GPW and the adjoint sweep uses plan 0 as well
    int gw[kPlans];
    gw[0] = G;
    if constexpr (MAXW > 1) {
      gw[1] = G > GPW ? GPW : G;
      gw[2] = G > GPW ? G - GPW : 0;
    }
    const int pl = (int)threadIdx.x / kSmallWarps, w = (int)threadIdx.x - pl * kSmallWarps;
    if (pl < kPlans) {
      const int gwp = pl == 0 ? gw[0] : (pl == 1 ? gw[kPlans > 1 ? 1 : 0] : gw[kPlans > 2 ? 2 : 0]);
      if (gwp > 0) {
        const int total = cx.s_b * gwp;
        SmallRun r;
        r.r0 = w * total / kSmallWarps;
        r.r1 = (w + 1) * total / kSmallWarps;
        r.s0 = r.r1 > r.r0 ? r.r0 / gwp : 0;
        r.s1 = r.r1 > r.r0 ? (r.r1 - 1) / gwp : -1;
        runs[pl * kSmallWarps + w] = r;
      }
    }
    __syncthreads();
#pragma unroll
    for (int p2 = 0; p2 < kPlans; ++p2)
      if (gw[p2] > 0)
        small_plan_window<RS, D>(gw[p2], runs + p2 * kSmallWarps, wplans + p2 * kSmallWarps, eplans + p2 * kEpiThreads);
  }
  unsigned phase = 0;  // bit b: parity chunk barrier b completes next
  double hsum = 0.0, msum = 0.0;
  const int Tn = a.timesteps;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int GW = gridDim.x * kSmallWarps;
  // forward Euler flow, T+1 snapshots kept for the adjoint (shooting.hpp:199-212)
  for (int t = 0; t < Tn; ++t) {
    const unsigned epi = kEpiEuler | (t == 0 ? kEpiFirstStep : 0u) | (t == Tn - 1 ? kEpiLastStep : 0u);
    small_step<T, D, kFwd, RS, MAXW>(a, cx, a.traj + (long long)t * a.snap_elems, nullptr, a.traj + (long long)(t + 1) * a.snap_elems,
                           epi, t + 1, tile, part, rowbuf, bars, phase, hsum, msum, exp_tbl, 8 * t);
    LMS_TRACE_POINT(a, 8 * t + 4);
    if (t == Tn - 1) {
      // per-warp partials of the two double sums: threads hold their rows' terms; fixed butterfly
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
        msum += __shfl_xor_sync(0xffffffffu, msum, off);
      }
      if (lane == 0) {
        a.warp_part[blockIdx.x * kSmallWarps + warp] = hsum;
        a.warp_part[GW + blockIdx.x * kSmallWarps + warp] = msum;
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
      // host-buffer calls: the scalars live in mapped host memory; the divergence word (final after the last forward
      // barrier: only the input check and the forward epilogues record) goes along as its fourth word
      unsigned long long* word_out = reinterpret_cast<unsigned long long*>(a.scalars + 3);
      if (word_out != a.diverged) *word_out = __ldcg(a.diverged);
    }
  }
  // discrete adjoint sweep t = T-1 .. 0 (shooting.hpp:300-307), final gradient fused into the t = 0 step
  T* adj_in = a.adj0;
  T* adj_out = a.adj1;
  for (int t = Tn - 1; t >= 0; --t) {
    small_step<T, D, kAdj, RS, MAXW>(a, cx, a.traj + (long long)t * a.snap_elems, adj_in, adj_out,
                           kEpiEuler | (t == 0 ? kEpiGradOut : 0u), t, tile, part, rowbuf, bars, phase, hsum, msum,
                           exp_tbl, 8 * (2 * Tn - 1 - t));
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
