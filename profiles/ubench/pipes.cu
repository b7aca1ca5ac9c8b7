// CUDA-core pipe microbenchmarks for sm_100a: the denominators of the pairwise-interaction
// roofline (SURVEY.md §8d asks for these before any kernel claim).
// Each kernel runs ITER iterations of NACC independent dependency chains per thread; every
// CTA has 256 threads and the grid is 148 x CTAS_PER_SM so every SMSP has 16 resident warps.
// Reported: warp-instructions / SM / clk and lane-ops / SM / clk, with the SM clock measured
// from clock64() against the CUDA-event wall time of the same launch.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int ITER = 2048;

__device__ __forceinline__ float ex2_approx(float x)
{
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(256) pipe_kernel(float* out, long long* cycles, float a, float b)
{
  long long t0 = clock64();
  float r = 0.f;
  if constexpr (MODE == 0) {  // FFMA, 16 chains
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(acc[k], a, b);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 1) {  // FFMA2 packed, 8 float2 chains (16 lanes of work)
    float2 acc[8];
    float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x * 1e-3f + k, k);
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(acc[k], a2, b2);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
  } else if constexpr (MODE == 2) {  // FADD
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = __fadd_rn(acc[k], a);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 3) {  // FMUL
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = __fmul_rn(acc[k], a);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 4) {  // MUFU.EX2
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = ex2_approx(acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 5) {  // 16 FFMA : 1 MUFU (the forward pair mix)
    float acc[16];
    float m = threadIdx.x * 1e-3f;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(acc[k], a, b);
      m = ex2_approx(m);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
    r += m;
  } else if constexpr (MODE == 6) {  // 8 FFMA2 : 2 MUFU (packed pair mix, 2 pairs)
    float2 acc[8];
    float m0 = threadIdx.x * 1e-3f, m1 = m0 + 1.f;
    float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x * 1e-3f + k, k);
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(acc[k], a2, b2);
      m0 = ex2_approx(m0);
      m1 = ex2_approx(m1);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
    r += m0 + m1;
  } else if constexpr (MODE == 7) {  // FADD2 packed
    float2 acc[8];
    float2 a2 = make_float2(a, a);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x * 1e-3f + k, k);
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __fadd2_rn(acc[k], a2);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
  } else if constexpr (MODE == 8) {  // FFMA with three distinct varying sources (register-bank pressure)
    float acc[16], x[4], y[4];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x * 1e-3f + k;
#pragma unroll
    for (int k = 0; k < 4; ++k) { x[k] = a + k; y[k] = b - k; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(x[k & 3], y[(k >> 2) & 3], acc[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) { x[k] = x[k] + 1e-7f; }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 9) {  // FFMA, three DISTINCT register sources per instruction, no operand reuse
    float acc[16], x[16], y[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { acc[k] = threadIdx.x * 1e-3f + k; x[k] = a + k * 1e-3f * threadIdx.x; y[k] = b - k * 1e-3f * threadIdx.x; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(x[k], y[k], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 10) {  // FFMA2, three distinct 64-bit register sources per instruction
    float2 acc[8], x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc[k] = make_float2(threadIdx.x * 1e-3f + k, k);
      x[k] = make_float2(a + k * 1e-3f * threadIdx.x, a - k * 1e-3f * threadIdx.x);
      y[k] = make_float2(b - k * 1e-3f * threadIdx.x, b + k * 1e-3f * threadIdx.x);
    }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(x[k], y[k], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
  } else if constexpr (MODE == 11) {  // FFMA2, two distinct register sources + one reused
    float2 acc[8], x[8];
    float2 c2 = make_float2(a, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc[k] = make_float2(threadIdx.x * 1e-3f + k, k);
      x[k] = make_float2(a + k * 1e-3f * threadIdx.x, a - k * 1e-3f * threadIdx.x);
    }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(x[k], c2, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
  } else if constexpr (MODE == 12) {  // FFMA, two distinct register sources + one reused
    float acc[16], x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { acc[k] = threadIdx.x * 1e-3f + k; x[k] = a + k * 1e-3f * threadIdx.x; }
    float c1 = b * threadIdx.x;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(x[k], c1, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) r += acc[k];
  } else if constexpr (MODE == 15) {  // FFMA2 acc2 += x2[k] * splat(y[k]): the .F32 broadcast operand form
    float2 acc[8], x[8];
    float y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc[k] = make_float2(threadIdx.x * 1e-3f + k, k);
      x[k] = make_float2(a + k * 1e-3f * threadIdx.x, a - k * 1e-3f * threadIdx.x);
      y[k] = b - k * 1e-3f * threadIdx.x;
    }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(x[k], make_float2(y[k], y[k]), acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k].x + acc[k].y;
  } else if constexpr (MODE == 16) {  // 8 FFMA + 8 FADD per iteration: do FADD and FFMA share one pipe?
    float acc[8], add[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc[k] = threadIdx.x * 1e-3f + k; add[k] = threadIdx.x * 2e-3f - k; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) { acc[k] = fmaf(acc[k], a, b); add[k] = __fadd_rn(add[k], a); }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) r += acc[k] + add[k];
  } else if constexpr (MODE == 17) {  // 4 FFMA2 + 4 FADD2 per iteration
    float2 acc[4], add[4];
    float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) { acc[k] = make_float2(threadIdx.x * 1e-3f + k, k); add[k] = make_float2(threadIdx.x * 2e-3f - k, k); }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { acc[k] = __ffma2_rn(acc[k], a2, b2); add[k] = __fadd2_rn(add[k], a2); }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) r += acc[k].x + acc[k].y + add[k].x + add[k].y;
  } else if constexpr (MODE == 13) {  // FMUL2 then dependent FFMA2 chain of length 3 x 8 independent (latency probe)
    float2 acc[2], x[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) { acc[k] = make_float2(threadIdx.x * 1e-3f + k, k); x[k] = make_float2(a + k, a - k); }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int rep = 0; rep < 4; ++rep)
#pragma unroll
        for (int k = 0; k < 2; ++k) acc[k] = __ffma2_rn(acc[k], x[k], x[k]);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) r += acc[k].x + acc[k].y;
  } else if constexpr (MODE == 14) {  // scalar FFMA dependent chains, 2 independent (latency probe)
    float acc[2], x[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) { acc[k] = threadIdx.x * 1e-3f + k; x[k] = a + k; }
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int rep = 0; rep < 8; ++rep)
#pragma unroll
        for (int k = 0; k < 2; ++k) acc[k] = fmaf(acc[k], x[k], x[k]);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) r += acc[k];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (r == 123.456f) out[0] = r;
}

template <int MODE>
__global__ void __launch_bounds__(256) pipe_kernel_f64(double* out, long long* cycles, double a, double b)
{
  long long t0 = clock64();
  double r = 0;
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if constexpr (MODE == 0) acc[k] = fma(acc[k], a, b);
      else if constexpr (MODE == 1) acc[k] = __dadd_rn(acc[k], a);
      else acc[k] = __dmul_rn(acc[k], a);
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) r += acc[k];
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (r == 123.456) out[0] = r;
}

struct Result { std::string name; double ms; double mhz; double winst_per_sm_clk; double lane_per_sm_clk; };

int main(int argc, char** argv)
{
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  const int ctas_per_sm = 8;  // 8 x 256 = 2048 threads: 16 warps per SMSP
  const int grid = sms * ctas_per_sm;
  float* d_out; long long* d_cyc; double* d_out64;
  CK(cudaMalloc(&d_out, 4)); CK(cudaMalloc(&d_out64, 8));
  CK(cudaMalloc(&d_cyc, sizeof(long long) * grid));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  std::vector<Result> results;
  std::vector<long long> h_cyc(grid);

  int cur_grid = grid;
  auto run = [&](const char* name, auto launch, double winst_per_thread_iter, double lanes_per_winst) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    CK(cudaMemcpy(h_cyc.data(), d_cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost));
    // all CTAs are co-resident, so the kernel's cycle span ~ max CTA cycles
    long long cmax = 0; for (int i = 0; i < cur_grid; ++i) cmax = h_cyc[i] > cmax ? h_cyc[i] : cmax;
    double mhz = cmax / (best * 1e-3) / 1e6;
    double warps_per_sm = (double)cur_grid / sms * 8.0;
    double winst = warps_per_sm * ITER * winst_per_thread_iter;  // per SM
    double per_clk = winst / cmax;
    results.push_back({name, best, mhz, per_clk, per_clk * 32 * lanes_per_winst});
    printf("%-28s %8.3f ms  clk %7.1f MHz  %6.3f winst/SM/clk  %7.2f lane-ops/SM/clk\n", name, best, mhz,
           per_clk, per_clk * 32 * lanes_per_winst);
  };

#define RUNK(NAME, KERN, PTR, A, B, W, L)                                                        \
  {                                                                                               \
    int per_sm = 0;                                                                               \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, KERN, 256, 0));                     \
    if (per_sm > ctas_per_sm) per_sm = ctas_per_sm;                                               \
    cur_grid = sms * per_sm;                                                                      \
    run(NAME, [&] { KERN<<<cur_grid, 256>>>(PTR, d_cyc, A, B); }, W, L);                          \
  }
  RUNK("ffma_3reg_distinct", pipe_kernel<9>, d_out, 1.0001f, 0.5f, 16, 1)
  RUNK("ffma2_3reg_distinct", pipe_kernel<10>, d_out, 1.0001f, 0.5f, 8, 2)
  RUNK("ffma2_2reg_1reused", pipe_kernel<11>, d_out, 1.0001f, 0.5f, 8, 2)
  RUNK("ffma_2reg_1reused", pipe_kernel<12>, d_out, 1.0001f, 0.5f, 16, 1)
  RUNK("ffma2_f32_broadcast_operand", pipe_kernel<15>, d_out, 1.0001f, 0.5f, 8, 2)
  cur_grid = grid;
  run("ffma", [&] { pipe_kernel<0><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 16, 1);
  run("ffma2_packed", [&] { pipe_kernel<1><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 8, 2);
  run("fadd", [&] { pipe_kernel<2><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 16, 1);
  run("fmul", [&] { pipe_kernel<3><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 16, 1);
  run("mufu_ex2", [&] { pipe_kernel<4><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 16, 1);
  run("mix_16ffma_1mufu", [&] { pipe_kernel<5><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 17, 1);
  run("mix_8ffma2_2mufu", [&] { pipe_kernel<6><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 10, 1.8);
  run("fadd2_packed", [&] { pipe_kernel<7><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 8, 2);
  run("ffma_3src", [&] { pipe_kernel<8><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 20, 1);
  run("ffma2_dep_chain_ilp2", [&] { pipe_kernel<13><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 8, 2);
  run("ffma_dep_chain_ilp2", [&] { pipe_kernel<14><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 16, 1);
  run("mix_8ffma_8fadd", [&] { pipe_kernel<16><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 16, 1);
  run("mix_4ffma2_4fadd2", [&] { pipe_kernel<17><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f); }, 8, 2);
  run("dfma", [&] { pipe_kernel_f64<0><<<grid, 256>>>(d_out64, d_cyc, 1.0001, 0.5); }, 8, 1);
  run("dadd", [&] { pipe_kernel_f64<1><<<grid, 256>>>(d_out64, d_cyc, 1.0001, 0.5); }, 8, 1);
  run("dmul", [&] { pipe_kernel_f64<2><<<grid, 256>>>(d_out64, d_cyc, 1.0001, 0.5); }, 8, 1);

  const char* path = argc > 1 ? argv[1] : "pipes.json";
  FILE* f = fopen(path, "w");
  if (f) {
    fprintf(f, "{\"gpu\": \"%s\", \"sms\": %d, \"results\": [", prop.name, sms);
    for (size_t i = 0; i < results.size(); ++i)
      fprintf(f, "%s{\"name\": \"%s\", \"ms\": %.4f, \"sm_mhz\": %.1f, \"winst_per_sm_clk\": %.4f, \"lane_ops_per_sm_clk\": %.3f}",
              i ? ", " : "", results[i].name.c_str(), results[i].ms, results[i].mhz, results[i].winst_per_sm_clk,
              results[i].lane_per_sm_clk);
    fprintf(f, "]}\n");
    fclose(f);
  }
  return 0;
}
