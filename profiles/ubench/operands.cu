// Register-file read bandwidth per operand form of the packed fp32 FMA on sm_100a, and the cost of moving a
// warp-uniform value into a uniform register (REDUX) so that it can enter FFMA2 as a UR operand.
// Every kernel: 256 threads per CTA, 148 x 4 CTAs (8 warps per SMSP), ITER iterations; reported as SMSP cycles
// per FFMA2 (2.0 = the FMA pipe's own rate).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)
constexpr int ITER = 4096;

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, long long* cycles, float a, float b, const float* gsrc)
{
  __shared__ __align__(16) float sm[256];
  sm[threadIdx.x] = gsrc[threadIdx.x];
  __syncthreads();
  float2 acc[16], x[4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = make_float2(a + i * 1e-3f * threadIdx.x, a - i * 1e-3f * threadIdx.x);
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
    if constexpr (MODE == 0) {  // acc(64) += x(64) * UR.F32 : 4 register words
      const float2 s = make_float2(b, b);
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __ffma2_rn(x[i & 3], s, acc[i]);
    } else if constexpr (MODE == 1 || MODE == 2) {
      // 4 column values per iteration from shared memory (uniform address); each feeds 4 FFMA2 (two row pairs x two
      // accumulators): MODE 1 as R.F32 broadcast operands (5 words), MODE 2 through REDUX -> UR (4 words)
      const float4 v = *reinterpret_cast<const float4*>(&sm[(it * 4) & 255]);
      float c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float cv = c[j];
        if constexpr (MODE == 2) cv = __uint_as_float(__reduce_or_sync(0xffffffffu, __float_as_uint(cv)));
        const float2 s = make_float2(cv, cv);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[4 * j + i] = __ffma2_rn(x[i], s, acc[4 * j + i]);
      }
    } else if constexpr (MODE == 3) {  // acc(64) += x(64) * y(64): 6 words
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __ffma2_rn(x[i & 3], x[(i + 1) & 3], acc[i]);
    } else if constexpr (MODE == 4) {  // REDUX alone: 4 per iteration
      const float4 v = *reinterpret_cast<const float4*>(&sm[(it * 4) & 255]);
      unsigned r0 = __reduce_or_sync(0xffffffffu, __float_as_uint(v.x)), r1 = __reduce_or_sync(0xffffffffu, __float_as_uint(v.y));
      unsigned r2 = __reduce_or_sync(0xffffffffu, __float_as_uint(v.z)), r3 = __reduce_or_sync(0xffffffffu, __float_as_uint(v.w));
      acc[0].x += __uint_as_float(r0 ^ r1 ^ r2 ^ r3);
    }
  }
  long long t1 = clock64();
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += acc[i].x + acc[i].y;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (r == 123.456f) out[0] = r;
}

// fp64: DFMA operand forms (16 DP lanes per SMSP: 2.0 cycles per warp instruction is the pipe's own rate)
template <int MODE>
__global__ void __launch_bounds__(256) kd(double* out, long long* cycles, double a, double b)
{
  double acc[16], x[4], y[4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) { x[i] = a + i * 1e-3 * threadIdx.x; y[i] = b - i * 1e-3 * threadIdx.x; }
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
    if constexpr (MODE == 0) {  // acc += x * (uniform)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(x[i & 3], b, acc[i]);
    } else if constexpr (MODE == 1) {  // acc += x * y: three distinct register sources
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(x[i & 3], y[(i >> 2) & 3], acc[i]);
    } else {  // acc = acc * (uniform) + (uniform): one register source
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += acc[i];
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (r == 123.456) out[0] = r;
}

int main()
{
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int grid = prop.multiProcessorCount * 4;
  float* d_out; long long* d_cyc; float* d_src;
  CK(cudaMalloc(&d_out, 4)); CK(cudaMalloc(&d_cyc, 8 * grid)); CK(cudaMalloc(&d_src, 1024));
  std::vector<float> h(256); for (int i = 0; i < 256; ++i) h[i] = 1.0f + 1e-4f * i;
  CK(cudaMemcpy(d_src, h.data(), 1024, cudaMemcpyHostToDevice));
  std::vector<long long> cyc(grid);
  auto run = [&](const char* name, auto launch, double ffma2_per_iter) {
    for (int w = 0; w < 2; ++w) launch();
    CK(cudaDeviceSynchronize());
    launch(); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), d_cyc, 8 * grid, cudaMemcpyDeviceToHost));
    long long cmax = 0; for (auto c : cyc) cmax = c > cmax ? c : cmax;
    // 8 warps per SMSP (4 CTAs x 8 warps / 4 SMSPs)
    double per = (double)cmax / (ITER * 8.0 * (ffma2_per_iter > 0 ? ffma2_per_iter : 1.0));
    printf("{\"name\": \"%s\", \"smsp_cycles_per_%s\": %.3f}\n", name, ffma2_per_iter > 0 ? "instruction" : "iteration_per_warp", per);
  };
  run("ffma2_x64_UR32_acc64 (4 words)", [&] { k<0><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f, d_src); }, 16);
  run("ffma2_x64_R32_acc64 from LDS (5 words)", [&] { k<1><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f, d_src); }, 16);
  run("ffma2_x64_UR32_acc64 via REDUX of the LDS value", [&] { k<2><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f, d_src); }, 16);
  run("ffma2_x64_y64_acc64 (6 words)", [&] { k<3><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f, d_src); }, 16);
  run("redux_x4_per_iteration", [&] { k<4><<<grid, 256>>>(d_out, d_cyc, 1.0001f, 0.5f, d_src); }, 0);
  double* d_out64; CK(cudaMalloc(&d_out64, 8));
  run("dfma_x_UR_acc (2 register sources)", [&] { kd<0><<<grid, 256>>>(d_out64, d_cyc, 1.0001, 0.5); }, 16);
  run("dfma_x_y_acc (3 register sources)", [&] { kd<1><<<grid, 256>>>(d_out64, d_cyc, 1.0001, 0.5); }, 16);
  run("dfma_acc_UR_UR (1 register source)", [&] { kd<2><<<grid, 256>>>(d_out64, d_cyc, 1.0001, 0.5); }, 16);
  return 0;
}
