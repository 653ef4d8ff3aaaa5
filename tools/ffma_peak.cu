// Microbenchmark: FP32 FFMA vs FFMA2 (fma.rn.f32x2) throughput on sm_100a.
// Outer-product register pattern (what the conv kernel's inner loop looks like):
// 16 weights x 4 inputs per step, accumulators held in registers.
#include <cstdio>
#include <cuda_runtime.h>

template <bool PAIR>
__global__ void __launch_bounds__(256) peak_kernel(const float* __restrict__ src, float* out, int iters) {
  float w[16], x[4];
#pragma unroll
  for (int i = 0; i < 16; i++) w[i] = src[(threadIdx.x + i) & 255];
#pragma unroll
  for (int i = 0; i < 4; i++) x[i] = src[(threadIdx.x * 7 + i) & 255];
  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
  for (int it = 0; it < iters; it++) {
    if (PAIR) {
#pragma unroll
      for (int i = 0; i < 16; i += 2)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          float2 r = __ffma2_rn(make_float2(w[i], w[i + 1]), make_float2(x[j], x[j]),
                                make_float2(acc[i][j], acc[i + 1][j]));
          acc[i][j] = r.x; acc[i + 1][j] = r.y;
        }
    } else {
#pragma unroll
      for (int i = 0; i < 16; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(w[i], x[j], acc[i][j]);
    }
    // perturb inputs so the compiler cannot hoist
#pragma unroll
    for (int j = 0; j < 4; j++) x[j] = __int_as_float(__float_as_int(x[j]) ^ 1);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) s += acc[i][j];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, clk);
  float *src, *out; cudaMalloc(&src, 1024 * 4); cudaMalloc(&out, 4); cudaMemset(src, 0, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int pair = 0; pair < 2; pair++) {
    for (int blocksPerSm = 1; blocksPerSm <= 4; blocksPerSm *= 2) {
      int grid = p.multiProcessorCount * blocksPerSm;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(a);
        if (pair) peak_kernel<true><<<grid, 256>>>(src, out, iters);
        else peak_kernel<false><<<grid, 256>>>(src, out, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double flops = 2.0 * 64 * iters * (double)grid * 256;
        if (rep == 2)
          printf("{\"mode\": \"%s\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
                 pair ? "ffma2" : "ffma", blocksPerSm, ms, flops / ms / 1e9);
      }
    }
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
