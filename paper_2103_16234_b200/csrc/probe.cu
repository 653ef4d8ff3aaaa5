// FP32 FFMA2 throughput probe: the measured denominator of the FP32 roofline
// (MEASURED_PEAKS.json carries HBM and bf16 figures only).  Same register
// pattern as the conv inner loop: 16 channels x 4 pixels of FFMA2 with a
// scalar-broadcast pixel operand.  Reports TFLOP/s from CUDA events, the SM
// clock the kernel actually ran at (per CTA: clock64 cycles over globaltimer
// nanoseconds of the same interval, averaged), and FMA/clk/SM = total FMAs /
// (SMs x wall time x that clock) — at most 128 on B200 (128 FP32 lanes/SM).
#include <cuda_runtime.h>

#include "../../include/b2conv.h"
#include "internal.h"

namespace {

__global__ void __launch_bounds__(256) ffma2_probe_kernel(const float *__restrict__ src, float *sink, int iters,
                                                          long long *stamps) {
  float w[16], x[4];
#pragma unroll
  for (int i = 0; i < 16; i++) w[i] = src[(threadIdx.x + i) & 255];
#pragma unroll
  for (int j = 0; j < 4; j++) x[j] = src[(threadIdx.x * 7 + j) & 255];
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  __syncthreads();
  long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
          acc[i][j] = __ffma2_rn(make_float2(w[2 * i], w[2 * i + 1]), make_float2(x[j], x[j]), acc[i][j]);
    }
#pragma unroll
    for (int j = 0; j < 4; j++) x[j] = __int_as_float(__float_as_int(x[j]) ^ 1);
  }
  __syncthreads();
  const long long t1 = clock64();
  long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) s += acc[i][j].x + acc[i][j].y;
  if (s == 1234.5f) sink[0] = s;
  if (threadIdx.x == 0) {
    stamps[2 * blockIdx.x] = t1 - t0;
    stamps[2 * blockIdx.x + 1] = g1 - g0;
  }
}

}  // namespace

extern "C" b2c_status b2c_probe_fp32_peak(int32_t iters, double *tflops, double *fma_per_clk_per_sm,
                                          double *sm_mhz) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = b2c::device_sm_count(dev);
  const int ctas_per_sm = 2, threads = 256;
  const int grid = sms * ctas_per_sm;
  float *src = nullptr, *sink = nullptr;
  long long *cyc = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  b2c_status st = B2C_OK;
  long long *host = new long long[2 * grid];
  float ms = 0.f;
  if (cudaMalloc(&src, 1024 * sizeof(float)) != cudaSuccess || cudaMalloc(&sink, sizeof(float)) != cudaSuccess ||
      cudaMalloc(&cyc, 2 * grid * sizeof(long long)) != cudaSuccess || cudaEventCreate(&a) != cudaSuccess ||
      cudaEventCreate(&b) != cudaSuccess) {
    st = B2C_CUDA_ERROR;
  } else {
    cudaMemset(src, 0, 1024 * sizeof(float));
    ffma2_probe_kernel<<<grid, threads>>>(src, sink, 64, cyc);  // warm-up
    cudaEventRecord(a);
    ffma2_probe_kernel<<<grid, threads>>>(src, sink, iters, cyc);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = B2C_CUDA_ERROR;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(host, cyc, 2 * grid * sizeof(long long), cudaMemcpyDeviceToHost);
  }
  if (st == B2C_OK) {
    const double fma_per_thread = 4.0 * 64.0 * iters;  // 4 rounds x 32 FFMA2 x 2 lanes
    const double total_fma = fma_per_thread * threads * grid;
    double cyc = 0, ns = 0;
    for (int i = 0; i < grid; i++) {
      cyc += (double)host[2 * i];
      ns += (double)host[2 * i + 1];
    }
    const double mhz = ns > 0 ? 1e3 * cyc / ns : 0.0;  // cycles per microsecond while the CTAs ran
    if (tflops) *tflops = 2.0 * total_fma / (ms * 1e-3) / 1e12;
    if (sm_mhz) *sm_mhz = mhz;
    if (fma_per_clk_per_sm) *fma_per_clk_per_sm = mhz > 0 ? total_fma / ((double)sms * ms * 1e3 * mhz) : 0.0;
  }
  delete[] host;
  if (src) cudaFree(src);
  if (sink) cudaFree(sink);
  if (cyc) cudaFree(cyc);
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  return st;
}
