// Microbenchmark: FFMA2 throughput with shared-memory operand loads
// interleaved, in the register pattern of the pointwise kernel (thread tile
// RM channels x 8 pixels: RM/4 LDS.128 of filters + 2 LDS.128 of pixels per
// channel, RM*4 FFMA2).  Answers: how much of the 128 FMA/clk/SM FFMA2 peak
// survives the operand traffic, per tile shape and warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/flp tools/probes/ffma_lds_probe.cu && /tmp/flp
#include <cstdio>
#include <cuda_runtime.h>

template <int RM, int MODE>  // MODE 0: no loads (registers only), 1: LDS.128 per channel, 2: LDS.64 weights
__global__ void __launch_bounds__(256) probe(const float *src, float *sink, int iters, int wdist) {
  __shared__ __align__(16) float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = src[i & 1023];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int mgi = lane >> 3, pgi = lane & 7;
  // filter reads: 4 distinct 16B words across the warp (mgi), pixels: 8 distinct (pgi)
  const float *ws = sm + (wdist ? mgi * 4 : 0);
  const float *xs = sm + 4096 + pgi * 4;
  float2 acc[RM / 2][8];
#pragma unroll
  for (int i = 0; i < RM / 2; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.f, 0.f);
  float2 wr[RM / 2];
  float xr[8];
#pragma unroll
  for (int i = 0; i < RM / 2; i++) wr[i] = make_float2(sm[i], sm[i + 1]);
#pragma unroll
  for (int j = 0; j < 8; j++) xr[j] = sm[100 + j];
  for (int it = 0; it < iters; it++) {
#pragma unroll 2
    for (int c = 0; c < 16; c++) {
      if (MODE == 1) {
#pragma unroll
        for (int k = 0; k < RM / 4; k++) {
          const float4 w = *reinterpret_cast<const float4 *>(ws + c * 132 + 16 * k);
          wr[2 * k] = make_float2(w.x, w.y);
          wr[2 * k + 1] = make_float2(w.z, w.w);
        }
        const float4 xa = *reinterpret_cast<const float4 *>(xs + c * 256);
        const float4 xb = *reinterpret_cast<const float4 *>(xs + c * 256 + 32);
        xr[0] = xa.x; xr[1] = xa.y; xr[2] = xa.z; xr[3] = xa.w;
        xr[4] = xb.x; xr[5] = xb.y; xr[6] = xb.z; xr[7] = xb.w;
      }
#pragma unroll
      for (int i = 0; i < RM / 2; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = __ffma2_rn(wr[i], make_float2(xr[j], xr[j]), acc[i][j]);
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 8; j++) xr[j] = __int_as_float(__float_as_int(xr[j]) ^ 1);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < RM / 2; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) s += acc[i][j].x + acc[i][j].y;
  if (s == 1234.5f) sink[0] = s;
}

template <int RM, int MODE>
void run(const char *name, int threads, int ctas_per_sm, int wdist) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *src, *sink;
  cudaMalloc(&src, 4096 * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 0, 4096 * 4);
  const int iters = 2000;
  const int grid = sms * ctas_per_sm;
  probe<RM, MODE><<<grid, threads>>>(src, sink, 10, wdist);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<RM, MODE><<<grid, threads>>>(src, sink, iters, wdist);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fma = (double)grid * threads * iters * 16.0 * RM * 8;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<RM, MODE>, threads, 0);
  printf("%-34s threads %3d ctas/SM %d (occ %d) wdist %d: %6.1f TFLOP/s  %5.1f FMA/clk/SM @1.92GHz  err=%s\n", name,
         threads, ctas_per_sm, occ, wdist, 2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / sms / 1.92e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(src);
  cudaFree(sink);
}

int main() {
  run<8, 0>("8x8 registers only", 256, 2, 1);
  run<8, 1>("8x8 LDS.128 (vec kernel)", 256, 2, 1);
  run<8, 1>("8x8 LDS.128 broadcast w", 256, 2, 0);
  run<8, 1>("8x8 LDS.128 (vec kernel)", 128, 4, 1);
  run<8, 1>("8x8 LDS.128 1 CTA", 256, 1, 1);
  run<16, 0>("16x8 registers only", 128, 3, 1);
  run<16, 1>("16x8 LDS.128", 128, 3, 1);
  run<16, 1>("16x8 LDS.128", 256, 1, 1);
  run<16, 1>("16x8 LDS.128", 128, 2, 1);
  return 0;
}
