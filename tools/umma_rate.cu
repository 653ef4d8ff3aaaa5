// Development probe: tcgen05.mma kind::tf32 throughput vs operand layout.
// One CTA per SM issues `iters` back-to-back UMMAs from shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/ur tools/umma_rate.cu && /tmp/ur
#include <cstdio>
#include "../paper_2103_16234_b200/csrc/conv_tc.cuh"
using namespace b2c::tc;

__global__ void rate(int layout, int n, int iters, int kind, unsigned long long *cyc, int extra = 0, int nacc = 1) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float *>(smem)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 32768;
    uint64_t ad, bd;
    if (layout == 0) {  // K-major, no swizzle: core matrices 8x16B, LBO 128 SBO 512 (our gather layout)
      ad = umma_desc(sa, 128, 512, LAYOUT_NONE); bd = umma_desc(sb, 128, 512, LAYOUT_NONE);
    } else if (layout == 1) {  // K-major no swizzle, halo style: SBO 128, LBO = 2 KB planes
      ad = umma_desc(sa, 2048, 128, LAYOUT_NONE); bd = umma_desc(sb, 128, 512, LAYOUT_NONE);
    } else if (layout == 2) {  // K-major SW128 both (rows of 32 tf32)
      ad = umma_desc(sa, 16, 1024, LAYOUT_SW128); bd = umma_desc(sb, 16, 1024, LAYOUT_SW128);
    } else {  // K-major SW64 both
      ad = umma_desc(sa, 16, 512, LAYOUT_SW64); bd = umma_desc(sb, 16, 512, LAYOUT_SW64);
    }
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t idesc16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);  // bf16
    const unsigned long long t0 = clock64();
    __shared__ uint64_t bar2, sink;
    mbar_init(smem_u32(&bar2), 1);
    mbar_arrive(smem_u32(&bar2));  // phase 0 complete: waits on parity 0 succeed at once
    mbar_init(smem_u32(&sink), 1 << 20);  // commits arrive here, the phase never completes
    for (int i = 0; i < iters; i++) {
      if (extra & 1) mbar_wait(smem_u32(&bar2), 0, 4000000000ull);
      if (extra & 2) tc_fence_after();
      if (kind == 0) umma_tf32(tslot + (i % nacc) * (256 / nacc), ad, bd, idesc, i > 0);
      else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                        ::"r"(tslot), "l"(ad), "l"(bd), "r"(idesc16), "r"((uint32_t)(i > 0)) : "memory");
      if (extra & 4) umma_commit(smem_u32(&sink));
    }
    umma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0, 4000000000ull);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(256) : "memory");
  }
}

int main() {
  unsigned long long *cyc;
  cudaMallocManaged(&cyc, 148 * 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int iters = 20000;
  for (int n : {64, 128, 256})
    for (int nacc : {1, 2, 4})
      for (int extra : {0, 1, 2, 4, 7}) {
        if (n * nacc > 256 && nacc > 1 && n == 256) continue;
        rate<<<148, 128, 70 * 1024>>>(2, n, iters, 0, cyc, extra, nacc);
        cudaError_t e = cudaDeviceSynchronize();
        const double macs = 128.0 * n * 8 * iters;
        printf("tf32 N=%3d accumulators=%d extra=%d (1 wait, 2 fence, 4 commit): %s %.1f clk/MMA %.0f MAC/clk/SM\n", n, nacc,
               extra, cudaGetErrorString(e), (double)cyc[0] / iters, macs / cyc[0]);
      }
  return 0;
}
