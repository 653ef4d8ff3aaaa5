// Development probe: one tcgen05.mma (kind::tf32, M=128, K=8) on operands
// written into shared memory by plain stores in a chosen canonical layout,
// accumulator read back with tcgen05.ld.  Checks descriptor/layout encodings
// in isolation from TMA.   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/up tools/umma_probe.cu && /tmp/up
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2103_16234_b200/csrc/conv_tc.cuh"

using namespace b2c::tc;

// logical byte offset -> physical (swizzle within 1 KB / 512 B atoms)
__host__ __device__ inline uint32_t swz(uint32_t L, int mode) {
  if (mode == 32) return L ^ (((L >> 7) & 3) << 5);  // 128B rows, 32-byte atoms (Swizzle<2,5,2>)
  if (mode == 128) return L ^ (((L >> 7) & 7) << 4);
  if (mode == 64) return L ^ (((L >> 7) & 3) << 4);
  return L;
}

struct Cfg {
  int a_mn;      // 1: A MN-major, 0: K-major
  int a_swz;     // 128 / 64
  int b_swz;     // 64 / 128 (K-major)
  int n;         // UMMA N
  int m_bit;     // 23 or 24: where M>>4 goes
};

__global__ void probe(const float *A, const float *B, float *D, Cfg c, uint32_t idesc, int *err) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t *sa = smem;           // 128 x 8 tf32
  uint8_t *sb = smem + 16384;   // n x 8 tf32
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  // A[m][k], m < 128, k < 8
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    uint32_t L;
    if (c.a_mn && c.a_swz == 32) {  // MN-major, 128B rows, 32B-atom swizzle: LBO 1024 (MN block), SBO 512 (4 K rows)
      L = (m / 32) * 1024 + (k / 4) * 512 + (k % 4) * 128 + (m % 32) * 4;
    } else if (c.a_mn) {
      const int T = c.a_swz / 4;  // MN elements per atom row
      L = (m / T) * (T * 4 * 8) /*LBO: one atom per MN block (K=8 only)*/ + k * c.a_swz + (m % T) * 4;
    } else {
      L = m * c.a_swz + k * 4;  // K-major rows of a_swz bytes (only first 32 B used)
    }
    *reinterpret_cast<float *>(sa + swz(L, c.a_swz)) = A[i];
  }
  for (int i = t; i < c.n * 8; i += blockDim.x) {
    const int nn = i / 8, k = i % 8;
    const uint32_t L = nn * c.b_swz + k * 4;
    *reinterpret_cast<float *>(sb + swz(L, c.b_swz)) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (t == 0) {
    uint64_t ad, bd;
    const uint64_t al = c.a_swz == 128 ? LAYOUT_SW128 : c.a_swz == 32 ? 1 : LAYOUT_SW64;
    const uint64_t bl = c.b_swz == 128 ? LAYOUT_SW128 : LAYOUT_SW64;
    if (c.a_mn && c.a_swz == 32) {
      ad = umma_desc(smem_u32(sa), 1024, 512, al);
    } else if (c.a_mn) {
      const int T = c.a_swz / 4;
      ad = umma_desc(smem_u32(sa), T * 4 * 8, 8 * c.a_swz, al);
    } else {
      ad = umma_desc(smem_u32(sa), 16, 8 * c.a_swz, al);
    }
    bd = umma_desc(smem_u32(sb), 16, 8 * c.b_swz, bl);
    umma_tf32(tm, ad, bd, idesc, 0);
    umma_commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&bar), 0, 2000000000ull, nullptr, 0);
  tc_fence_after();
  if (t < 128) {
    const int q = (t >> 5) & 3;
    for (int j0 = 0; j0 < c.n; j0 += 32) {
      uint32_t r[32];
      tmem_ld32(tm + ((uint32_t)(q * 32) << 16) + j0, r);
      for (int j = 0; j < 32 && j0 + j < c.n; j++) D[(q * 32 + (t & 31)) * c.n + j0 + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256) : "memory");
  }
}

int main() {
  float *A, *B, *D;
  int *err;
  cudaMallocManaged(&A, 128 * 8 * 4);
  cudaMallocManaged(&B, 256 * 8 * 4);
  cudaMallocManaged(&D, 128 * 256 * 4);
  cudaMallocManaged(&err, 4);
  for (int i = 0; i < 128 * 8; i++) A[i] = (float)((i * 7) % 13 - 6);
  for (int i = 0; i < 256 * 8; i++) B[i] = (float)((i * 5) % 11 - 5);
  Cfg cfgs[] = {{0, 128, 64, 16, 24}, {1, 32, 64, 16, 24}, {1, 32, 64, 64, 24}, {1, 32, 128, 256, 24},
                {1, 32, 64, 48, 24}, {1, 128, 64, 16, 24}};
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (const Cfg &c : cfgs) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)c.a_mn << 15) |
                           ((uint32_t)(c.n >> 3) << 17) | ((uint32_t)(128 >> 4) << c.m_bit);
    cudaMemset(D, 0, 128 * 256 * 4);
    probe<<<1, 128, 64 * 1024>>>(A, B, D, c, idesc, err);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("cfg a_mn=%d a_swz=%d b_swz=%d n=%d mbit=%d: CUDA error %s\n", c.a_mn, c.a_swz, c.b_swz, c.n, c.m_bit,
             cudaGetErrorString(e));
      return 1;
    }
    double maxerr = 0, maxref = 0;
    int nz = 0;
    for (int m = 0; m < 128; m++)
      for (int n = 0; n < c.n; n++) {
        double ref = 0;
        for (int k = 0; k < 8; k++) ref += (double)A[m * 8 + k] * B[n * 8 + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * c.n + n]));
        maxref = fmax(maxref, fabs(ref));
        nz += D[m * c.n + n] != 0.0f;
      }
    printf("cfg a_mn=%d a_swz=%d b_swz=%d n=%d mbit=%d: maxerr %.3g (maxref %.3g) nonzero %d  D[0][0..3]=%g %g %g %g\n",
           c.a_mn, c.a_swz, c.b_swz, c.n, c.m_bit, maxerr, maxref, nz, D[0], D[1], D[2], D[3]);
  }
  return 0;
}
