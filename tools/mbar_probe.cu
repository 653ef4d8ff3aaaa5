// Development probe: cost of the tensor-core kernel's mbarrier ring with no
// payload.  warp 0 = producer, warp 1 = "MMA" (releases via tcgen05.commit or
// a plain arrive), warps 2..9 = loaders.  Prints ns per k-block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/mp tools/mbar_probe.cu && /tmp/mp
#include <cstdio>

#include "../paper_2103_16234_b200/csrc/conv_tc.cuh"

using namespace b2c::tc;

__device__ int g_wait_kind;
__device__ __forceinline__ bool probe_wait_once(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  if (g_wait_kind == 1) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  } else if (g_wait_kind == 2) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity), "r"(20) : "memory");
  } else {
    return mbar_try_wait(bar, parity);
  }
  return ok != 0;
}
#define mbar_wait(bar, par, lim) while (!probe_wait_once(bar, par)) {}

__device__ int g_roles;
__global__ void __launch_bounds__(320, 1) ring(int KB, int S, int use_commit, int poll_mode, unsigned long long *out) {
  const int roles = g_roles;
  __shared__ uint64_t bars[3 * 8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bb = smem_u32(bars);
  auto full = [&](int s) { return bb + 8u * s; };
  auto ready = [&](int s) { return bb + 8u * (S + s); };
  auto empty = [&](int s) { return bb + 8u * (2 * S + s); };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(full(s), 1);
      mbar_init(ready(s), 8);
      mbar_init(empty(s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned long long t0 = clock64();
  const unsigned long long lim = 2000000000ull;
  if (warp == 0) {
    if (lane == 0 && (roles & 1))
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(empty(s), ((kb / S) - 1) & 1, lim);
        mbar_arrive(full(s));
      }
  } else if (warp == 1) {
    if (lane == 0)
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        if (roles & 1) mbar_wait(full(s), (kb / S) & 1, lim);
        if (roles & 2) mbar_wait(ready(s), (kb / S) & 1, lim);
        tc_fence_after();
        if (use_commit) umma_commit(empty(s));
        else mbar_arrive(empty(s));
      }
  } else if (roles & 2) {
    for (int kb = 0; kb < KB; kb++) {
      const int s = kb % S;
      if (kb >= S) {
        if (poll_mode == 0) {
          if (lane == 0) mbar_wait(empty(s), ((kb / S) - 1) & 1, lim);
          __syncwarp();
        } else {
          mbar_wait(empty(s), ((kb / S) - 1) & 1, lim);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(ready(s));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(32) : "memory");
  }
}

int main() {
  unsigned long long *out;
  cudaMallocManaged(&out, 148 * 8);
  const int KB = 2000;
  for (int combo = 0; combo < 4; combo++) {
  const int kind = 0, roles = combo;
  cudaMemcpyToSymbol(g_wait_kind, &kind, 4);
  cudaMemcpyToSymbol(g_roles, &roles, 4);
  printf("roles %d (1 producer, 2 loaders)\n", roles);
  printf("wait kind %d (0 try_wait, 1 test_wait spin, 2 try_wait hint 20ns)\n", kind);
  for (int use_commit = 0; use_commit < 2; use_commit++)
    for (int poll = 0; poll < 1; poll++)
      for (int S : {6}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        ring<<<148, 320>>>(KB, S, use_commit, poll, out);
        cudaEventRecord(a);
        ring<<<148, 320>>>(KB, S, use_commit, poll, out);
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("commit=%d poll_all_lanes=%d S=%d: %s  %.1f ns per k-block, %.0f clk per k-block (CTA 0)\n", use_commit,
               poll, S, cudaGetErrorString(e), ms * 1e6 / KB, (double)out[0] / KB);
      }
  }
  return 0;
}
