// Development probe: which TMA tiled loads are legal for the tensor-core conv?
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/tp tools/tma_probe.cu && /tmp/tp
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "../paper_2103_16234_b200/csrc/conv_tc.cuh"

using namespace b2c::tc;

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct P {
  CUtensorMap map;
  int c0, c1, c2, c3;
  float *out;
  int bytes;
};

__global__ void k(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(smem_u32(&bar), p.bytes);
    tma_load_4d(smem_u32(smem), &p.map, smem_u32(&bar), p.c0, p.c1, p.c2, p.c3);
    mbar_wait(smem_u32(&bar), 0, 1000000000ull, nullptr, 0);
    for (int i = 0; i < p.bytes / 4; i++) p.out[i] = reinterpret_cast<float *>(smem)[i];
  }
}

int main(int argc, char **argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int idx = -1;
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  struct T {
    const char *name;
    unsigned W, H, C, N, bx, by;
    CUtensorMapSwizzle sw;
    int c0, c1;
    int strides_mode;  // 0 natural, 1 flat-like (stride1 == stride0)
  } tests[] = {
      {"flat-like 196x1", 196, 1, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 0, 0, 0},
      {"rows 32x8 (0,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 0, 0, 0},
      {"rows 32x8 (-1,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, -1, 0, 0},
      {"rows 32x8 (0,-1)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 0, -1, 0},
      {"rows 32x8 (1,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 1, 0, 0},
      {"rows 32x8 sw128 (-1,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B, -1, 0, 0},
      {"rows 32x8 none (-1,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_NONE, -1, 0, 0},
      {"rows 32x8 sw128 (0,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B, 0, 0, 0},
      {"rows 16x16 box16x2 (0,0)", 16, 16, 16, 1, 16, 2, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 0, 0, 0},
      {"rows 16x16 box16x2 (-1,-1)", 16, 16, 16, 1, 16, 2, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, -1, -1, 0},
      {"flat 196 (-1)", 196, 1, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, -1, 0, 0},
      {"rows 32x8 sw128 (-32,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B, -32, 0, 0},
      {"rows 32x8 a32 (-4,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, -4, 0, 0},
      {"rows 32x8 a32 (-8,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, -8, 0, 0},
      {"rows 32x8 a32 (4,0)", 32, 8, 16, 1, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 4, 0, 0},
      {"rows 32x8 sw64 box16 (-1,0)", 32, 8, 16, 1, 16, 1, CU_TENSOR_MAP_SWIZZLE_64B, -1, 0, 0},
  };
  float *x, *out;
  cudaMalloc(&x, 256 * 256 * 16 * 4);
  cudaMallocManaged(&out, 65536);
  for (const T &t : tests) {
    if (++idx != only && only >= 0) continue;
    P p;
    memset(&p, 0, sizeof(p));
    cuuint64_t dim[4] = {t.W, t.H, t.C, t.N};
    cuuint64_t str[3] = {(cuuint64_t)t.W * 4, (cuuint64_t)t.W * t.H * 4, (cuuint64_t)t.W * t.H * t.C * 4};
    cuuint32_t box[4] = {t.bx, t.by, 16, 1};
    cuuint32_t ones[4] = {1, 1, 1, 1};
    CUresult r = enc(&p.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dim, str, box, ones, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     t.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    p.c0 = t.c0;
    p.c1 = t.c1;
    p.out = out;
    p.bytes = t.bx * t.by * 16 * 4;
    if (r != CUDA_SUCCESS) {
      printf("%-30s encode failed %d\n", t.name, (int)r);
      continue;
    }
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    k<<<1, 32, 8192>>>(p);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-30s %s\n", t.name, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    if (e != cudaSuccess) {
      cudaDeviceReset();
      cudaMalloc(&x, 256 * 256 * 16 * 4);
      cudaMallocManaged(&out, 65536);
    }
  }
  return 0;
}
