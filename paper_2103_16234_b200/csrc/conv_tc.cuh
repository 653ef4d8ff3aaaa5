// Tensor-core (tcgen05 + TMEM + TMA) implicit-GEMM forward convolution for
// sm_100a — the optional TF32 variant named by the north star, in two
// precisions:
//   PASSES = 3  "3xTF32": every operand is split as v = hi + lo with
//               hi = v with the low 13 mantissa bits cleared (exactly a tf32)
//               and lo = v - hi (exact in fp32), and the product is
//               accumulated as a_hi*b_hi + a_hi*b_lo + a_lo*b_hi in fp32 in
//               TMEM: fp32-class accuracy (tolerance tol(K), same as the FFMA
//               engine) at tensor-core rate.
//   PASSES = 1  plain TF32 (operands truncated to tf32): its own, looser
//               tolerance (5e-3 relative, stated in DESIGN.md).
//
// GEMM view (no im2col, no input re-layout): for every filter tap t=(ky,kx)
// and input channel block cb, D[p][m] += X_t[p][c] * W_t[m][c] where p runs
// over output pixels and X_t is the input shifted by the tap.  The shifted
// A tile (128 pixels x 16 channels) is gathered straight from the NCHW input
// by the loader warps (coalesced 4-byte loads along output rows, L1-cached so
// the hf*wf taps re-use each input row; out-of-image positions read as +0.0,
// the reference's virtual zero padding, tensor.py:112-123) -- TMA cannot do
// this shift, its tiled boxes need a 16-byte aligned innermost coordinate.
// Filters arrive by TMA.  Taps are reduced into the same TMEM accumulator,
// so the paper's two reductions (channels within a filter row, then across
// filter rows) both happen inside the tensor core.  Any
// stride, padding, plane size and channel count are covered.
//
// Roles (320 threads, 1 CTA per SM):
//   warp 0      TMA producer of the filter tiles (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..9  A gather (+ 3xTF32 lo twins of A and of the filter tile),
//               then the epilogue (tcgen05.ld -> coalesced fp32 stores).
// The tensor core reads an fp32 operand as tf32 by truncation (measured), so
// the "hi" operands are the raw fp32 tiles and only the lo twins are written.
// Tile: UMMA M = 128 output pixels = 4 chunks of 32 (a chunk is RC output
// rows x XW output columns with RC*XW = 32 -- 1x32, 2x16 or 4x8 -- or 32
// consecutive pixels of the flattened plane for unpadded 1x1 layers),
// UMMA N = NF output channels (16..256), K = 16 input channels per pipeline
// stage (2 UMMA K-steps of 8).
//
// Shared-memory operand layouts (canonical UMMA layouts):
//   A (pixels, MN-major): chunk i at i*2 KB, [16 c][32 px] rows of 128 B,
//       128B swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B: the only
//       MN-major layout tf32 operands support), LBO = 2 KB (next chunk),
//       SBO = 512 B (next 4 channels)
//   B (filters, K-major, by TMA): [NF m][16 c] rows of 64 B, SWIZZLE_64B,
//       SBO = 512 B
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace b2c {
namespace tc {

constexpr int BC = 16;          // input channels per pipeline stage
constexpr int TILE_P = 128;     // output pixels per tile (UMMA M)
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 gather/split + epilogue
constexpr int A_BYTES = TILE_P * BC * 4;  // 8 KB

struct TcParams {
  CUtensorMap wmap;  // 3-D (c, m, tap) view of the filters [tap][m][cp]
  const float *x;    // input [n][c][h][w]
  float *y;
  int C, H, W, HW, S;
  int flat;          // unpadded stride-1 1x1: chunks run over the flattened plane
  int M, Wo, HoWo;   // output geometry (Wo = HoWo for flattened 1x1)
  int Ho;            // output rows (1 for flattened)
  int xw, rc;        // chunk = rc output rows x xw output columns (xw * rc = 32)
  int rgroups;       // chunk rows per image: ceil(Ho / rc)
  int xblocks;       // chunks per row group: ceil(Wo / xw)
  long long nchunks; // N * rgroups * xblocks
  int PH, PW, WF, taps;
  int NF, mtiles, cblocks;
  int stages;
  int b_bytes;       // NF * 64
  int stage_bytes;   // (A_BYTES + b_bytes) * (PASSES == 3 ? 2 : 1)
  int tmem_cols;
  uint32_t idesc;    // UMMA instruction descriptor (kind::tf32, M=128, N=NF)
  unsigned long long spin_limit;  // mbarrier wait bound (ns) before __trap: no silent hangs
  unsigned int *dbg;              // development only (B2C_TC_DEBUG): wait-timeout codes and CTA-0 dumps
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
// `limit_ns` is wall time (globaltimer), checked every 256 polls.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, unsigned long long limit_ns,
                                          unsigned int *dbg = nullptr, unsigned code = 0) {
  unsigned long long t0 = 0;
  unsigned n = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++n & 255u) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) {
        t0 = t;
      } else if (t - t0 > limit_ns) {
        if (dbg) atomicExch(dbg, code);
        __threadfence_system();
        __trap();
      }
    }
  }
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// UMMA shared-memory descriptor (sm100 layout: start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset 0, layout type [61,64)).
enum : uint64_t { LAYOUT_SW128_BASE32B = 1, LAYOUT_SW128 = 2, LAYOUT_SW64 = 4 };
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// chunk index -> (n, first output row, first output x)
struct Chunk {
  int n, y0, x0;
};
__device__ __forceinline__ Chunk chunk_coords(long long ch, const TcParams &p) {
  const int per_img = p.rgroups * p.xblocks;
  Chunk c;
  c.n = (int)(ch / per_img);
  const int r = (int)(ch - (long long)c.n * per_img);
  const int g = r / p.xblocks;
  c.y0 = g * p.rc;
  c.x0 = (r - g * p.xblocks) * p.xw;
  return c;
}

template <int PASSES>
__global__ void __launch_bounds__(THREADS, 1) conv_tc_kernel(const __grid_constant__ TcParams p) {
  constexpr int CPT = TILE_P / 32;           // chunks per tile
  constexpr uint32_t A_LBO = 32 * BC * 4;    // chunk stride: 2 KB
  constexpr uint32_t A_SBO = 4 * 128;        // 4 channel rows of 128 B
  constexpr uint32_t A_KSTEP = 8 * 128;      // one UMMA K-step (8 channels)
  constexpr int LOADERS = THREADS - 64;      // warps 2.. : operand gather/split + epilogue
  constexpr int CH_PER_LOADER = BC * TILE_P / LOADERS;

  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
  // bars[0,S): full (filter TMA landed), [S,2S): ready (A gathered + split), [2S,3S): empty (MMA done), [3S]: accum
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mt = blockIdx.x % p.mtiles;
  const long long pt = blockIdx.x / p.mtiles;
  const int m0 = mt * p.NF;
  const long long ch0 = pt * CPT;
  const int KB = p.cblocks * p.taps;
  const uint32_t smem_base = smem_u32(smem);
  const uint32_t bar_base = smem_u32(bars);
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto ready_bar = [&](int s) { return bar_base + 8u * (S + s); };
  auto empty_bar = [&](int s) { return bar_base + 8u * (2 * S + s); };
  const uint32_t accum_bar = bar_base + 8u * (3 * S);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(full_bar(s), 1);
      mbar_init(ready_bar(s), LOADERS);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM allocation: whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&p.wmap) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;
  // Programmatic dependent launch: everything above overlaps the previous grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ filter-tile TMA producer
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(empty_bar(s), ((kb / S) - 1) & 1, p.spin_limit, p.dbg, 0x100000u | kb);
        const int cb = kb / p.taps;
        const int t = kb - cb * p.taps;
        mbar_expect_tx(full_bar(s), p.b_bytes);
        tma_load_3d(smem_base + (uint32_t)s * p.stage_bytes + A_BYTES, &p.wmap, full_bar(s), cb * BC, m0, t);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        const uint32_t ph = (kb / S) & 1;
        if (PASSES == 1) mbar_wait(full_bar(s), ph, p.spin_limit, p.dbg, 0x200000u | kb);
        mbar_wait(ready_bar(s), ph, p.spin_limit, p.dbg, 0x280000u | kb);
        tc_fence_after();
        if (p.dbg && kb == 0 && blockIdx.x == 0) {  // dump stage 0 of CTA 0
          const uint32_t *src = reinterpret_cast<const uint32_t *>(smem);
          for (int i = 0; i < p.stage_bytes / 4 && i < 65536; i++) p.dbg[16 + i] = src[i];
        }
        const uint32_t sa = smem_base + (uint32_t)s * p.stage_bytes;
        const uint32_t sb = sa + A_BYTES;
        const uint32_t lo = A_BYTES + p.b_bytes;  // offset of the lo twins
#pragma unroll
        for (int k = 0; k < BC / 8; k++) {
          const uint64_t a_hi = umma_desc(sa + k * A_KSTEP, A_LBO, A_SBO, LAYOUT_SW128_BASE32B);
          const uint64_t b_hi = umma_desc(sb + k * 32, 16, 512, LAYOUT_SW64);
          umma_tf32(tmem_d, a_hi, b_hi, p.idesc, (kb | k) != 0);
          if (PASSES == 3) {
            const uint64_t a_lo = umma_desc(sa + lo + k * A_KSTEP, A_LBO, A_SBO, LAYOUT_SW128_BASE32B);
            const uint64_t b_lo = umma_desc(sb + lo + k * 32, 16, 512, LAYOUT_SW64);
            umma_tf32(tmem_d, a_hi, b_lo, p.idesc, 1);
            umma_tf32(tmem_d, a_lo, b_hi, p.idesc, 1);
          }
        }
        umma_commit(empty_bar(s));  // frees the stage once these MMAs have read it
      }
      umma_commit(accum_bar);
    }
  } else {
    const int lt = threadIdx.x - 64;  // 0..LOADERS-1
    // ----------------------------------------------- A-operand gather (+ split)
    // Loader lt owns tile pixel pix = lt % 128 and CH_PER_LOADER channels of
    // each 16-channel block.  The shifted input element for tap (ky, kx) is
    // read straight from global (L1-cached: the 3x3 / 5x5 taps re-touch the
    // same rows); out-of-image positions read as +0.0 (virtual padding,
    // tensor.py:112-123).  TMA cannot do this shift: tiled boxes need a
    // 16-byte aligned innermost coordinate.
    const int pix = lt & (TILE_P - 1);
    const int cgrp = lt / TILE_P;
    long long pbase = -1;  // element offset of (n, 0, iy0, ix0) or -1 for a padding pixel of the tile
    int iy0 = 0, ix0 = 0;
    {
      const long long ch = ch0 + (pix >> 5);
      if (ch < p.nchunks) {
        const Chunk c = chunk_coords(ch, p);
        const int yy = (pix & 31) / p.xw;
        const int y = c.y0 + yy;
        const int x = c.x0 + (pix & 31) - yy * p.xw;
        if (y < p.Ho && x < p.Wo) {
          iy0 = p.flat ? 0 : y * p.S - p.PH;
          ix0 = p.flat ? x : x * p.S - p.PW;
          pbase = (long long)c.n * p.C * p.HW;
        }
      }
    }
    // smem byte offset of (channel c, pixel pix) in the A tile (32B-atom swizzle)
    auto a_off = [&](int c) -> uint32_t {
      const uint32_t L = (uint32_t)((pix >> 5) * 2048 + (c >> 2) * 512 + (c & 3) * 128 + (pix & 31) * 4);
      return L ^ (((L >> 7) & 3u) << 5);
    };
    const float *xg = p.x;
    const int Hh = p.flat ? 1 : p.H;     // flattened 1x1: one "row" of H*W pixels
    const int Ww = p.flat ? p.HW : p.W;
    for (int kb = 0; kb < KB; kb++) {
      const int s = kb % S;
      const int cb = kb / p.taps;
      const int t = kb - cb * p.taps;
      const int ky = t / p.WF;
      const int kx = t - ky * p.WF;
      // gather into registers before waiting for the stage to be free
      float v[CH_PER_LOADER];
      const int c0 = cb * BC + cgrp * CH_PER_LOADER;
      const int iy = iy0 + ky, ix = ix0 + kx;
      const bool ok = pbase >= 0 && iy >= 0 && iy < Hh && ix >= 0 && ix < Ww;
      const float *src = xg + pbase + (long long)c0 * p.HW + (long long)iy * Ww + ix;
#pragma unroll
      for (int j = 0; j < CH_PER_LOADER; j++) v[j] = (ok && c0 + j < p.C) ? __ldg(src + (long long)j * p.HW) : 0.0f;
      if (kb >= S) mbar_wait(empty_bar(s), ((kb / S) - 1) & 1, p.spin_limit, p.dbg, 0x300000u | kb);
      uint8_t *st = smem + (size_t)s * p.stage_bytes;
      const uint32_t lo = A_BYTES + p.b_bytes;
#pragma unroll
      for (int j = 0; j < CH_PER_LOADER; j++) {
        const uint32_t o = a_off(cgrp * CH_PER_LOADER + j);
        *reinterpret_cast<float *>(st + o) = v[j];  // the tensor core reads tf32 = v truncated
        if (PASSES == 3) {
          const float h = __uint_as_float(__float_as_uint(v[j]) & 0xFFFFE000u);
          *reinterpret_cast<float *>(st + lo + o) = v[j] - h;
        }
      }
      if (PASSES == 3) {  // filter lo twins once the filter TMA has landed
        mbar_wait(full_bar(s), (kb / S) & 1, p.spin_limit, p.dbg, 0x380000u | kb);
        const float4 *b = reinterpret_cast<const float4 *>(st + A_BYTES);
        float4 *bl = reinterpret_cast<float4 *>(st + lo + A_BYTES);
        for (int i = lt; i < p.b_bytes / 16; i += LOADERS) {
          const float4 a = b[i];
          float4 l;
          l.x = a.x - __uint_as_float(__float_as_uint(a.x) & 0xFFFFE000u);
          l.y = a.y - __uint_as_float(__float_as_uint(a.y) & 0xFFFFE000u);
          l.z = a.z - __uint_as_float(__float_as_uint(a.z) & 0xFFFFE000u);
          l.w = a.w - __uint_as_float(__float_as_uint(a.w) & 0xFFFFE000u);
          bl[i] = l;
        }
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(ready_bar(s));
    }
    // ------------------------------------------------------------------ epilogue
    mbar_wait(accum_bar, 0, p.spin_limit, p.dbg, 0x400000u);
    tc_fence_after();
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // which 32-column groups this warp drains
    const int row = q * 32 + lane;
    const int ci = row >> 5;
    const int yi = (row & 31) / p.xw;
    const int xi = (row & 31) - yi * p.xw;
    const long long ch = ch0 + ci;
    bool valid = ch < p.nchunks;
    long long obase = 0;
    if (valid) {
      const Chunk c = chunk_coords(ch, p);
      const int x = c.x0 + xi;
      const int y = c.y0 + yi;
      valid = x < p.Wo && y < p.Ho;
      obase = ((long long)c.n * p.M + m0) * p.HoWo + (long long)y * p.Wo + x;
    }
    const int mlim = min(p.NF, p.M - m0);
    for (int j0 = half * 32; j0 < p.NF; j0 += 64) {
      uint32_t r[32];
      tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + j0, r);
      if (p.dbg && blockIdx.x == 0) {  // dump the raw accumulator of CTA 0: [row][col]
        for (int j = 0; j < 32; j++) p.dbg[16 + 65536 + row * 256 + j0 + j] = r[j];
      }
      if (valid) {
#pragma unroll
        for (int j = 0; j < 32; j++)
          if (j0 + j < mlim) p.y[obase + (long long)(j0 + j) * p.HoWo] = __uint_as_float(r[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(p.tmem_cols) : "memory");
  }
}

// Filters [m][c][ky][kx] -> [tap][m][cp] (cp = C rounded up to 4, zero padded):
// the K-major layout TMA needs (16-byte row strides).  Weight-only (no input
// data is transformed), one launch per call, 4*taps*M*cp bytes of workspace.
__global__ void __launch_bounds__(256) filter_relayout_kernel(const float *__restrict__ w, float *__restrict__ wp,
                                                              int M, int C, int Cp, int taps) {
  const long long total = (long long)taps * M * Cp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cp);
    const long long r = i / Cp;
    const int m = (int)(r % M);
    const int t = (int)(r / M);
    wp[i] = c < C ? w[((long long)m * C + c) * taps + t] : 0.0f;
  }
}

}  // namespace tc
}  // namespace b2c
