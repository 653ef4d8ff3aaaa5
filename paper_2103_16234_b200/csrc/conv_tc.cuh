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
// Filters arrive by bulk copy (pre-tiled once per call).  Taps are reduced into the same TMEM accumulator,
// so the paper's two reductions (channels within a filter row, then across
// filter rows) both happen inside the tensor core.  Any
// stride, padding, plane size and channel count are covered.
//
// Roles (576 threads, 1 CTA per SM):
//   warp 0      bulk-copy producer of the filter tiles (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..17 A gather in two groups taking alternate k-blocks (+ 3xTF32
//               lo twins of A), then the epilogue (tcgen05.ld -> coalesced
//               fp32 stores).
// The tensor core reads an fp32 operand as tf32 by truncation (measured), so
// the "hi" operands are the raw fp32 tiles and only the lo twins are written.
// Tile: UMMA M = 128 output pixels = 4 chunks of 32 (a chunk is RC output
// rows x XW output columns with RC*XW = 32 -- 1x32, 2x16 or 4x8 -- or 32
// consecutive pixels of the flattened plane for unpadded 1x1 layers),
// UMMA N = NF output channels (16..256), K = 16 input channels per pipeline
// stage (2 UMMA K-steps of 8).
//
// Shared-memory operand layout (canonical UMMA, both operands K-major, no
// swizzle): core matrices of 8 rows x 4 channels (128 B), K-adjacent ones
// 128 B apart (LBO), 8-row groups 512 B apart (SBO).  A (pixels) is written
// by the loaders with 16-byte stores, B (filters) arrives as one bulk copy
// of the pre-tiled hi [+ lo] planes per stage.  The 3xTF32 lo planes of the
// filters are computed once per call by the pre-tiling kernel.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"

namespace b2c {
namespace tc {

constexpr int BC = 16;          // input channels per pipeline stage
constexpr int TILE_P = 128;     // output pixels per tile (UMMA M)
constexpr int THREADS = 576;  // warp 0 bulk copies, warp 1 MMA, warps 2-17 gather + epilogue
constexpr int A_BYTES = TILE_P * BC * 4;  // 8 KB

struct TcParams {
  const float *wt;   // filters pre-tiled by filter_tile_kernel: [cb][tap][mtile][plane][NF/8][4][8][4]
  const float *x;    // input [n][c][h][w]
  float *y;
  int N, C, H, W, HW, S;
  int Hp, Wp, halo;  // halo variant: padded stack geometry, staged positions per tile
  int mh;            // halo variant: 128-position M halves per tile (1 or 2), sharing every filter tile
  int abufs;         // halo variant: staged halo buffers (ring of channel blocks in flight, >= 2)
  int flat;          // unpadded stride-1 1x1: chunks run over the flattened plane
  int M, Wo, HoWo;   // output geometry (Wo = HoWo for flattened 1x1)
  int Ho;            // output rows (1 for flattened)
  int xw, rc;        // chunk = rc output rows x xw output columns (xw * rc = 32)
  int rgroups;       // chunk rows per image: ceil(Ho / rc)
  int xblocks;       // chunks per row group: ceil(Wo / xw)
  long long nchunks; // N * rgroups * xblocks
  int PH, PW, WF, taps;
  int NF, mtiles, cblocks, Mp;
  int kpack, taps_full;      // gather mode K packing: k-blocks of 16 (channel, tap) pairs; taps == 1 then
  int splits, kb_per_split;  // split-K over k-blocks (blockIdx.y); partial planes summed by stage2_sum_kernel
  float *partials;           // [split][n][m][ho][wo] when splits > 1
  long long part_stride;
  int stages;
  int b_bytes;       // NF * 64
  int stage_bytes;   // (A_BYTES + b_bytes) * (PASSES == 3 ? 2 : 1)
  int tmem_cols;
  uint32_t idesc;    // UMMA instruction descriptor (kind::tf32, M=128, N=NF)
  unsigned long long spin_limit;  // mbarrier wait bound (ns) before __trap; 0 = unbounded (watchdog_ns())
  int mode;                       // development builds only (-DB2C_DEV, B2C_TC_MODE): 1 skip gather, 2 skip MMA, 4 skip B split,
                                  // 8 skip filter copy, 16 skip proxy fence, 32 skip A stores, 128 dumps
  unsigned int *dbg;              // development builds only (-DB2C_DEV, B2C_TC_DEBUG): wait-timeout codes and CTA-0 dumps
};

// Development instrumentation (role skipping, CTA-0 cycle dumps) exists only in
// builds with -DB2C_DEV (tools/ab_lib.sh); release builds compile it out.
#ifdef B2C_DEV
#define TC_MODE(bit) (p.mode & (bit))
#define TC_DBG p.dbg
#else
#define TC_MODE(bit) 0
#define TC_DBG (static_cast<unsigned int *>(nullptr))
#endif

// ------------------------------------------------------------------ PTX helpers
// smem_u32, mbarrier helpers and elect_one: ptx.cuh

__device__ __forceinline__ void sts32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float tf32_hi(float a) { return __uint_as_float(__float_as_uint(a) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_lo(float a) { return a - tf32_hi(a); }
// two floats -> packed bf16x2 (round to nearest even), low half = first
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void sts128u(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// UMMA shared-memory descriptor (sm100 layout: start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset 0, layout type [61,64)).
enum : uint64_t { LAYOUT_NONE = 0, LAYOUT_SW128_BASE32B = 1, LAYOUT_SW128 = 2, LAYOUT_SW64 = 4 };
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
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
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
  constexpr int CPT = TILE_P / 32;             // chunks per tile
  constexpr int LOADERS = THREADS - 64;        // warps 2.. : A gather + epilogue
  constexpr int GROUPS = 2;                    // loader groups, alternating k-blocks
  constexpr int GROUP_THREADS = LOADERS / GROUPS;
  constexpr int CH_PER_LOADER = BC * TILE_P / GROUP_THREADS;  // 8: two 4-channel core-matrix rows
  constexpr int LA = 2;                        // per-group look-ahead (k-blocks of loads in flight)
  constexpr uint32_t A_TILE = A_BYTES;         // one A plane (hi or lo)
  static_assert(CH_PER_LOADER == 8, "loader mapping assumes 8 channels per thread");

  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
  // bars[0,S): full (filter tile landed), [S,2S): ready (A gathered), [2S,3S): empty (MMA done), [3S]: accum
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mt = blockIdx.x % p.mtiles;
  const long long pt = blockIdx.x / p.mtiles;
  const int m0 = mt * p.NF;
  const long long ch0 = pt * CPT;
  // split-K: this CTA reduces k-blocks [kb_base, kb_base + KB) of the
  // (channel block, tap) sequence; kb below is local to the split
  const int kb_base = blockIdx.y * p.kb_per_split;
  const int KB = min(p.cblocks * p.taps - kb_base, p.kb_per_split);
  const uint32_t smem_base = smem_u32(smem);
  const uint32_t bar_base = smem_u32(bars);
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto ready_bar = [&](int s) { return bar_base + 8u * (S + s); };
  auto empty_bar = [&](int s) { return bar_base + 8u * (2 * S + s); };
  const uint32_t accum_bar = bar_base + 8u * (3 * S);
  // stage layout: [A hi | A lo (3xTF32) | B hi | B lo (3xTF32)], every operand in
  // no-swizzle K-major core matrices (8 rows x 16 B; K-adjacent 128 B apart,
  // 8-row groups 512 B apart)
  // PASSES 3: [A hi | A lo | B hi | B lo] fp32 planes; PASSES 2: [A fp32 | A bf16(hi) |
  // A bf16(lo) | B fp32 | B bf16(hi) | B bf16(lo)] (corrections as bf16 MMAs)
  const uint32_t b_off = A_TILE * (PASSES >= 2 ? 2 : 1);
  const uint32_t b_plane = (uint32_t)p.NF * BC * 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(full_bar(s), 1);
      mbar_init(ready_bar(s), GROUP_THREADS / 32);
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;
  // Programmatic dependent launch: everything above overlaps the previous grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    const bool leader = elect_one();
    {
      // ------------------------------------------------ filter-tile bulk-copy producer
      const bool prof = TC_DBG && blockIdx.x == 0 && leader;
      unsigned long long qt_wait = 0;
      const unsigned long long qt_start = prof ? clock64() : 0;
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        const unsigned long long c0 = prof ? clock64() : 0;
        if (kb >= S) mbar_wait(empty_bar(s), ((kb / S) - 1) & 1, p.spin_limit, TC_DBG, 0x100000u | kb);
        if (prof) qt_wait += clock64() - c0;
        if (TC_MODE(8)) {
          if (leader) mbar_arrive(full_bar(s));
          continue;
        }
        // the (cb, tap, filter tile) hi [+ lo] planes are one contiguous pre-tiled block
        const float *src = p.wt + ((long long)(kb_base + kb) * p.mtiles + mt) * (p.b_bytes / 4);
        if (leader) {
          mbar_expect_tx(full_bar(s), p.b_bytes);
          bulk_load(smem_base + (uint32_t)s * p.stage_bytes + b_off, src, p.b_bytes, full_bar(s));
        }
        __syncwarp();
      }
      if (prof) { TC_DBG[5] = (unsigned)qt_wait; TC_DBG[6] = (unsigned)(clock64() - qt_start); }
    }
  } else if (warp == 1) {
    const bool leader = elect_one();
    {
      // ------------------------------------------------------------ MMA issuer
      const bool prof = TC_DBG && blockIdx.x == 0 && leader;
      unsigned long long mt_wait = 0, mt_issue = 0;
      const unsigned long long mt_start = prof ? clock64() : 0;
      // both operands: no-swizzle K-major core matrices, LBO 128 B (K), SBO 512 B (rows)
      const uint64_t a_desc0 = umma_desc(smem_base, 128, 512, LAYOUT_NONE);
      const uint32_t idesc = p.idesc;
      const uint32_t nf = (uint32_t)p.NF;
      // bf16 planes: core matrices of 8 rows x 8 channels, SBO 256 B instead of 512 B
      const uint64_t sbo_delta = umma_desc(0, 128, 256, LAYOUT_NONE) - umma_desc(0, 128, 512, LAYOUT_NONE);
      const uint32_t idesc16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.NF >> 3) << 17) | (8u << 24);
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        const uint32_t ph = (kb / S) & 1;
        unsigned long long c0 = prof ? clock64() : 0;
        mbar_wait(full_bar(s), ph, p.spin_limit, TC_DBG, 0x200000u | kb);
        mbar_wait(ready_bar(s), ph, p.spin_limit, TC_DBG, 0x280000u | kb);
        tc_fence_after();
        if (prof) { const unsigned long long c = clock64(); mt_wait += c - c0; c0 = c; }
        // descriptors advanced by adding 16-byte units to the start-address field
        const uint64_t a0 = a_desc0 + (((uint32_t)s * p.stage_bytes) >> 4);
        const uint64_t b0 = a0 + (b_off >> 4);
        if (leader && !TC_MODE(2)) {
#pragma unroll
          for (int k = 0; k < BC / 8; k++) {
            const uint32_t acc = (kb | k) != 0;
            umma_tf32(tmem_d, a0 + k * 16, b0 + k * 16, idesc, acc);
            if (PASSES == 3) {  // correction terms into their own accumulator (columns NF..2NF):
              // the main accumulator then sees a third of the accumulation steps
              umma_tf32(tmem_d + nf, a0 + k * 16, b0 + (b_plane >> 4) + k * 16, idesc, acc);
              umma_tf32(tmem_d + nf, a0 + (A_TILE >> 4) + k * 16, b0 + k * 16, idesc, 1);
            }
          }
          if (PASSES == 2) {  // bf16 corrections, one K=16 MMA each: bf16(a_hi)*bf16(b_lo) + bf16(a_lo)*bf16(b_hi)
            const uint64_t a16 = a0 + (A_TILE >> 4) + sbo_delta;
            const uint64_t b16 = b0 + (b_plane >> 4) + sbo_delta;
            umma_f16(tmem_d + nf, a16, b16 + (uint64_t)(nf * 32 >> 4), idesc16, kb != 0);
            umma_f16(tmem_d + nf, a16 + (A_TILE / 2 >> 4), b16, idesc16, 1);
          }
        }
        if (leader) umma_commit(empty_bar(s));  // frees the stage once these MMAs have read it
        __syncwarp();
        if (prof) mt_issue += clock64() - c0;
      }
      if (leader) umma_commit(accum_bar);
      if (prof) { TC_DBG[3] = (unsigned)mt_wait; TC_DBG[4] = (unsigned)mt_issue; TC_DBG[2] = (unsigned)(clock64() - mt_start); }
    }
  } else {
    const int lt = threadIdx.x - 64;  // 0..LOADERS-1
    // ----------------------------------------------------------- A-operand gather
    // Two loader groups take alternate k-blocks (the per-k-block chain of
    // barrier waits and shared stores is latency-bound, so the groups overlap).
    // In a group, thread (pix, cg) owns tile pixel pix and channels 8cg..8cg+7
    // of each 16-channel block: two 16-byte K-major core-matrix rows.  The
    // shifted input element for tap (ky, kx) is read straight from global
    // (L1-cached: the hf*wf taps re-touch the same rows); out-of-image
    // positions read as +0.0 (virtual padding, tensor.py:112-123).
    const int grp = lt / GROUP_THREADS;
    const int gt = lt - grp * GROUP_THREADS;
    const int pix = gt & (TILE_P - 1);
    const int cgrp = gt / TILE_P;  // 0 or 1
    long long pbase = -1;  // element offset of image n, or -1 for a padding pixel of the tile
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
    // shared byte offset of this thread's first core-matrix row; the second
    // (channels +4) is 128 B further
    const uint32_t a_row = (uint32_t)((pix >> 3) * 512 + (2 * cgrp) * 128 + (pix & 7) * 16);
    const float *xg = p.x;
    const int Hh = p.flat ? 1 : p.H;  // flattened 1x1: one "row" of H*W pixels
    const int Ww = p.flat ? p.HW : p.W;
    auto gather = [&](int kb, float (&v)[CH_PER_LOADER]) {
      if (p.kpack) {
        // K packing (few input channels, e.g. a 7x7 stem on RGB): the reduction
        // index k = c*taps + tap runs contiguously over (channel, tap) pairs, so
        // a k-block holds 16 of them instead of 16 mostly-padding channels
        const int k0 = (kb_base + kb) * BC + cgrp * CH_PER_LOADER;
#pragma unroll
        for (int j = 0; j < CH_PER_LOADER; j++) {
          const int k = k0 + j;
          const int c = k / p.taps_full;
          const int t = k - c * p.taps_full;
          const int ky = t / p.WF, kx = t - (t / p.WF) * p.WF;
          const int iy = iy0 + ky, ix = ix0 + kx;
          const bool ok = pbase >= 0 && c < p.C && iy >= 0 && iy < Hh && ix >= 0 && ix < Ww;
          v[j] = ok ? __ldg(xg + pbase + (long long)c * p.HW + iy * Ww + ix) : 0.0f;
        }
        return;
      }
      const int cb = (kb_base + kb) / p.taps;
      const int t = (kb_base + kb) - cb * p.taps;
      const int ky = t / p.WF;
      const int kx = t - ky * p.WF;
      const int c0 = cb * BC + cgrp * CH_PER_LOADER;
      const int iy = iy0 + ky, ix = ix0 + kx;
      const bool ok = pbase >= 0 && iy >= 0 && iy < Hh && ix >= 0 && ix < Ww && !TC_MODE(1);
      const float *src = xg + pbase + (long long)c0 * p.HW + iy * Ww + ix;
      const int nc = ok ? min(CH_PER_LOADER, p.C - c0) : 0;
#pragma unroll
      for (int j = 0; j < CH_PER_LOADER; j++) v[j] = j < nc ? __ldg(src + (long long)j * p.HW) : 0.0f;
    };
    const bool prof = TC_DBG && blockIdx.x == 0 && lt == 0;  // development timing of loader warp 2
    unsigned long long pt_wait_e = 0, pt_store = 0, pt_fence = 0, pt_gather = 0;
    auto commit = [&](int kb, const float (&v)[CH_PER_LOADER]) {
      const int s = kb % S;
      unsigned long long c0 = prof ? clock64() : 0;
      if (kb >= S) {  // one lane polls, the warp follows
        if (lane == 0) mbar_wait(empty_bar(s), ((kb / S) - 1) & 1, p.spin_limit, TC_DBG, 0x300000u | kb);
        __syncwarp();
      }
      if (prof) { const unsigned long long c = clock64(); pt_wait_e += c - c0; c0 = c; }
      const uint32_t st = smem_base + (uint32_t)s * p.stage_bytes + a_row;
      if (!TC_MODE(32)) {
        sts128(st, make_float4(v[0], v[1], v[2], v[3]));  // the tensor core reads tf32 = v truncated
        sts128(st + 128, make_float4(v[4], v[5], v[6], v[7]));
        if (PASSES == 3) {
          sts128(st + A_TILE, make_float4(tf32_lo(v[0]), tf32_lo(v[1]), tf32_lo(v[2]), tf32_lo(v[3])));
          sts128(st + A_TILE + 128, make_float4(tf32_lo(v[4]), tf32_lo(v[5]), tf32_lo(v[6]), tf32_lo(v[7])));
        }
        if (PASSES == 2) {  // this thread's 8 channels are one bf16 core-matrix row (16 B)
          const uint32_t d16 = smem_base + (uint32_t)s * p.stage_bytes + A_TILE + (uint32_t)((pix >> 3) * 256 +
                               cgrp * 128 + (pix & 7) * 16);
          sts128u(d16, pack_bf16(tf32_hi(v[0]), tf32_hi(v[1])), pack_bf16(tf32_hi(v[2]), tf32_hi(v[3])),
                  pack_bf16(tf32_hi(v[4]), tf32_hi(v[5])), pack_bf16(tf32_hi(v[6]), tf32_hi(v[7])));
          sts128u(d16 + A_TILE / 2, pack_bf16(tf32_lo(v[0]), tf32_lo(v[1])), pack_bf16(tf32_lo(v[2]), tf32_lo(v[3])),
                  pack_bf16(tf32_lo(v[4]), tf32_lo(v[5])), pack_bf16(tf32_lo(v[6]), tf32_lo(v[7])));
        }
      }
      if (prof) { const unsigned long long c = clock64(); pt_store += c - c0; c0 = c; }
      // generic-proxy smem writes -> visible to the tensor core (async proxy);
      // one arrival per warp
      if (!TC_MODE(16)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(ready_bar(s));
      if (prof) pt_fence += clock64() - c0;
    };
    // software pipeline over this group's k-blocks: LA of them in flight
    float v[LA][CH_PER_LOADER];
    const unsigned long long pt_start = prof ? clock64() : 0;
#pragma unroll
    for (int u = 0; u < LA; u++)
      if (grp + GROUPS * u < KB) gather(grp + GROUPS * u, v[u]);
    for (int kb0 = grp; kb0 < KB; kb0 += GROUPS * LA) {
#pragma unroll
      for (int u = 0; u < LA; u++) {
        const int kb = kb0 + GROUPS * u;
        if (kb < KB) {
          commit(kb, v[u]);
          const unsigned long long c0 = prof ? clock64() : 0;
          if (kb + GROUPS * LA < KB) gather(kb + GROUPS * LA, v[u]);
          if (prof) pt_gather += clock64() - c0;
        }
      }
    }
    if (prof) {
      TC_DBG[7] = (unsigned)pt_wait_e; TC_DBG[8] = (unsigned)pt_store; TC_DBG[11] = (unsigned)pt_fence;
      TC_DBG[12] = (unsigned)pt_gather; TC_DBG[13] = (unsigned)(clock64() - pt_start);
    }
    // ------------------------------------------------------------------ epilogue
    if (lane == 0) mbar_wait(accum_bar, 0, p.spin_limit, TC_DBG, 0x400000u);
    __syncwarp();
    tc_fence_after();
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int colgrp = (warp - 2) >> 2;  // which 32-column groups this warp drains
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
    constexpr int COLGRPS = LOADERS / 128;
    for (int j0 = colgrp * 32; j0 < p.NF; j0 += 32 * COLGRPS) {
      uint32_t r[32];
      tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + j0, r);
      if (PASSES >= 2) {  // main + correction accumulator, fp32 round-to-nearest
        uint32_t c[32];
        tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + p.NF + j0, c);
#pragma unroll
        for (int j = 0; j < 32; j++) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(c[j]));
      }
      if (valid) {
        float *dst = p.splits > 1 ? p.partials + (long long)blockIdx.y * p.part_stride : p.y;
#pragma unroll
        for (int j = 0; j < 32; j++)
          if (j0 + j < mlim) dst[obase + (long long)(j0 + j) * p.HoWo] = __uint_as_float(r[j]);
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

// ---------------------------------------------------------------------------
// Halo variant (stride 1): the padded input is viewed as one flattened stack
// of rows of width Wp = W + 2*pw (image n occupies rows n*Hp .. n*Hp+Hp-1,
// Hp = H + 2*ph).  An output pixel at flattened position q = r*Wp + x needs
// input position q + ky*Wp + kx for tap (ky, kx): a CONSTANT shift.  So per
// 16-channel block the loaders stage the tile's halo -- positions
// [q0, q0 + 128 + (hf-1)*Wp + (wf-1)) -- once, K-major with one 16-byte row
// per position (8-position core-matrix groups 128 B apart, so position p sits
// at p*16 bytes), and every tap's A operand is the same buffer with the
// descriptor start moved by shift*16 bytes.  Loader work per channel block
// drops from hf*wf*128 positions to ~128 + (hf-1)*Wp, and the MMA issuer
// runs all taps of a block back to back.  Positions that fall on padding
// columns/rows or between images produce junk outputs that are not stored.
template <int PASSES, int MH>
__global__ void __launch_bounds__(THREADS, 1) conv_tc_halo_kernel(const __grid_constant__ TcParams p) {
  constexpr int LOADERS = THREADS - 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;                            // filter-tile ring depth

  const int TP = TILE_P * MH;                        // output positions per tile
  const uint32_t a_plane = (uint32_t)p.halo * 16u;   // bytes of one 4-channel K-core plane
  const uint32_t a_bytes = a_plane * 4u;             // one A plane (hi or lo): 16 channels
  // PASSES 3: fp32 hi + fp32 lo planes; PASSES 2: fp32 hi + bf16(hi) + bf16(lo)
  // planes (the correction products run as bf16 MMAs, K=16 at twice the rate)
  const uint32_t a_buf = a_bytes * (PASSES >= 2 ? 2u : 1u);
  const uint32_t b_plane = (uint32_t)p.NF * BC * 4;  // one fp32 filter plane
  const uint32_t b_stage = b_plane * (PASSES >= 2 ? 2u : 1u);
  const int SA = p.abufs;                            // halo ring depth (channel blocks in flight)
  uint8_t *bring = smem + (size_t)SA * a_buf;
  uint64_t *bars = reinterpret_cast<uint64_t *>(bring + (size_t)S * b_stage);
  // bars: [0,S) b_full (filter planes landed), [S,2S) unused, [2S,3S) b_empty,
  //       [3S, 3S+SA) a_full, [3S+SA, 3S+2SA) a_empty, 3S+2SA accum
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 2 * SA + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mt = blockIdx.x % p.mtiles;
  const long long pt = blockIdx.x / p.mtiles;
  const int m0 = mt * p.NF;
  const long long q0 = pt * TP;
  const int cb_per_split = p.kb_per_split / p.taps;
  const int cb_base = blockIdx.y * cb_per_split;
  const int NCB = min(p.cblocks - cb_base, cb_per_split);
  const int KB = NCB * p.taps;
  const uint32_t smem_base = smem_u32(smem);
  const uint32_t bring_base = smem_u32(bring);
  const uint32_t bar_base = smem_u32(bars);
  auto b_full = [&](int s) { return bar_base + 8u * s; };
  auto b_empty = [&](int s) { return bar_base + 8u * (2 * S + s); };
  auto a_full = [&](int b) { return bar_base + 8u * (3 * S + b); };
  auto a_empty = [&](int b) { return bar_base + 8u * (3 * S + SA + b); };
  const uint32_t accum_bar = bar_base + 8u * (3 * S + 2 * SA);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(b_full(s), 1);
      mbar_init(b_empty(s), 1);
    }
    for (int b = 0; b < SA; b++) {
      mbar_init(a_full(b), LOADERS / 32);
      mbar_init(a_empty(b), 1);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;
  if (TC_DBG && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 64) TC_DBG[11] = (unsigned)clock64();
  // TMEM columns: main accumulator of half h at h*NF, 3xTF32 correction at (MH+h)*NF
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    const bool leader = elect_one();
    {
      // ------------------------------------------- filter-tile (hi plane) bulk copies
      const bool prof = TC_DBG && blockIdx.x == 0 && blockIdx.y == 0 && leader;
      unsigned long long qt_wait = 0;
      const unsigned long long qt_start = prof ? clock64() : 0;
      for (int kb = 0; kb < KB; kb++) {
        const int s = kb % S;
        const unsigned long long c0 = prof ? clock64() : 0;
        if (kb >= S) mbar_wait(b_empty(s), ((kb / S) - 1) & 1, p.spin_limit, TC_DBG, 0x110000u | kb);
        if (prof) qt_wait += clock64() - c0;
        const uint32_t bytes = b_stage;  // fp32 hi [+ lo, or bf16 hi + lo] planes, one contiguous block
        const float *src = p.wt + ((long long)(cb_base * p.taps + kb) * p.mtiles + mt) * (bytes / 4);
        if (leader) {
          if (TC_MODE(8)) {
            mbar_arrive(b_full(s));
          } else {
            mbar_expect_tx(b_full(s), bytes);
            bulk_load(bring_base + (uint32_t)s * b_stage, src, bytes, b_full(s));
          }
        }
        __syncwarp();
      }
      if (prof) { TC_DBG[5] = (unsigned)qt_wait; TC_DBG[6] = (unsigned)(clock64() - qt_start); }
    }
  } else if (warp == 1) {
    const bool leader = elect_one();
    {
      // ------------------------------------------------------------ MMA issuer
      // Descriptors are built once per buffer / stage and advanced by adding
      // the 16-byte-unit offset to their start-address field (all operand
      // addresses stay below 256 KB, so the 14-bit field never carries).
      const bool prof = TC_DBG && blockIdx.x == 0 && blockIdx.y == 0 && leader;
      unsigned long long mt_wait = 0, mt_wait_a = 0;
      const unsigned long long mt_start = prof ? clock64() : 0;
      const uint64_t a_desc0 = umma_desc(smem_base, a_plane, 128, LAYOUT_NONE);
      const uint64_t b_desc0 = umma_desc(bring_base, 128, 512, LAYOUT_NONE);
      // bf16 planes: K-cores of 8 channels; A rows stay 16 B per position (LBO = halo*16),
      // B: LBO 128 B (next 8 channels), SBO 256 B (next 8 filters)
      const uint64_t a16_desc0 = umma_desc(smem_base, a_plane, 128, LAYOUT_NONE);
      const uint64_t b16_delta = umma_desc(0, 128, 256, LAYOUT_NONE) - umma_desc(0, 128, 512, LAYOUT_NONE);
      const uint32_t idesc16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.NF >> 3) << 17) | (8u << 24);
      (void)a16_desc0;
      const uint32_t idesc = p.idesc;
      const uint32_t nf = (uint32_t)p.NF;
      const int taps = p.taps, wf = p.WF, wp = p.Wp;
      for (int i = 0; i < NCB; i++) {
        const int buf = i % SA;
        unsigned long long c0 = prof ? clock64() : 0;
        mbar_wait(a_full(buf), (i / SA) & 1, p.spin_limit, TC_DBG, 0x210000u | i);
        if (prof) mt_wait_a += clock64() - c0;
        tc_fence_after();
        const uint64_t a_buf_desc = a_desc0 + ((buf * a_buf) >> 4);
        int ky = 0, kx = 0;
        for (int t = 0; t < taps; t++) {
          const int kb = i * taps + t;
          const int s = kb % S;
          c0 = prof ? clock64() : 0;
          mbar_wait(b_full(s), (kb / S) & 1, p.spin_limit, TC_DBG, 0x220000u | kb);
          if (prof) mt_wait += clock64() - c0;
          tc_fence_after();
          const uint64_t a0 = a_buf_desc + (uint64_t)((ky * wp + kx) & 0xFFFF);  // tap shift: 16 B per position
          const uint64_t b0 = b_desc0 + (uint64_t)((s * b_stage) >> 4);
          if (leader) {
#pragma unroll
            for (int k = 0; k < BC / 8; k++) {
              const uint64_t bh = b0 + k * 16;                       // +256 B per UMMA K-step
              const uint64_t bl = bh + (b_plane >> 4);
              const uint64_t ak = a0 + k * (2 * a_plane >> 4);       // +2 K-core planes
              const uint32_t acc = (kb | k) != 0;
              // consecutive MMAs target different accumulators (main of every
              // half, then the correction terms) so their latencies overlap
#pragma unroll
              for (int h = 0; h < MH; h++)
                if (!TC_MODE(2)) umma_tf32(tmem_d + h * nf, ak + h * (TILE_P * 16 >> 4), bh, idesc, acc);
              if (PASSES == 2 && k == 0) {
                // bf16 corrections over the whole 16-channel block (one K=16 MMA each)
                const uint32_t acc16 = kb != 0;
                const uint64_t bh16 = b0 + (b_plane >> 4) + b16_delta, bl16 = bh16 + (uint64_t)(nf * 32 >> 4);
#pragma unroll
                for (int h = 0; h < MH; h++) {
                  const uint64_t ah16 = a0 + (a_bytes >> 4) + h * (TILE_P * 16 >> 4);
                  if (!TC_MODE(2)) {
                    umma_f16(tmem_d + (MH + h) * nf, ah16, bl16, idesc16, acc16);
                  }
                }
#pragma unroll
                for (int h = 0; h < MH; h++) {
                  const uint64_t al16 = a0 + ((a_bytes + a_bytes / 2) >> 4) + h * (TILE_P * 16 >> 4);
                  if (!TC_MODE(2)) umma_f16(tmem_d + (MH + h) * nf, al16, bh16, idesc16, 1);
                }
              }
              if (PASSES == 3) {
#pragma unroll
                for (int h = 0; h < MH; h++)
                  if (!TC_MODE(2)) umma_tf32(tmem_d + (MH + h) * nf, ak + h * (TILE_P * 16 >> 4), bl, idesc, acc);
#pragma unroll
                for (int h = 0; h < MH; h++)
                  if (!TC_MODE(2))
                    umma_tf32(tmem_d + (MH + h) * nf, ak + h * (TILE_P * 16 >> 4) + (a_bytes >> 4), bh, idesc, 1);
              }
            }
            umma_commit(b_empty(s));
          }
          __syncwarp();
          if (++kx == wf) {
            kx = 0;
            ++ky;
          }
        }
        if (leader) umma_commit(a_empty(buf));  // the halo buffer is free once this block's MMAs have read it
        __syncwarp();
      }
      if (leader) umma_commit(accum_bar);
      if (prof) { TC_DBG[3] = (unsigned)mt_wait; TC_DBG[4] = (unsigned)mt_wait_a; TC_DBG[2] = (unsigned)(clock64() - mt_start); }
    }
  } else {
    // --------------------------------------- halo loaders (+ filter lo planes)
    // halo item = (position, 4-channel group): 4 strided loads, one 16-byte
    // store (+ the lo twin).  Consecutive lanes take consecutive positions
    // (coalesced rows of the input).
    const int lt = threadIdx.x - 64;
    const int items = p.halo * 4;
    const float *xg = p.x;
    const bool prof = TC_DBG && blockIdx.x == 0 && blockIdx.y == 0 && lt == 0;
    unsigned long long lt_wait = 0, lt_fill = 0;
    const unsigned long long lt_start = prof ? clock64() : 0;
    for (int i = 0; i < NCB; i++) {
      const int buf = i % SA;
      unsigned long long c0 = prof ? clock64() : 0;
      if (i >= SA) {
        if (lane == 0) mbar_wait(a_empty(buf), ((i / SA) - 1) & 1, p.spin_limit, TC_DBG, 0x310000u | i);
        __syncwarp();
      }
      if (prof) { const unsigned long long c = clock64(); lt_wait += c - c0; c0 = c; }
      const int cbase = (cb_base + i) * BC;
      const uint32_t sa = smem_base + buf * a_buf;
      for (int it = lt; it < items; it += LOADERS) {
        const int j = it / p.halo;          // 4-channel group
        const int pos = it - j * p.halo;    // halo position
        const long long pp = q0 + pos;      // flattened padded-stack index
        const long long r = pp / p.Wp;
        const int xx = (int)(pp - r * p.Wp) - p.PW;
        const int n = (int)(r / p.Hp);
        const int yy = (int)(r - (long long)n * p.Hp) - p.PH;
        const int c0 = cbase + j * 4;
        float v[4];
        const bool ok = n < p.N && yy >= 0 && yy < p.H && xx >= 0 && xx < p.W && !TC_MODE(1);
        const float *src = xg + ((long long)n * p.C + c0) * p.HW + (long long)yy * p.W + xx;
        const int nc = ok ? min(4, p.C - c0) : 0;
#pragma unroll
        for (int e = 0; e < 4; e++) v[e] = e < nc ? __ldg(src + (long long)e * p.HW) : 0.0f;
        const uint32_t dst = sa + (uint32_t)j * a_plane + (uint32_t)pos * 16u;
        sts128(dst, make_float4(v[0], v[1], v[2], v[3]));
        if (PASSES == 3)
          sts128(dst + a_bytes, make_float4(tf32_lo(v[0]), tf32_lo(v[1]), tf32_lo(v[2]), tf32_lo(v[3])));
        if (PASSES == 2) {  // bf16(hi), bf16(lo): K-core j/2 (8 channels), 8-byte half-row (j%2)
          const uint32_t d16 = sa + a_bytes + (uint32_t)(j >> 1) * a_plane + (uint32_t)pos * 16u + (j & 1) * 8u;
          sts64(d16, pack_bf16(tf32_hi(v[0]), tf32_hi(v[1])), pack_bf16(tf32_hi(v[2]), tf32_hi(v[3])));
          sts64(d16 + a_bytes / 2, pack_bf16(tf32_lo(v[0]), tf32_lo(v[1])), pack_bf16(tf32_lo(v[2]), tf32_lo(v[3])));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full(buf));
      if (prof) lt_fill += clock64() - c0;
    }
    if (prof) { TC_DBG[7] = (unsigned)lt_wait; TC_DBG[8] = (unsigned)lt_fill; TC_DBG[13] = (unsigned)(clock64() - lt_start); }
    // ------------------------------------------------------------------ epilogue
    const unsigned long long e0 = prof ? clock64() : 0;
    if (lane == 0) mbar_wait(accum_bar, 0, p.spin_limit, TC_DBG, 0x410000u);
    __syncwarp();
    tc_fence_after();
    if (prof) TC_DBG[9] = (unsigned)(clock64() - e0);
    const int q = warp & 3;
    const int colgrp = (warp - 2) >> 2;
    constexpr int COLGRPS = LOADERS / 128;
    const int mlim = min(p.NF, p.M - m0);
    float *dst = p.splits > 1 ? p.partials + (long long)blockIdx.y * p.part_stride : p.y;
    for (int h = 0; h < MH; h++) {
      const int row = q * 32 + lane;
      const long long qq = q0 + h * TILE_P + row;
      const long long r = qq / p.Wp;
      const int x = (int)(qq - r * p.Wp);
      const int n = (int)(r / p.Hp);
      const int y = (int)(r - (long long)n * p.Hp);
      const bool valid = n < p.N && y < p.Ho && x < p.Wo;
      const long long obase = ((long long)n * p.M + m0) * p.HoWo + (long long)y * p.Wo + x;
      for (int j0 = colgrp * 32; j0 < p.NF; j0 += 32 * COLGRPS) {
        uint32_t rr[32];
        tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + h * p.NF + j0, rr);
        if (PASSES >= 2) {
          uint32_t c[32];
          tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + (MH + h) * p.NF + j0, c);
#pragma unroll
          for (int j = 0; j < 32; j++) rr[j] = __float_as_uint(__uint_as_float(rr[j]) + __uint_as_float(c[j]));
        }
        if (valid) {
#pragma unroll
          for (int j = 0; j < 32; j++)
            if (j0 + j < mlim) dst[obase + (long long)(j0 + j) * p.HoWo] = __uint_as_float(rr[j]);
        }
      }
    }
  }
  if (TC_DBG && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 64) TC_DBG[10] = (unsigned)clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(p.tmem_cols) : "memory");
  }
}

// Filters [m][c][ky][kx] -> pre-tiled [cb][tap][filter tile][plane][NF/8][4][8][4]:
// for every 16-channel block cb, tap and filter tile, the NF x 16 operand in
// the UMMA no-swizzle K-major core-matrix order (8 rows x 16 bytes per core
// matrix; K-adjacent core matrices 128 B apart, 8-row groups 512 B apart),
// zero padded beyond M and C.  planes = 2 (3xTF32) appends the lo plane
// w - tf32(w).  Every pipeline stage's filter operands are then ONE
// contiguous block moved by a single bulk copy.  Weight-only (no input data
// is transformed): one launch per call.
__global__ void __launch_bounds__(256) filter_tile_kernel(const float *__restrict__ w, float *__restrict__ wt, int M,
                                                          int C, int taps, int NF, int mtiles, int cblocks,
                                                          int planes) {
  const long long tile = (long long)NF * BC;
  const long long total = (long long)cblocks * taps * mtiles * planes * tile;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int within = (int)(i % tile);
    const long long blk = i / tile;
    const int plane = (int)(blk % planes);
    const long long kbm = blk / planes;  // (cb, tap, filter tile)
    const int mt = (int)(kbm % mtiles);
    const long long kb = kbm / mtiles;
    const int t = (int)(kb % taps);
    const int cb = (int)(kb / taps);
    const int e = within & 3;         // element within a 16-byte core-matrix row
    const int r = (within >> 2) & 7;  // row within the core matrix
    const int j = (within >> 5) & 3;  // core matrix along K (4 channels each)
    const int g = within >> 7;        // 8-row group
    const int m = mt * NF + g * 8 + r;
    const int c = cb * BC + j * 4 + e;
    const float v = (m < M && c < C) ? w[((long long)m * C + c) * taps + t] : 0.0f;
    wt[i] = plane == 0 ? v : tf32_lo(v);
  }
}

// Filter tiles for the bf16-correction 3xTF32 variant (PASSES 2): per
// (cb, tap, filter tile) block, the fp32 plane (as filter_tile_kernel) then
// bf16(hi) and bf16(lo) planes in bf16 K-major core-matrix order (8 filters x
// 8 channels = 128 B per core matrix; K-adjacent 128 B apart, 8-filter groups
// 256 B apart).
__global__ void __launch_bounds__(256) filter_tile_bf16corr_kernel(const float *__restrict__ w, float *__restrict__ wt,
                                                                   int M, int C, int taps, int NF, int mtiles,
                                                                   int cblocks) {
  const long long tile = (long long)NF * BC;  // elements of one block
  const long long total = (long long)cblocks * taps * mtiles * tile;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long blk = i / tile;  // (cb, tap, filter tile)
    const int within = (int)(i - blk * tile);
    const int mt = (int)(blk % mtiles);
    const long long kb = blk / mtiles;
    const int t = (int)(kb % taps);
    const int cb = (int)(kb / taps);
    const int ml = within / BC, cl = within - (within / BC) * BC;  // local filter row, channel
    const int m = mt * NF + ml;
    const int c = cb * BC + cl;
    const float v = (m < M && c < C) ? w[((long long)m * C + c) * taps + t] : 0.0f;
    float *base = wt + blk * 2 * tile;  // 2 fp32-plane equivalents per block
    // fp32 plane: core (g = ml/8, j = cl/4), row ml%8, element cl%4
    base[(ml >> 3) * 128 + (cl >> 2) * 32 + (ml & 7) * 4 + (cl & 3)] = v;
    __nv_bfloat16 *b16 = reinterpret_cast<__nv_bfloat16 *>(base + tile);
    const int o16 = (ml >> 3) * 128 + (cl >> 3) * 64 + (ml & 7) * 8 + (cl & 7);  // in bf16 elements
    b16[o16] = __float2bfloat16_rn(tf32_hi(v));
    b16[NF * BC + o16] = __float2bfloat16_rn(tf32_lo(v));
  }
}

}  // namespace tc
}  // namespace b2c
