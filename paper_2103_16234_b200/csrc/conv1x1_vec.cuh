// Pointwise (1x1, stride 1, no padding) fp32 convolution with 16-byte operand
// paths, for planes with H*W % 4 == 0 (GoogLeNet 28x28/14x14, ResNet 56/28/14).
//
// Same arithmetic contract as the fused engine of conv_kernel.cuh (FFMA2,
// per-output order: channels ascending within each split range; split ranges
// combined by stage2_sum_kernel), different register/shared-memory mapping:
//
//   warp tile   = 32 output channels x 64 output pixels, as 4 channel groups x
//                 8 pixel groups of lanes; thread = 8 channels x 8 pixels
//                 (channels {4g..4g+3, 16+4g..16+4g+3}, pixels {4h..4h+3,
//                 32+4h..32+4h+3}), so per input channel a thread issues two
//                 LDS.128 for filters and two LDS.128 for pixels (each warp-wide
//                 load touches 4 or 8 distinct 16-byte words, conflict-free)
//                 against 32 FFMA2 — a third of the shared-memory wavefronts of
//                 the broadcast mapping.
//   CTA         = WM x WP warps (BM = 32*WM channels x BP = 64*WP pixels)
//   staging     = pixels as 16-byte cp.async groups (4 consecutive pixels never
//                 straddle an image when H*W % 4 == 0), filters transposed to
//                 [c][m] by 4-byte cp.async, 3-stage pipeline over BC channels.
//   epilogue    = STG.128 of 4 consecutive pixels per channel.
#pragma once

#include <type_traits>

#include "conv_kernel.cuh"

namespace b2c {

// VEC = false: planes with H*W % 4 != 0 (7x7 GoogLeNet 5a/5b, 27x27) and
// stride-S 1x1 layers (ResNet projection shortcuts): the same register /
// shared mapping, pixels staged by 4-byte cp.async with a per-pixel input
// offset (subsampled by S; a 4-pixel group may straddle two images) and
// scalar output stores.
// TM = channel groups of 4 per thread: TM = 2 -> a thread holds 8 channels x
// 8 pixels (warp tile 32 x 64), TM = 4 -> 16 channels x 8 pixels (warp tile
// 64 x 64).  Per channel a thread loads TM + 2 float4 from shared memory for
// 16*TM FFMA2 (32*TM FMAs): 16 B of operands per 8 FMAs at TM = 2 — exactly
// the 128 B/clk shared-memory rate at the 128 FMA/clk FFMA2 peak (measured:
// ~3.8 wavefronts per LDS.128, FMA pipe ~67 % active, the two pipes
// co-limiting) — and 24 B per 16 FMAs at TM = 4 (75 % of the shared-memory
// rate at peak), at 128 accumulators per thread: 4-warp CTAs, 3 per SM.
template <int WM, int WP, int BC, int TM = 2>
struct Vec1x1Tile {
  static constexpr int BM = 16 * TM * WM;
  static constexpr int BP = 64 * WP;
  static constexpr int NT = 32 * WM * WP;
  static constexpr int WS = BM + 4;  // filter row stride (floats)
  static constexpr int STAGES = BC >= 32 ? 2 : 3;  // 32-channel chunks: two stages fit two CTAs per SM
  static constexpr int XG = BC * BP / 4;  // 16-byte pixel groups per chunk
  static constexpr int XG_PER_THREAD = (XG + NT - 1) / NT;
  static constexpr int STAGE_FLOATS = BC * BP + BC * WS;
  static constexpr int MIN_BLOCKS = TM == 2 ? (NT >= 512 ? 1 : 512 / NT) : (NT <= 128 ? 3 : 1);
};

// split-C through DSMEM (see cluster_reduce_tile in conv_kernel.cuh): park the
// accumulator tile [BM][BP] in this CTA's shared memory, then reduce.
template <int BM, int BP, int TM>
__device__ __forceinline__ void vec_park_tile(const float2 (&acc)[2 * TM][8], float *tile, int wrow, int xcol) {
  __syncthreads();  // every warp is done with the pipeline stages the tile overwrites
#pragma unroll
  for (int g = 0; g < 2; g++)
#pragma unroll
    for (int r = 0; r < 4 * TM; r++) {
      const int pr = r >> 1;
      const bool hi = r & 1;
      float4 v;
      v.x = hi ? acc[pr][4 * g + 0].y : acc[pr][4 * g + 0].x;
      v.y = hi ? acc[pr][4 * g + 1].y : acc[pr][4 * g + 1].x;
      v.z = hi ? acc[pr][4 * g + 2].y : acc[pr][4 * g + 2].x;
      v.w = hi ? acc[pr][4 * g + 3].y : acc[pr][4 * g + 3].x;
      const int row = wrow + (r & 3) + (r >> 2) * 16;
      *reinterpret_cast<float4 *>(tile + row * BP + xcol + 32 * g) = v;
    }
}

template <int BM, int BP, int NT, int TM>
__device__ __forceinline__ void vec_cluster_epilogue(const KParams &p, const float2 (&acc)[2 * TM][8], float *tile,
                                                     int m0, int q0, int wrow, int xcol) {
  vec_park_tile<BM, BP, TM>(acc, tile, wrow, xcol);
  cluster_reduce_tile<BM, BP, NT>(p, tile, m0, q0);
}

// Work items: (split, pixel tile, channel tile) flattened as
//   item = split * (mtiles * ptiles) + pt * mtiles + mt,
// the channel tiles of one pixel tile adjacent (they share the staged pixels
// through L2).  A CTA processes items blockIdx.y * gridDim.x + blockIdx.x,
// then + gridDim.x * gridDim.y, ...: grid = (items, 1) runs one item per CTA,
// grid = (tiles, splits) is the cluster launch (the splits of a tile form one
// cluster), and a smaller grid makes the kernel persistent (p.persistent): the
// cp.async pipeline then runs continuously across item boundaries — the next
// item's first chunks are in flight while this item's last chunks compute and
// its accumulators are stored — so the per-tile prologue and pipeline fill of
// a one-tile-per-CTA launch disappear (the short-K layers: ResNet C = 64 is 4
// chunks per tile).  Per-item setup is a few integer ops per thread: every
// thread's pixel group is the same for all of its channel rows, and its filter
// elements are fixed (m, c) offsets.
//
// PACKED (kind 9, with VEC): p.x is not the caller's x but its pixels packed by
// pack_pixels_kernel into x'[C][qp] (q = n*Ho*Wo + oy*Wo + ox, the stride
// applied), so 4 consecutive pixels are one 16-byte group whatever the plane
// size or stride — the 16-byte path for 7x7 planes and projection shortcuts.
// Outputs are stored to the caller's NCHW y (float4 when Ho*Wo % 4 == 0, else
// per pixel).  Same per-output arithmetic as every other pointwise family.
template <int WM, int WP, int BC, bool VEC = true, int TM = 2, bool PACKED = false>
__global__ void __launch_bounds__(Vec1x1Tile<WM, WP, BC, TM>::NT, Vec1x1Tile<WM, WP, BC, TM>::MIN_BLOCKS)
    conv1x1_vec_kernel(const KParams p) {
  static_assert(!PACKED || VEC, "packed pixels are staged as 16-byte groups");
  using T = Vec1x1Tile<WM, WP, BC, TM>;
  constexpr int BM = T::BM, BP = T::BP, NT = T::NT, WS = T::WS, STAGES = T::STAGES;
  constexpr int GPR = BP / 4;                  // 16-byte pixel groups per channel row of a chunk
  constexpr int XK = T::XG_PER_THREAD;         // channel rows per thread per chunk
  constexpr int CSTEP = NT / GPR;              // channel distance between a thread's rows
  constexpr int WK = BM * BC / NT;             // filter elements per thread per chunk
  static_assert(NT % GPR == 0 && XK * CSTEP == BC && (BM * BC) % NT == 0 && NT % BC == 0, "tile shape");
  extern __shared__ __align__(16) float smem[];

  const int tid = threadIdx.x;
  const unsigned long long t_start = p.trace ? global_ns() : 0ull;
  const int lane = tid & 31, wid = tid >> 5;
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int mgi = lane >> 3, pgi = lane & 7;
  const int hw = p.HoWo;            // output plane (== input plane for VEC: 1x1, stride 1, no padding)
  const int in_hw = PACKED ? p.qp : p.H * p.W;  // input plane (!VEC may subsample: stride S, no padding)
  const long long chw = (long long)p.C * in_hw;
  const long long tiles = (long long)p.mtiles * p.ptiles;
  const long long items = tiles * p.splits;
  const long long step = (long long)gridDim.x * gridDim.y;

  // fixed per-thread loader geometry
  const int pg = tid % GPR;         // this thread's pixel group (same for all its channel rows)
  const int c_row0 = tid / GPR;     // its first channel row; rows c_row0 + k*CSTEP
  const int wc = tid % BC;          // filter elements (m = tid/BC + j*NT/BC, c = wc)
  const int wm0 = tid / BC;

  // ---- per-item decoding ---------------------------------------------------------
  struct Item {
    int m0, q0, split, cb, ce;      // channel/pixel tile origin, split, chunk range [cb, ce)
  };
  auto decode = [&](long long it) {
    Item d;
    d.split = (int)(it / tiles);
    const long long t = it - (long long)d.split * tiles;
    const int pt = (int)(t / p.mtiles);
    d.m0 = (int)(t - (long long)pt * p.mtiles) * BM;
    d.q0 = pt * BP;
    d.cb = d.split * p.chunks_per_split;
    d.ce = min(p.nchunks, d.cb + p.chunks_per_split);
    return d;
  };

  // ---- loader state: the item whose chunks are being staged --------------------------
  constexpr int PX = VEC ? 1 : 4;
  using Off = typename std::conditional<VEC, long long, int>::type;  // !VEC: the planner guarantees n*c*h*w < 2^31
  Off xoff[PX];  // element offset of this thread's pixel(s) at channel 0 (-1: beyond the last pixel)
  const float *wrow = nullptr;  // &w[m0 + wm0][wc]
  int l_m0 = 0;
  auto setup_loader = [&](const Item &d) {
#pragma unroll
    for (int e = 0; e < PX; e++) {
      const int q = d.q0 + 4 * pg + e;
      if (q < p.Q) {
        const int n = q / hw;
        const int r = q - n * hw;
        if (PACKED) {
          xoff[e] = (Off)q;
        } else if (VEC) {
          xoff[e] = (Off)((long long)n * chw + r);
        } else {
          const int oy = r / p.Wo;
          const int ox = r - oy * p.Wo;
          xoff[e] = (Off)((long long)n * chw + (long long)oy * p.S * p.W + ox * p.S);
        }
      } else {
        xoff[e] = -1;
      }
    }
    l_m0 = d.m0;
    wrow = p.w + (long long)(d.m0 + wm0) * p.C + wc;
  };
  auto load_chunk = [&](int chunk, float *stage) {
    const int c0 = chunk * BC;
#pragma unroll
    for (int k = 0; k < XK; k++) {
      const int c = c_row0 + k * CSTEP;
      float *dst = stage + c * BP + 4 * pg;
      const bool cok = c0 + c < p.C;
      const float *src = p.x + (long long)(c0 + c) * in_hw;
      if (VEC) {
        if (xoff[0] >= 0 && cok)
          cp_async16(dst, src + xoff[0]);
        else
          *reinterpret_cast<float4 *>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int e = 0; e < PX; e++) {
          if (xoff[e] >= 0 && cok)
            cp_async4(dst + e, src + xoff[e]);
          else
            dst[e] = 0.0f;
        }
      }
    }
    float *ws = stage + BC * BP;
    const bool c_ok = c0 + wc < p.C;
#pragma unroll
    for (int j = 0; j < WK; j++) {
      const int m = wm0 + j * (NT / BC);
      float *dst = ws + wc * WS + m;
      if (l_m0 + m < p.M && c_ok)
        cp_async4(dst, wrow + (long long)j * (NT / BC) * p.C + c0);
      else
        *dst = 0.0f;
    }
  };

  float2 acc[2 * TM][8];
#pragma unroll
  for (int i = 0; i < 2 * TM; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.f, 0.f);

  const long long item0 = (long long)blockIdx.y * gridDim.x + blockIdx.x;
  if (item0 >= items) return;
  if (p.trace && tid == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.trace[5 * cta] = smid();
    p.trace[5 * cta + 1] = t_start;
    p.trace[5 * cta + 2] = global_ns();
  }

  // loader cursor (l_it, l_chunk) runs STAGES-1 chunks ahead of the compute cursor
  long long l_it = item0;
  Item ld = decode(l_it);
  int l_chunk = ld.cb;
  setup_loader(ld);
  auto advance_loader = [&]() {
    if (++l_chunk >= ld.ce) {
      l_it += step;
      if (l_it < items) {
        ld = decode(l_it);
        l_chunk = ld.cb;
        setup_loader(ld);
      }
    }
  };

  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (l_it < items) {
      load_chunk(l_chunk, smem + s * T::STAGE_FLOATS);
      advance_loader();
    }
    cp_async_commit();
  }
  const int xcol = wp * 64 + pgi * 4;
  const int wrow_s = wm * (16 * TM) + mgi * 4;
  long long c_it = item0;
  Item cd = decode(c_it);
  int c_chunk = cd.cb;
  for (int i = 0;; i++) {
    // issue chunk i+STAGES-1 into the stage freed by chunk i-1
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (l_it < items) {
      load_chunk(l_chunk, smem + ((i + STAGES - 1) % STAGES) * T::STAGE_FLOATS);
      advance_loader();
    }
    cp_async_commit();

    const float *xs = smem + (i % STAGES) * T::STAGE_FLOATS;
    const float *ws = xs + BC * BP + wrow_s;
    xs += xcol;
    const int cvalid = min(BC, p.C - c_chunk * BC);
#pragma unroll 2
    for (int c = 0; c < cvalid; c++) {
      float2 wp2[2 * TM];
#pragma unroll
      for (int k = 0; k < TM; k++) {
        const float4 wk = *reinterpret_cast<const float4 *>(ws + 16 * k);
        wp2[2 * k] = make_float2(wk.x, wk.y);
        wp2[2 * k + 1] = make_float2(wk.z, wk.w);
      }
      const float4 xa = *reinterpret_cast<const float4 *>(xs);
      const float4 xb = *reinterpret_cast<const float4 *>(xs + 32);
      ws += WS;
      xs += BP;
      const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int r = 0; r < 2 * TM; r++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[r][j] = __ffma2_rn(wp2[r], make_float2(xv[j], xv[j]), acc[r][j]);
    }
    if (++c_chunk < cd.ce) continue;

    // ---- item complete: epilogue ---------------------------------------------------
    const bool last = c_it + step >= items;
    if (last) {
      cp_async_wait<0>();
      if (p.trace && tid == 0) {
        const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        p.trace[5 * cta + 3] = global_ns();
      }
      if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    const int m0 = cd.m0, q0 = cd.q0;
    if (p.cluster) {  // one item per CTA (cluster launch)
      vec_cluster_epilogue<BM, BP, NT, TM>(p, acc, smem, m0, q0, wrow_s, xcol);
      break;
    }
    float *dst = p.splits > 1 ? p.partials + (long long)cd.split * p.part_stride : p.y;
    if (!VEC && !p.vec_out) {  // one item per CTA: transpose through shared memory, then coalesced per-pixel stores
      vec_park_tile<BM, BP, TM>(acc, smem, wrow_s, xcol);
      __syncthreads();
      store_tile_coalesced<BM, BP, NT>(p, smem, dst, m0, q0, 0, BM * BP);
      break;
    }
    if (PACKED && !p.vec_out) {  // Ho*Wo % 4 != 0: a 4-pixel group may straddle two images
#pragma unroll
      for (int g = 0; g < 2; g++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int q = q0 + xcol + 32 * g + j;
          if (q >= p.Q) continue;
          const int n = q / hw;
          const long long base = (long long)n * p.M * hw + (q - n * hw);
#pragma unroll
          for (int r = 0; r < 4 * TM; r++) {
            const int m = m0 + wrow_s + (r & 3) + (r >> 2) * 16;
            if (m >= p.M) continue;
            const float2 a = acc[r >> 1][4 * g + j];
            dst[base + (long long)m * hw] = (r & 1) ? a.y : a.x;
          }
        }
    } else
#pragma unroll
    for (int g = 0; g < 2; g++) {
      const int q = q0 + xcol + 32 * g;
      if (q >= p.Q) continue;
      const int n = q / hw;
      const long long base = (long long)n * p.M * hw + (q - n * hw);
#pragma unroll
      for (int r = 0; r < 4 * TM; r++) {
        const int m = m0 + wrow_s + (r & 3) + (r >> 2) * 16;
        if (m >= p.M) continue;
        const int pr = r >> 1;  // channel pair: rows {0,1}->0 {2,3}->1 {16,17}->2 {18,19}->3
        const bool hi = r & 1;
        float4 v;
        v.x = hi ? acc[pr][4 * g + 0].y : acc[pr][4 * g + 0].x;
        v.y = hi ? acc[pr][4 * g + 1].y : acc[pr][4 * g + 1].x;
        v.z = hi ? acc[pr][4 * g + 2].y : acc[pr][4 * g + 2].x;
        v.w = hi ? acc[pr][4 * g + 3].y : acc[pr][4 * g + 3].x;
        *reinterpret_cast<float4 *>(dst + base + (long long)m * hw) = v;
      }
    }
    if (last) break;
#pragma unroll
    for (int a = 0; a < 2 * TM; a++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[a][j] = make_float2(0.f, 0.f);
    c_it += step;
    cd = decode(c_it);
    c_chunk = cd.cb;
  }
  if (p.trace && tid == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.trace[5 * cta + 4] = global_ns();
  }
}

// Pixel packing for the packed pointwise families (kind 9): xp[c][q] =
// x[n][c][oy*S][ox*S] for q = n*Ho*Wo + oy*Wo + ox < Q, +0.0 for Q <= q < qp.
// HBM-bound gather (grid: qp/4/256 x C); its output stays largely in L2 for the
// convolution that follows.
__global__ void __launch_bounds__(256) pack_pixels_kernel(const KParams p, const float *__restrict__ x,
                                                          float *__restrict__ xp) {
  const int c = blockIdx.y;
  const int q = 4 * (blockIdx.x * 256 + threadIdx.x);
  if (q >= p.qp) return;
  const long long chw = (long long)p.C * p.H * p.W;
  const float *xc = x + (long long)c * p.H * p.W;
  float v[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int qq = q + j;
    v[j] = 0.0f;
    if (qq < p.Q) {
      const int n = fdiv(qq, p.mHoWo);
      const int r = qq - n * p.HoWo;
      const int oy = fdiv(r, p.mWo);
      const int ox = r - oy * p.Wo;
      v[j] = __ldg(xc + n * chw + (long long)oy * p.S * p.W + ox * p.S);
    }
  }
  *reinterpret_cast<float4 *>(xp + (long long)c * p.qp + q) = make_float4(v[0], v[1], v[2], v[3]);
}

}  // namespace b2c
