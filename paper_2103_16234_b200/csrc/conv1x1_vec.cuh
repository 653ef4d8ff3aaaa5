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
template <int WM, int WP, int BC>
struct Vec1x1Tile {
  static constexpr int BM = 32 * WM;
  static constexpr int BP = 64 * WP;
  static constexpr int NT = 32 * WM * WP;
  static constexpr int WS = BM + 4;  // filter row stride (floats)
  static constexpr int STAGES = 3;
  static constexpr int XG = BC * BP / 4;  // 16-byte pixel groups per chunk
  static constexpr int XG_PER_THREAD = (XG + NT - 1) / NT;
  static constexpr int STAGE_FLOATS = BC * BP + BC * WS;
  static constexpr int MIN_BLOCKS = NT >= 512 ? 1 : 512 / NT;
};

// split-C through DSMEM (see cluster_reduce_tile in conv_kernel.cuh): park the
// accumulator tile [BM][BP] in this CTA's shared memory, then reduce.
template <int BM, int BP>
__device__ __forceinline__ void vec_park_tile(const float2 (&acc)[4][8], float *tile, int wrow, int xcol) {
  __syncthreads();  // every warp is done with the pipeline stages the tile overwrites
#pragma unroll
  for (int g = 0; g < 2; g++)
#pragma unroll
    for (int r = 0; r < 8; r++) {
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

template <int BM, int BP, int NT>
__device__ __forceinline__ void vec_cluster_epilogue(const KParams &p, const float2 (&acc)[4][8], float *tile,
                                                     int m0, int q0, int wrow, int xcol) {
  vec_park_tile<BM, BP>(acc, tile, wrow, xcol);
  cluster_reduce_tile<BM, BP, NT>(p, tile, m0, q0);
}

template <int WM, int WP, int BC, bool VEC = true>
__global__ void __launch_bounds__(Vec1x1Tile<WM, WP, BC>::NT, Vec1x1Tile<WM, WP, BC>::MIN_BLOCKS)
    conv1x1_vec_kernel(const KParams p) {
  using T = Vec1x1Tile<WM, WP, BC>;
  constexpr int BM = T::BM, BP = T::BP, NT = T::NT, WS = T::WS, STAGES = T::STAGES;
  extern __shared__ __align__(16) float smem[];

  const int tid = threadIdx.x;
  const unsigned long long t_start = p.trace ? global_ns() : 0ull;
  const int lane = tid & 31, wid = tid >> 5;
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int mgi = lane >> 3, pgi = lane & 7;
  const int tile = blockIdx.x;
  const int mt = tile % p.mtiles;
  const int pt = tile / p.mtiles;
  const int m0 = mt * BM;
  const int q0 = pt * BP;
  const int split = blockIdx.y;
  const int hw = p.HoWo;            // output plane (== input plane for VEC: 1x1, stride 1, no padding)
  const int in_hw = p.H * p.W;      // input plane (!VEC may subsample: stride S, no padding)
  const long long chw = (long long)p.C * in_hw;

  // per-thread 16-byte pixel groups of a chunk: global offset relative to the
  // chunk's first channel (or -1 beyond the last pixel)
  constexpr int PX = VEC ? 1 : 4;  // offsets per 4-pixel group
  using Off = typename std::conditional<VEC, long long, int>::type;  // !VEC: the planner guarantees n*c*h*w < 2^31
  Off xoff[T::XG_PER_THREAD][PX];
  int xdst[T::XG_PER_THREAD];
#pragma unroll
  for (int k = 0; k < T::XG_PER_THREAD; k++) {
    const int gi = tid + k * NT;
    const int c = gi / (BP / 4);
    const int pg = gi - c * (BP / 4);
    const int q = q0 + 4 * pg;
    xdst[k] = gi < T::XG ? c * BP + 4 * pg : -1;
#pragma unroll
    for (int e = 0; e < PX; e++) {
      const int qe = q + e;
      if (gi < T::XG && qe < p.Q) {
        const int n = qe / hw;
        const int r = qe - n * hw;
        const int oy = r / p.Wo;
        const int ox = r - oy * p.Wo;
        xoff[k][e] = (Off)((long long)n * chw + (long long)c * in_hw + (long long)oy * p.S * p.W + ox * p.S);
      } else {
        xoff[k][e] = -1;
      }
    }
  }
  const float *wsrc0 = p.w + (long long)m0 * p.C;
  if (p.trace && tid == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.trace[5 * cta] = smid();
    p.trace[5 * cta + 1] = t_start;
    p.trace[5 * cta + 2] = global_ns();
  }

  auto load_chunk = [&](int chunk, float *stage) {
    const int c0 = chunk * BC;
    const int cvalid = min(BC, p.C - c0);
    const float *xsrc = p.x + (long long)c0 * in_hw;
#pragma unroll
    for (int k = 0; k < T::XG_PER_THREAD; k++) {
      if (xdst[k] < 0) continue;
      float *dst = stage + xdst[k];
      const int c = xdst[k] / BP;
      if (VEC) {
        if (xoff[k][0] >= 0 && c < cvalid)
          cp_async16(dst, xsrc + xoff[k][0]);
        else
          *reinterpret_cast<float4 *>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int e = 0; e < PX; e++) {
          if (xoff[k][e] >= 0 && c < cvalid)
            cp_async4(dst + e, xsrc + xoff[k][e]);
          else
            dst[e] = 0.0f;
        }
      }
    }
    float *ws = stage + BC * BP;
    const float *wsrc = wsrc0 + c0;
    for (int e = tid; e < BM * BC; e += NT) {
      const int m = e / BC;
      const int c = e - m * BC;
      float *dst = ws + c * WS + m;
      if (m0 + m < p.M && c < cvalid)
        cp_async4(dst, wsrc + (long long)m * p.C + c);
      else
        *dst = 0.0f;
    }
  };

  float2 acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.f, 0.f);

  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int chunk_begin = split * p.chunks_per_split;
  const int chunk_end = min(p.nchunks, chunk_begin + p.chunks_per_split);
  const int nck = chunk_end - chunk_begin;
  // prologue: STAGES-1 chunks in flight
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nck) load_chunk(chunk_begin + s, smem + s * T::STAGE_FLOATS);
    cp_async_commit();
  }
  const int xcol = wp * 64 + pgi * 4;
  const int wrow = wm * 32 + mgi * 4;
  for (int i = 0; i < nck; i++) {
    // issue chunk i+STAGES-1 into the stage freed by chunk i-1
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (i + STAGES - 1 < nck) load_chunk(chunk_begin + i + STAGES - 1, smem + ((i + STAGES - 1) % STAGES) * T::STAGE_FLOATS);
    cp_async_commit();

    const float *xs = smem + (i % STAGES) * T::STAGE_FLOATS;
    const float *ws = xs + BC * BP;
    const int cvalid = min(BC, p.C - (chunk_begin + i) * BC);
#pragma unroll 2
    for (int c = 0; c < cvalid; c++) {
      const float4 wa = *reinterpret_cast<const float4 *>(ws + c * WS + wrow);
      const float4 wb = *reinterpret_cast<const float4 *>(ws + c * WS + wrow + 16);
      const float4 xa = *reinterpret_cast<const float4 *>(xs + c * BP + xcol);
      const float4 xb = *reinterpret_cast<const float4 *>(xs + c * BP + xcol + 32);
      const float2 wp2[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                             make_float2(wb.z, wb.w)};
      const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[r][j] = __ffma2_rn(wp2[r], make_float2(xv[j], xv[j]), acc[r][j]);
    }
  }
  cp_async_wait<0>();

  if (p.trace && tid == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.trace[5 * cta + 3] = global_ns();
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (p.cluster) {
    vec_cluster_epilogue<BM, BP, NT>(p, acc, smem, m0, q0, wrow, xcol);
    if (p.trace && tid == 0) {
      const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      p.trace[5 * cta + 4] = global_ns();
    }
    return;
  }
  // epilogue: VEC -> one 16-byte store per 4 consecutive pixels of a channel;
  // !VEC (planes with H*W % 4 != 0, strided) -> the tile goes through shared
  // memory and every warp stores runs of consecutive pixels
  float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : p.y;
  if (!VEC) {  // transpose through shared memory, then coalesced per-pixel stores
    vec_park_tile<BM, BP>(acc, smem, wrow, xcol);
    __syncthreads();
    store_tile_coalesced<BM, BP, NT>(p, smem, dst, m0, q0, 0, BM * BP);
    if (p.trace && tid == 0) {
      const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      p.trace[5 * cta + 4] = global_ns();
    }
    return;
  }
#pragma unroll
  for (int g = 0; g < 2; g++) {
    const int q = q0 + xcol + 32 * g;
    if (q >= p.Q) continue;
    const int n = q / hw;
    const long long base = (long long)n * p.M * hw + (q - n * hw);
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int m = m0 + wrow + (r & 3) + (r >> 2) * 16;
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
  if (p.trace && tid == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.trace[5 * cta + 4] = global_ns();
  }
}

}  // namespace b2c
