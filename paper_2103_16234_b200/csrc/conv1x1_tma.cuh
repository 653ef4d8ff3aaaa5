// TMA-fed pointwise (1x1, stride 1, no padding, H*W % 4 == 0) fp32
// convolution: the register tile and arithmetic of conv1x1_vec_kernel, with
// every operand moved by the TMA engine instead of per-thread cp.async.
//
// Same arithmetic contract as the other fused kernels: per output, channels
// ascending (one FFMA each) within each split range — bitwise identical to
// them for equal split ranges.
//
// Why: ncu on conv1x1_vec_kernel (ResNet layer1, N=256) puts ~11 % of the
// warp samples in the staging code (address math + 2 x 8 cp.async per thread
// per 32-channel chunk) and ~6 % at the per-chunk __syncthreads.  Here:
//   * per stage ONE thread issues a 2-D TMA of the filter tile (the caller's
//     [M][C] filters, box {BC+4, BM}: 4 extra columns give the rows a 20-float
//     pitch so the 4 channel groups of a warp hit distinct banks; the extra
//     values are never read) and one or two 3-D TMAs of the pixel tile from x
//     viewed as [N][C][H*W] (box {BP, BC, 1}; a tile that runs into the next
//     image takes a second box started at r0 - H*W of image n0+1: both boxes
//     zero-fill what lies outside their image, and a thread picks, per 4-pixel
//     group, the box of the group's image — groups never straddle, H*W % 4 == 0);
//   * completion = the stage's full mbarrier (transaction bytes);
//   * release = a named barrier per stage: the warps arrive without waiting,
//     the issuing warp syncs on it before refilling the stage — the only wait
//     left is the issuer waiting for the slowest warp to finish the chunk it is
//     about to overwrite, ST-1 chunks behind.
// All 8 warps compute (no producer warp: 4 warps per sub-partition of 128
// registers fill the register file, so there is no room for one).
//
//   thread = 8 output channels {mgi + 4k} x 8 pixels {4pgi..+3, 32+4pgi..+3}
//            (lane = 8*mgi + pgi); per input channel 8 scalar filter loads (4
//            distinct words per warp, one wavefront each) + 2 LDS.128 for 32
//            FFMA2 — the 8x8 tile's 1.0 wavefront per FMA-pipe cycle.
//   warp   = 32 channels x 64 pixels; CTA = WM x WP warps.
#pragma once

#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace b2c {

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int x0, int x1, int x2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x0), "r"(x1), "r"(x2), "r"(bar)
      : "memory");
}

template <int WM, int WP, int BC, int ST>
struct Pw1x1TmaTile {
  static constexpr int BM = 32 * WM;
  static constexpr int BP = 64 * WP;
  static constexpr int NT = 32 * WM * WP;
  static constexpr int WROW = BC + 4;           // filter row pitch in shared memory (TMA box width)
  static constexpr int WFLOATS = BM * WROW;
  static constexpr int XFLOATS = BC * BP;       // one pixel box
  static constexpr int STAGE_FLOATS = WFLOATS + 2 * XFLOATS;
  static constexpr int SMEM_BYTES = 128 + 4 * ST * STAGE_FLOATS;
  static constexpr int MIN_BLOCKS = 2;
  static_assert(WFLOATS % 32 == 0 && XFLOATS % 32 == 0, "boxes must stay 128-byte aligned");
  static_assert(ST >= 2 && ST <= 15, "one named barrier per stage (ids 1..ST)");
};

template <int WM, int WP, int BC, int ST>
__global__ void __launch_bounds__(Pw1x1TmaTile<WM, WP, BC, ST>::NT, Pw1x1TmaTile<WM, WP, BC, ST>::MIN_BLOCKS)
    conv1x1_tma_kernel(const __grid_constant__ KParams p, const __grid_constant__ CUtensorMap wmap,
                       const __grid_constant__ CUtensorMap xmap) {
  using T = Pw1x1TmaTile<WM, WP, BC, ST>;
  constexpr int BM = T::BM, BP = T::BP, NT = T::NT, WROW = T::WROW;
  constexpr int WFLOATS = T::WFLOATS, XFLOATS = T::XFLOATS, STAGE_FLOATS = T::STAGE_FLOATS;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);
  float *stages = reinterpret_cast<float *>(smem_raw + 128);

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int mgi = lane >> 3, pgi = lane & 7;
  const int tile = blockIdx.x;
  const int mt = tile % p.mtiles;
  const long long pt = tile / p.mtiles;
  const int m0 = mt * BM;
  const long long q0 = pt * BP;
  const int split = blockIdx.y;
  const int hw = p.HoWo;
  const int n0 = (int)(q0 / hw);
  const int r0 = (int)(q0 - (long long)n0 * hw);
  const bool two = r0 + BP > hw && n0 + 1 < p.N;   // the tile runs into image n0+1
  const int chunk_begin = split * p.chunks_per_split;
  const int chunk_end = min(p.nchunks, chunk_begin + p.chunks_per_split);
  const int nch = chunk_end - chunk_begin;
  const uint32_t tx_bytes = 4u * (WFLOATS + (two ? 2 : 1) * XFLOATS);

  if (tid == 0) {
    for (int s = 0; s < ST; s++) mbar_init(smem_u32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

  auto issue = [&](int i) {  // chunk chunk_begin + i into stage i % ST (thread 0)
    const int s = i % ST;
    const uint32_t bar = smem_u32(&full[s]);
    float *st = stages + s * STAGE_FLOATS;
    const int c0 = (chunk_begin + i) * BC;
    mbar_expect_tx_only(bar, tx_bytes);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    tma_load_2d(smem_u32(st), &wmap, c0, m0, bar);
    tma_load_3d(smem_u32(st + WFLOATS), &xmap, r0, c0, n0, bar);
    if (two) tma_load_3d(smem_u32(st + WFLOATS + XFLOATS), &xmap, r0 - hw, c0, n0 + 1, bar);
  };
  if (tid == 0)
    for (int i = 0; i < ST - 1 && i < nch; i++) issue(i);

  // this thread's two 4-pixel groups and the box each one lives in
  const int pa = wp * 64 + 4 * pgi;
  const int pb = pa + 32;
  const int boxa = (r0 + pa >= hw) ? XFLOATS : 0;
  const int boxb = (r0 + pb >= hw) ? XFLOATS : 0;

  float2 acc[4][8];  // channel pairs (mgi + 8k, mgi + 8k + 4) x 8 pixels
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.0f, 0.0f);

  for (int i = 0; i < nch; i++) {
    const int s = i % ST;
    if (wid == 0 && i + ST - 1 < nch) {
      // refill the stage of chunk i-1 with chunk i+ST-1 once every warp is done with it
      if (i >= 1) named_bar_sync(1 + (i - 1) % ST, NT);
      if (lane == 0) issue(i + ST - 1);
      __syncwarp();
    }
    mbar_wait(smem_u32(&full[s]), (i / ST) & 1, p.spin_limit);
    const float *st = stages + s * STAGE_FLOATS;
    const float *wc = st + (wm * 32 + mgi) * WROW;
    const float *xa = st + WFLOATS + boxa + pa;
    const float *xb = st + WFLOATS + boxb + pb;
    const int cvalid = min(BC, p.C - (chunk_begin + i) * BC);
    // one channel per trip: unrolling merges (c, c+1) of a filter row into
    // LDS.64 and then rebuilds the channel pairs with register moves on the
    // FMA pipe (ncu: ~10 % of the loop)
#pragma unroll 1
    for (int c = 0; c < cvalid; c++) {
      const float4 va = *reinterpret_cast<const float4 *>(xa + c * BP);
      const float4 vb = *reinterpret_cast<const float4 *>(xb + c * BP);
      const float xv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
      float2 w2[4];
#pragma unroll
      for (int k = 0; k < 4; k++) w2[k] = make_float2(wc[(8 * k) * WROW + c], wc[(8 * k + 4) * WROW + c]);
#pragma unroll
      for (int k = 0; k < 4; k++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[k][j] = __ffma2_rn(w2[k], make_float2(xv[j], xv[j]), acc[k][j]);
    }
    // the stage of chunk i is refilled with chunk i+ST (by warp 0, which syncs instead)
    if (wid != 0 && i + ST < nch) named_bar_arrive(1 + s, NT);
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- epilogue: float4 stores (H*W % 4 == 0: a group shares one image) ----------
  float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : p.y;
#pragma unroll
  for (int g = 0; g < 2; g++) {
    const long long q = q0 + (g ? pb : pa);
    if (q >= p.Q) continue;
    const long long n = q / hw;
    const long long base = n * p.M * hw + (q - n * hw);
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int m = m0 + wm * 32 + mgi + 8 * k + 4 * h;
        if (m >= p.M) continue;
        const float2 *a = acc[k] + 4 * g;
        const float4 v = h ? make_float4(a[0].y, a[1].y, a[2].y, a[3].y) : make_float4(a[0].x, a[1].x, a[2].x, a[3].x);
        *reinterpret_cast<float4 *>(dst + base + (long long)m * hw) = v;
      }
  }
}

}  // namespace b2c
