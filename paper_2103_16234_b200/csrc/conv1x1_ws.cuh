// Warp-specialised pointwise (1x1, any stride, no padding) fp32 convolution —
// the producer/consumer pipeline of conv_row_ws_kernel (conv_row.cuh) applied
// to the flattened pixel tiles of the pointwise families.
//
// Same arithmetic contract as conv_direct_kernel / conv1x1_vec_kernel: per
// output, channels ascending (one FFMA each) within each split range, split
// ranges summed in ascending order by stage2_sum_kernel — bitwise identical to
// them for equal splits.
//
//   thread = 16 output channels (all lanes of a warp: filter loads are
//            broadcasts) x 8 output pixels as two groups of 4 consecutive
//            pixels (LDS.128 each; lane l takes pixels 4l.. and 128+4l..)
//   warp   = 16 channels x 256 pixels; CTA = WM x WP = 8 consumer warps (BM
//            = 16*WM channels x BP = 256*WP pixels) + a producer warpgroup
//   per input channel a consumer issues 16 scalar broadcast loads + 2 LDS.128
//   (24 wavefronts) for 64 FFMA2 (128 FMA-pipe cycles): 75 % of the
//   shared-memory crossbar at the FFMA2 peak, the FMA pipe binds.
//   producer = per ST-deep stage: the filter tile [BM][BC] by one 2-D TMA load
//            from the caller's [M][C] filters (4-byte cp.async when C*4 is not
//            16-byte aligned), the pixel tile [BC][BP] by 16-byte cp.async for
//            aligned runs of 4 (H*W % 4 == 0, stride 1) and 4-byte cp.async
//            otherwise (7x7 planes, strided projection shortcuts), completion
//            handed to the stage's full mbarrier; consumers release stages
//            through the empty mbarrier.  No CTA-wide barrier in the loop.
//   epilogue = float4 stores of 4 consecutive pixels per channel when
//            Ho*Wo % 4 == 0 (a warp writes 512 contiguous bytes per channel).
#pragma once

#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace b2c {

template <int WM, int WP, int BC, int ST>
struct Pw1x1WsTile {
  static constexpr int RM = 16;
  static constexpr int BM = RM * WM;
  static constexpr int BP = 256 * WP;
  static constexpr int NCW = WM * WP;             // consumer warps: two warpgroups
  static constexpr int NT = 32 * (NCW + 4);       // + one producer warpgroup (one working warp)
  static constexpr int WFLOATS = BM * BC;   // filter tile [BM][BC]
  static constexpr int XFLOATS = BC * BP;   // pixel tile [BC][BP]
  static constexpr int STAGE_FLOATS = WFLOATS + XFLOATS;
  static constexpr int TABLE_BYTES = (4 * (BP + BP / 4) + 127) & ~127;
  static constexpr int SMEM_BYTES = 128 + TABLE_BYTES + 4 * ST * STAGE_FLOATS;
  // Registers: 128 accumulators need ~200 per consumer thread, and each SM
  // sub-partition holds 16K registers for its warps.  The CTA launches 12 warps
  // at 168 registers (the whole register file), then the producer warpgroup
  // gives registers back (setmaxnreg.dec to 40) and the consumers take them
  // (setmaxnreg.inc to 232): per sub-partition 2 consumer + 1 producer warp.
  static constexpr int MIN_BLOCKS = 1;
  static constexpr int PRODUCER_REGS = 40, CONSUMER_REGS = 232;
  static_assert(NCW == 8, "two consumer warpgroups");
  static_assert(WFLOATS % 32 == 0, "stages must stay 128-byte aligned");
};

template <int WM, int WP, int BC, int ST>
__global__ void __launch_bounds__(Pw1x1WsTile<WM, WP, BC, ST>::NT, 1)
    conv1x1_ws_kernel(const __grid_constant__ KParams p, const __grid_constant__ CUtensorMap wmap) {
  using T = Pw1x1WsTile<WM, WP, BC, ST>;
  constexpr int RM = T::RM, BM = T::BM, BP = T::BP, NCW = T::NCW, NT = T::NT;
  constexpr int WFLOATS = T::WFLOATS, XFLOATS = T::XFLOATS, STAGE_FLOATS = T::STAGE_FLOATS;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);  // full[ST] | empty[ST]
  int *goff = reinterpret_cast<int *>(smem_raw + 128);      // per tile pixel: input offset at channel 0
  int *gtab = goff + BP;                                     // per 4-pixel group: aligned run offset or -1
  float *stages = reinterpret_cast<float *>(smem_raw + 128 + T::TABLE_BYTES);

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int tile = blockIdx.x;
  const int mt = tile % p.mtiles;
  const int pt = tile / p.mtiles;
  const int m0 = mt * BM;
  const long long q0 = (long long)pt * BP;
  const int split = blockIdx.y;
  const int n0 = (int)(q0 / p.HoWo);
  const int in_hw = p.H * p.W;
  const long long chw = (long long)p.C * in_hw;

  if (tid == 0) {
    for (int s = 0; s < ST; s++) {
      mbar_init(smem_u32(&bars[s]), 32);
      mbar_init(smem_u32(&bars[ST + s]), NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gather table: tile pixel -> element offset (relative to image n0, channel 0);
  // -1 past the last pixel (staged as +0.0, never stored)
  for (int i = tid; i < BP; i += NT) {
    const long long q = q0 + i;
    int g = -1;
    if (q < p.Q) {
      const int n = (int)(q / p.HoWo);
      const int r = (int)(q - (long long)n * p.HoWo);
      const int oy = r / p.Wo;
      const int ox = r - oy * p.Wo;
      g = (int)((long long)(n - n0) * chw + (long long)oy * p.S * p.W + ox * p.S);
    }
    goff[i] = g;
  }
  for (int s = 0; s < ST; s++) {
    float4 *xz = reinterpret_cast<float4 *>(stages + s * STAGE_FLOATS + WFLOATS);
    for (int i = tid; i < XFLOATS / 4; i += NT) xz[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  for (int G = tid; G < BP / 4; G += NT) {
    const int g0 = goff[4 * G], g1 = goff[4 * G + 1], g2 = goff[4 * G + 2], g3 = goff[4 * G + 3];
    gtab[G] = (p.vec_ok && g0 >= 0 && (g0 & 3) == 0 && g1 == g0 + 1 && g2 == g0 + 2 && g3 == g0 + 3) ? g0 : -1;
  }
  __syncthreads();  // barriers initialised, tables and zeros visible

  const int chunk_begin = split * p.chunks_per_split;
  const int chunk_end = min(p.nchunks, chunk_begin + p.chunks_per_split);
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

  if (wid >= NCW) {
    // ---------------- producer warpgroup: warp NCW works, the others leave ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::PRODUCER_REGS));
    if (wid != NCW) return;
    const float *xtile = p.x + (long long)n0 * chw;
    const bool tma = p.w_tma != 0;
    for (int chunk = chunk_begin; chunk < chunk_end; chunk++) {
      const int i = chunk - chunk_begin;
      const int s = i % ST;
      const int k = i / ST;
      const uint32_t full = smem_u32(&bars[s]);
      if (k > 0) mbar_wait(smem_u32(&bars[ST + s]), (k - 1) & 1, p.spin_limit);
      float *wst = stages + s * STAGE_FLOATS;
      float *xst = wst + WFLOATS;
      const int c0 = chunk * BC;
      const int cvalid = min(BC, p.C - c0);
      if (tma) {
        if (lane == 0) {
          mbar_expect_tx_only(full, WFLOATS * 4);
          tma_load_2d(smem_u32(wst), &wmap, c0, m0, full);
        }
      } else {
        const float *wsrc = p.w + (long long)m0 * p.C + c0;
        for (int e = lane; e < BM * BC; e += 32) {
          const int m = e / BC, c = e - (e / BC) * BC;
          if (m0 + m < p.M && c < cvalid) cp_async4(wst + e, wsrc + (long long)m * p.C + c);
        }
      }
      const float *xsrc = xtile + (long long)c0 * in_hw;
      for (int G = lane; G < BP / 4; G += 32) {
        const int t = gtab[G];
        float *dst = xst + 4 * G;
        if (t >= 0) {
          const float *src = xsrc + t;
#pragma unroll 4
          for (int c = 0; c < cvalid; c++) cp_async16(dst + c * BP, src + (long long)c * in_hw);
        } else {
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int g = goff[4 * G + e];
            if (g < 0) continue;
            const float *src = xsrc + g;
            for (int c = 0; c < cvalid; c++) cp_async4(dst + c * BP + e, src + (long long)c * in_hw);
          }
        }
      }
      cp_async_mbar_arrive_noinc(full);
    }
    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // ---------------- consumer warps ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(T::CONSUMER_REGS));
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int pa = wp * 256 + 4 * lane;  // pixel groups pa..pa+3 and pa+128..pa+131
  // acc[r][j]: output channels (2r, 2r+1) of this warp's 16, pixel j of this
  // thread's 8 (j < 4: group a, j >= 4: group b).  FFMA2 pairs two filter
  // values (two scalar loads straight into an even/odd register pair) against
  // one pixel; the pair is the reused operand across the 8 pixels.
  float2 acc[RM / 2][8];
#pragma unroll
  for (int i = 0; i < RM / 2; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.0f, 0.0f);

  for (int chunk = chunk_begin; chunk < chunk_end; chunk++) {
    const int i = chunk - chunk_begin;
    const int s = i % ST;
    mbar_wait(smem_u32(&bars[s]), (i / ST) & 1, p.spin_limit);
    const float *wst = stages + s * STAGE_FLOATS;
    const float *wc = wst + (wm * RM) * BC;
    const float *xc = wst + WFLOATS + pa;
    const int cvalid = min(BC, p.C - chunk * BC);
    // one channel per trip: unrolling pairs (c, c+1) of a filter row into
    // LDS.64 and then needs register moves (on the FMA pipe) to form pairs
#pragma unroll 1
    for (int c = 0; c < cvalid; c++) {
      const float4 xa = *reinterpret_cast<const float4 *>(xc + c * BP);
      const float4 xb = *reinterpret_cast<const float4 *>(xc + c * BP + 128);
      const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
      float2 w2[RM / 2];
#pragma unroll
      for (int r = 0; r < RM / 2; r++) w2[r] = make_float2(wc[(2 * r) * BC + c], wc[(2 * r + 1) * BC + c]);
#pragma unroll
      for (int r = 0; r < RM / 2; r++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[r][j] = __ffma2_rn(w2[r], make_float2(xv[j], xv[j]), acc[r][j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars[ST + s]));
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- epilogue ------------------------------------------------------------------
  float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : p.y;
  const int hw = p.HoWo;
#pragma unroll
  for (int g = 0; g < 2; g++) {
    const long long qg = q0 + pa + 128 * g;
    if (qg >= p.Q) continue;
    if (p.vec_out) {  // Ho*Wo % 4 == 0: the 4 pixels share an image, 16-byte aligned
      const int n = (int)(qg / hw);
      const long long base = (long long)n * p.M * hw + (qg - (long long)n * hw);
#pragma unroll
      for (int r = 0; r < RM; r++) {
        const int m = m0 + wm * RM + r;
        if (m >= p.M) break;
        const float2 *a = acc[r >> 1];
        const float4 v = (r & 1) ? make_float4(a[4 * g].y, a[4 * g + 1].y, a[4 * g + 2].y, a[4 * g + 3].y)
                                 : make_float4(a[4 * g].x, a[4 * g + 1].x, a[4 * g + 2].x, a[4 * g + 3].x);
        *reinterpret_cast<float4 *>(dst + base + (long long)m * hw) = v;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const long long q = qg + e;
        if (q >= p.Q) break;
        const int n = (int)(q / hw);
        const long long base = (long long)n * p.M * hw + (q - (long long)n * hw);
#pragma unroll
        for (int r = 0; r < RM; r++) {
          const int m = m0 + wm * RM + r;
          if (m >= p.M) break;
          const float2 v = acc[r >> 1][4 * g + e];
          dst[base + (long long)m * hw] = (r & 1) ? v.y : v.x;
        }
      }
    }
  }
}

}  // namespace b2c
