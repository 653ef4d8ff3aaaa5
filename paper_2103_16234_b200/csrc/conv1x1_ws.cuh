// Persistent warp-specialised pointwise (1x1, any stride, no padding) fp32
// convolution — the producer/consumer pipeline of conv_row_ws_kernel
// (conv_row.cuh) over the flattened pixel tiles of the pointwise families,
// with a persistent grid so that short-K layers (ResNet C = 64..256: 4-16
// channel chunks per tile) never pay a pipeline fill per tile.
//
// Same arithmetic contract as conv_direct_kernel / conv1x1_vec_kernel: per
// output, channels ascending (one FFMA each) within each split range, split
// ranges summed in ascending order by stage2_sum_kernel — bitwise identical to
// them for equal splits.
//
//   CTA    = 2 consumer warpgroups (8 warps) + 1 producer warpgroup, one CTA
//            per SM walking work items (split, pixel tile, channel tile)
//            blockIdx.x, +gridDim.x, ...  The stage ring runs continuously
//            across items: the producers fill the next item's first stages
//            while the consumers finish and store the current one.
//   thread = 16 output channels (all lanes of a warp: filter loads are
//            broadcasts) x 8 output pixels as two groups of 4 consecutive
//            pixels (LDS.128 each; lane l takes pixels 4l.. and 128+4l..);
//            FFMA2 pairs two filter values (loaded straight into an even/odd
//            register pair) against one pixel.
//   warp   = 16 channels x 256 pixels; consumers WM x WP (BM = 16*WM, BP =
//            256*WP).  Per input channel a consumer issues 16 scalar broadcast
//            loads + 2 LDS.128 (24 wavefronts) for 64 FFMA2 (128 FMA-pipe
//            cycles): 75 % of the shared-memory crossbar at the FFMA2 peak.
//   producers = 128 threads, 4-pixel groups G = thread + 128k: per stage the
//            filter tile [BM][BC] by one 2-D TMA load from the caller's [M][C]
//            filters (4-byte cp.async when C*4 is not 16-byte aligned) and the
//            pixel tile [BC][BP] by 16-byte cp.async (H*W % 4 == 0, stride 1)
//            or 4-byte cp.async (7x7 planes, strided projection shortcuts),
//            each producer thread hands the completion of its copies of a stage
//            to the stage's full mbarrier (cp.async.mbarrier.arrive.noinc);
//            consumers release a stage for refill through a
//            named barrier (arrive without waiting; the producers sync on it).  No CTA-wide barrier after setup.
//   registers = 12 warps launch at 168 (the whole file); the producer
//            warpgroup drops to 40 (setmaxnreg.dec) and the consumers rise to
//            232 (setmaxnreg.inc) for their 128 accumulators.
//   Pixels past the last output and filter rows past M are never stored, so
//   their shared-memory slots are not cleared (garbage only reaches outputs
//   that are discarded).
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
  static constexpr int NPT = 128;                 // producer threads: one warpgroup
  static constexpr int NT = 32 * NCW + NPT;
  static constexpr int WFLOATS = BM * BC;         // filter tile [BM][BC]
  static constexpr int XFLOATS = BC * BP;         // pixel tile [BC][BP]
  static constexpr int STAGE_FLOATS = WFLOATS + XFLOATS;
  static constexpr int SMEM_BYTES = 128 + 4 * ST * STAGE_FLOATS;
  static constexpr int MIN_BLOCKS = 1;
  static constexpr int PRODUCER_REGS = 40, CONSUMER_REGS = 232;
  static constexpr int GPT = (BP / 4 + NPT - 1) / NPT;  // 4-pixel groups per producer thread
  static_assert(NCW == 8, "two consumer warpgroups");
  static_assert(ST >= 1 && ST <= 15, "one named barrier per stage (ids 1..ST)");
  static_assert(WFLOATS % 32 == 0, "stages must stay 128-byte aligned");
};

template <int WM, int WP, int BC, int ST>
__global__ void __launch_bounds__(Pw1x1WsTile<WM, WP, BC, ST>::NT, 1)
    conv1x1_ws_kernel(const __grid_constant__ KParams p, const __grid_constant__ CUtensorMap wmap) {
  using T = Pw1x1WsTile<WM, WP, BC, ST>;
  constexpr int RM = T::RM, BM = T::BM, BP = T::BP, NCW = T::NCW;
  constexpr int WFLOATS = T::WFLOATS, STAGE_FLOATS = T::STAGE_FLOATS;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);  // full[ST]
  float *stages = reinterpret_cast<float *>(smem_raw + 128);

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const long long tiles = (long long)p.mtiles * p.ptiles;
  const long long items = tiles * p.splits;
  if (tid == 0) {
    for (int s = 0; s < ST; s++) {
      mbar_init(smem_u32(&bars[s]), T::NPT);     // producer threads' arrivals (+ TMA bytes)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

  // chunks this CTA walks over all its items: a stage is released for refill
  // (named barrier 1 + s) only if a later chunk reuses it
  long long total = 0;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const int sp = (int)(it / tiles);
    total += min(p.nchunks, (sp + 1) * p.chunks_per_split) - sp * p.chunks_per_split;
  }
  auto decode = [&](long long it, int &m0, long long &q0, int &cb, int &ce, int &split) {
    split = (int)(it / tiles);
    const long long t = it - (long long)split * tiles;
    const long long pt = t / p.mtiles;
    m0 = (int)(t - pt * p.mtiles) * BM;
    q0 = pt * BP;
    cb = split * p.chunks_per_split;
    ce = min(p.nchunks, cb + p.chunks_per_split);
  };

  if (wid >= NCW) {
    // ---------------- producer warpgroup ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::PRODUCER_REGS));
    const int pt_id = tid - 32 * NCW;            // 0..127
    const int in_hw = p.H * p.W;
    const long long chw = (long long)p.C * in_hw;
    const bool tma = p.w_tma != 0;
    constexpr int GPT = T::GPT;
    long long gi = 0;                             // stage-ring position (chunks issued so far)
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
      int m0, cb, ce, split;
      long long q0;
      decode(it, m0, q0, cb, ce, split);
      // input offsets of this thread's pixel groups G = pt_id + NPT*k (4 pixels
      // each; -1: past the last output or past the tile)
      long long off[GPT][4];
      bool vec[GPT];
#pragma unroll
      for (int k = 0; k < GPT; k++) {
        const int G = pt_id + T::NPT * k;
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const long long q = q0 + 4 * G + e;
          off[k][e] = -1;
          if (G < BP / 4 && q < p.Q) {
            const long long n = q / p.HoWo;
            const int r = (int)(q - n * p.HoWo);
            const int oy = r / p.Wo;
            const int ox = r - oy * p.Wo;
            off[k][e] = n * chw + (long long)oy * p.S * p.W + (long long)ox * p.S;
          }
        }
        vec[k] = p.vec_ok && off[k][0] >= 0 && (off[k][0] & 3) == 0 && off[k][1] == off[k][0] + 1 &&
                 off[k][2] == off[k][0] + 2 && off[k][3] == off[k][0] + 3;
      }
      for (int chunk = cb; chunk < ce; chunk++, gi++) {
        const int s = (int)(gi % ST);
        const long long kk = gi / ST;
        const uint32_t full = smem_u32(&bars[s]);
        if (kk > 0) named_bar_sync(1 + s, T::NT);  // every consumer is done with the stage's previous chunk
        float *wst = stages + s * STAGE_FLOATS;
        const int c0 = chunk * BC;
        const int cvalid = min(BC, p.C - c0);
        if (tma) {
          if (pt_id == 0) {
            mbar_expect_tx_only(full, WFLOATS * 4);
            tma_load_2d(smem_u32(wst), &wmap, c0, m0, full);
          }
        } else {
          const float *wsrc = p.w + (long long)m0 * p.C + c0;
          for (int e = pt_id; e < BM * BC; e += T::NPT) {
            const int m = e / BC, c = e - (e / BC) * BC;
            if (m0 + m < p.M && c < cvalid) cp_async4(wst + e, wsrc + (long long)m * p.C + c);
          }
        }
        const float *xsrc = p.x + (long long)c0 * in_hw;
#pragma unroll
        for (int k = 0; k < GPT; k++) {
          float *xst = wst + WFLOATS + 4 * (pt_id + T::NPT * k);
          if (vec[k]) {
#pragma unroll 4
            for (int c = 0; c < cvalid; c++) cp_async16(xst + c * BP, xsrc + off[k][0] + (long long)c * in_hw);
          } else {
#pragma unroll
            for (int e = 0; e < 4; e++)
              if (off[k][e] >= 0)
                for (int c = 0; c < cvalid; c++)
                  cp_async4(xst + c * BP + e, xsrc + off[k][e] + (long long)c * in_hw);
          }
        }
        cp_async_mbar_arrive_noinc(full);  // the arrive fires when this thread's copies have landed
      }
    }
    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // ---------------- consumer warpgroups ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(T::CONSUMER_REGS));
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int pa = wp * 256 + 4 * lane;  // pixel groups pa..pa+3 and pa+128..pa+131
  const int hw = p.HoWo;
  long long gi = 0;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    int m0, cb, ce, split;
    long long q0;
    decode(it, m0, q0, cb, ce, split);
    // acc[r][j]: output channels (2r, 2r+1) of this warp's 16, pixel j of this
    // thread's 8 (j < 4: group a, j >= 4: group b)
    float2 acc[RM / 2][8];
#pragma unroll
    for (int i = 0; i < RM / 2; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.0f, 0.0f);
    for (int chunk = cb; chunk < ce; chunk++, gi++) {
      const int s = (int)(gi % ST);
      mbar_wait(smem_u32(&bars[s]), (int)((gi / ST) & 1), p.spin_limit);
      const float *wst = stages + s * STAGE_FLOATS;
      const float *wc = wst + (wm * RM) * BC;
      const float *xc = wst + WFLOATS + pa;
      const int cvalid = min(BC, p.C - chunk * BC);
      // one channel per trip: unrolling merges (c, c+1) of a filter row into
      // LDS.64 and then needs register moves (on the FMA pipe) to form pairs;
      // explicitly prefetching channel c+1's operands measured slower
      // (profiles/ab/r2_pointwise_ws_ab.txt)
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
      if (gi + ST < total) named_bar_arrive(1 + s, T::NT);  // release the stage for refill
    }

    // ---- epilogue of this item (the producers are already filling the next) ----
    float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : p.y;
#pragma unroll
    for (int g = 0; g < 2; g++) {
      const long long qg = q0 + pa + 128 * g;
      if (qg >= p.Q) continue;
      if (p.vec_out) {  // Ho*Wo % 4 == 0: the 4 pixels share an image, 16-byte aligned
        const long long n = qg / hw;
        const long long base = n * p.M * hw + (qg - n * hw);
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
          const long long n = q / hw;
          const long long base = n * p.M * hw + (q - n * hw);
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
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace b2c
