// Row-segment direct convolution (fused FFMA2 engine, any filter size and
// stride) — the 3x3 / 5x5 / 7x7 families' shared-memory-lean mapping.
//
// Same arithmetic contract as conv_direct_kernel (conv_kernel.cuh): per output
// the order is "channels ascending, filter taps row-major inside each
// channel" within each split range, one FFMA per tap, so for equal splits the
// two kernels are bitwise identical.  Only the register/shared-memory mapping
// differs.
//
// conv_direct_kernel gives a thread 16 channels x 4 output pixels strided
// across the tile: per (channel, tap) it issues 4 LDS.128 of filters (a warp
// broadcast still costs 4 wavefronts) and 4 scalar pixel loads for 32 FFMA2,
// i.e. 20 wavefronts per 64 FMA-pipe cycles of a warp — the shared-memory
// crossbar, not the FMA pipe, bounds it at 80 % of the FFMA2 peak (measured
// 67 % FMA-pipe active, ncu, profiles/r2).
//
// Here a thread owns 16 output channels x RX consecutive outputs of ONE
// output row (a "segment").  Per (channel, filter row) it loads the
// (RX-1)*S+WF input columns under the segment once and reuses them for all WF
// taps of that filter row (a register sliding window), so per (channel,
// filter row) it issues WF x 4 LDS.128 of filters plus (RX-1)*S+WF scalar
// loads against WF*8*RX FFMA2.  3x3, stride 1, RX = 7: 57 wavefronts per 336
// FMA-pipe cycles (68 % of the crossbar at the FFMA2 peak); stride 2: 63.  The
// FMA pipe becomes the bound.
//
//   warp   = 16 channels (all lanes; filter loads are broadcasts) x 32
//            segments (consecutive segment ids: along a row, then down rows
//            and across images — virtual rows, as in conv_direct_kernel)
//   CTA    = WM channel groups x WP segment groups of warps
//            (BM = 16*WM channels x 32*WP segments)
//   RX = 7 divides every output width of the BASELINE layers (224, 112, 56,
//   28, 14, 7); other widths compute the tail of their last segment and drop
//   it at the store.
//   staging = the halo band of conv_direct_kernel (build_halo_tables /
//   stage_halo_chunk: 16-byte cp.async for aligned runs, virtual zero
//   padding) with a row stride the planner picks so that the 32 segment
//   origins of a warp fall on distinct banks; filters transposed [c][tap][m];
//   two-stage cp.async pipeline over BC-channel chunks.
#pragma once

#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace b2c {

template <int HF, int WF, int S, int RX, int WM, int WP, int BC, int MINB>
struct RowTile {
  static constexpr int RM = 16;
  static constexpr int BM = RM * WM;
  static constexpr int SEG = 32 * WP;            // segments per CTA
  static constexpr int NT = 32 * WM * WP;
  static constexpr int WS = BM + 4;              // filter row stride (floats)
  static constexpr int PXN = (RX - 1) * S + WF;  // input columns under one segment and filter row
  static constexpr int MIN_BLOCKS = MINB;
};

template <int HF, int WF, int S, int RX, int WM, int WP, int BC, int MINB>
__global__ void __launch_bounds__(RowTile<HF, WF, S, RX, WM, WP, BC, MINB>::NT, MINB)
    conv_row_kernel(const KParams p) {
  using T = RowTile<HF, WF, S, RX, WM, WP, BC, MINB>;
  constexpr int RM = T::RM, BM = T::BM, SEG = T::SEG, NT = T::NT, WS = T::WS, PXN = T::PXN;
  constexpr int TAPS = HF * WF;

  extern __shared__ __align__(16) float smem[];
  int *goff = reinterpret_cast<int *>(smem);
  int *gtab = goff + p.XCS;
  const int ngroups = p.XCS >> 2;
  const int xfloats = BC * p.XCS;
  const int stage_floats = xfloats + BC * TAPS * WS;
  float *stage0 = smem + p.XCS + ((ngroups + 3) & ~3);

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int tile = blockIdx.x;
  const int mt = tile % p.mtiles;
  const int pt = tile / p.mtiles;
  const int m0 = mt * BM;
  const int split = blockIdx.y;
  const int nb = p.nb;                          // segments per output row
  const int s0 = pt * SEG;                      // first segment of the tile (< 2^31: planner)

  // ---- tile origin in virtual-row space (exact hardware division, once) -------
  const int R0 = s0 / nb;                       // output row over (n, oy)
  const int n0 = R0 / p.Ho;
  const int oy0 = R0 - n0 * p.Ho;
  const int vlo = n0 * p.Hp + oy0 * S;
  const long long chw = (long long)p.C * p.H * p.W;
  const int hw = p.H * p.W;
  const int shift = (((oy0 * S - p.PH) * p.W - p.PW) % 4 + 4) % 4;
  build_halo_tables<NT>(p, goff, gtab, vlo, n0, shift, 0, chw);

  // ---- this thread's segment ---------------------------------------------------
  const int sraw = s0 + wp * 32 + lane;
  const bool seg_ok = sraw < p.segs;
  const int sg = seg_ok ? sraw : p.segs - 1;
  const int R = sg / nb;
  const int b = sg - R * nb;
  const int n = R / p.Ho;
  const int oy = R - n * p.Ho;
  const int pix_base = shift + ((n - n0) * p.Hp + (oy - oy0) * S) * p.RS + b * RX * S;
  __syncthreads();  // tables visible

  const float *xtile = p.x + (long long)n0 * chw;
  auto load_chunk = [&](int chunk, float *stage) {
    const int c0 = chunk * BC;
    const int cvalid = min(BC, p.C - c0);
    stage_halo_chunk<BC>(p, goff, gtab, stage, xtile + (long long)c0 * hw, cvalid, hw, threadIdx.x, NT);
    stage_filter_chunk<NT, BM>(p, stage + xfloats, p.w + ((long long)m0 * p.C + c0) * TAPS, BC * TAPS, TAPS,
                               cvalid * TAPS, true, m0);
  };

  float2 acc[RM / 2][RX];  // channel pairs (2i, 2i+1) x RX outputs
#pragma unroll
  for (int i = 0; i < RM / 2; i++)
#pragma unroll
    for (int j = 0; j < RX; j++) acc[i][j] = make_float2(0.0f, 0.0f);

  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int chunk_begin = split * p.chunks_per_split;
  const int chunk_end = min(p.nchunks, chunk_begin + p.chunks_per_split);
  if (chunk_begin < chunk_end) {
    load_chunk(chunk_begin, stage0);
    cp_async_commit();
  }
  for (int chunk = chunk_begin; chunk < chunk_end; chunk++) {
    const int buf = (chunk - chunk_begin) & 1;
    const float *cur = stage0 + buf * stage_floats;
    if (chunk + 1 < chunk_end) {
      load_chunk(chunk + 1, stage0 + (buf ^ 1) * stage_floats);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    const int cvalid = min(BC, p.C - chunk * BC);
    const float *xc = cur + pix_base;
    const float *wc = cur + xfloats + wm * RM;
    constexpr int YU = HF <= 3 ? HF : 1;  // 3x3: whole channel step unrolled (next row's loads overlap)
#pragma unroll 1
    for (int c = 0; c < cvalid; c++) {
#pragma unroll YU
      for (int yy = 0; yy < HF; yy++) {
        const float *xr = xc + yy * p.RS;
        float px[PXN];
#pragma unroll
        for (int k = 0; k < PXN; k++) px[k] = xr[k];
#pragma unroll
        for (int xx = 0; xx < WF; xx++) {
          const float *wt = wc + (yy * WF + xx) * WS;
          float2 w2[RM / 2];
#pragma unroll
          for (int i = 0; i < RM / 4; i++) {
            const float4 v = *reinterpret_cast<const float4 *>(wt + 4 * i);
            w2[2 * i] = make_float2(v.x, v.y);
            w2[2 * i + 1] = make_float2(v.z, v.w);
          }
#pragma unroll
          for (int i = 0; i < RM / 2; i++)
#pragma unroll
            for (int j = 0; j < RX; j++) {
              const float xv = px[j * S + xx];
              acc[i][j] = __ffma2_rn(w2[i], make_float2(xv, xv), acc[i][j]);
            }
        }
      }
      xc += p.XCS;
      wc += TAPS * WS;
    }
    __syncthreads();
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- epilogue: this segment's RX outputs of 16 channels ----------------------
  // splits == 1: fully overwrite y; else partial plane `split` of the workspace
  // (y layout), summed in ascending order by stage2_sum_kernel.
  if (!seg_ok) return;
  float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : p.y;
  const long long pix0 = (long long)n * p.M * p.HoWo + (long long)oy * p.Wo + b * RX;
  const int jmax = min(RX, p.Wo - b * RX);
#pragma unroll
  for (int i = 0; i < RM; i++) {
    const int m = m0 + wm * RM + i;
    if (m >= p.M) break;
    float *row = dst + pix0 + (long long)m * p.HoWo;
#pragma unroll
    for (int j = 0; j < RX; j++)
      if (j < jmax) row[j] = (i & 1) ? acc[i >> 1][j].y : acc[i >> 1][j].x;
  }
}

// ---------------------------------------------------------------------------------
// Warp-specialised row-segment kernel (kind 4).  Same mapping and arithmetic
// order as conv_row_kernel (bitwise identical for equal splits), but the CTA
// never stops at a CTA-wide barrier inside the channel loop: WM*WP consumer
// warps only compute, one producer warp fills an ST-deep ring of stages;
// per stage a full mbarrier (producer -> consumers: every producer lane's
// cp.async completion plus the TMA bytes) and a named barrier the consumers
// arrive on without waiting (consumers -> producer, before refill) order
// them.  Per stage the producer moves
//   * the filter tile [BM][BC*taps] (row m = w[m0+m][c0..c0+BC)[taps], dense)
//     with ONE 2-D TMA load straight from the caller's [M][C][hf][wf] tensor
//     (C*hf*wf*4 bytes per row must be 16-byte aligned; otherwise 4-byte
//     cp.async per element), out-of-range rows/columns zero-filled;
//   * the BC-channel halo band with 16-byte / 4-byte cp.async, whose
//     completion it hands to the stage's full barrier
//     (cp.async.mbarrier.arrive.noinc).
// Padding is written as +0.0 once per tile (it sits at the same positions in
// every channel and stage), so the producer never stores to shared memory.
// Consumers read the 16 filters of a (channel, tap) as 16 broadcast scalar
// loads (one wavefront each — the same crossbar cost as 4 LDS.128).
// NP = producer warps: 2 for stride-2 bands staged by 4-byte copies (4x the
// cp.async instructions of a 16-byte-staged band), where one producer warp
// sharing its sub-partition with FFMA2-bound consumers starves them
template <int HF, int WF, int S, int RX, int WM, int WP, int BC, int ST, int NP = 1>
struct RowWsTile {
  static constexpr int RM = 16;
  static constexpr int BM = RM * WM;
  static constexpr int SEG = 32 * WP;
  static constexpr int NCW = WM * WP;             // consumer warps
  static constexpr int NT = 32 * (NCW + NP);      // + the producer warps
  static constexpr int TAPS = HF * WF;
  static constexpr int WROW = BC * TAPS;          // filter tile row (floats)
  static constexpr int WFLOATS = BM * WROW;       // multiple of 32: stages stay 128-byte aligned
  static constexpr int PXN = (RX - 1) * S + WF;
  static constexpr int MIN_BLOCKS = NCW <= 4 ? 2 : 1;
  static_assert(WFLOATS % 32 == 0, "filter tile must keep 128-byte alignment");
  static_assert(ST >= 1 && ST <= 14, "one named barrier per stage (ids 1..ST; 15: cluster epilogue)");
};

template <int HF, int WF, int S, int RX, int WM, int WP, int BC, int ST, int NP = 1>
__global__ void __launch_bounds__(RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, NP>::NT,
                                  RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, NP>::MIN_BLOCKS)
    conv_row_ws_kernel(const __grid_constant__ KParams p, const __grid_constant__ CUtensorMap wmap) {
  using T = RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, NP>;
  constexpr int RM = T::RM, BM = T::BM, SEG = T::SEG, NCW = T::NCW, TAPS = T::TAPS, WROW = T::WROW;
  constexpr int WFLOATS = T::WFLOATS, PXN = T::PXN;

  // [full[ST] barriers: 128 B][goff: XCS ints][gtab][pad to 128 B][stages]
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
  int *goff = reinterpret_cast<int *>(smem_raw + 128);
  int *gtab = goff + p.XCS;
  const int xfloats = ((BC * p.XCS) + 31) & ~31;
  const int stage_floats = WFLOATS + xfloats;
  float *stages = reinterpret_cast<float *>(smem_raw + 128 + ((4 * (p.XCS + (p.XCS >> 2)) + 127) & ~127));

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int tile = blockIdx.x;
  const int mt = tile % p.mtiles;
  const int pt = tile / p.mtiles;
  const int m0 = mt * BM;
  const int split = blockIdx.y;
  const int nb = p.nb;
  const int s0 = pt * SEG;
  const int R0 = s0 / nb;
  const int n0 = R0 / p.Ho;
  const int oy0 = R0 - n0 * p.Ho;
  const int vlo = n0 * p.Hp + oy0 * S;
  const long long chw = (long long)p.C * p.H * p.W;
  const int hw = p.H * p.W;
  const int shift = (((oy0 * S - p.PH) * p.W - p.PW) % 4 + 4) % 4;

  if (tid == 0) {
    for (int s = 0; s < ST; s++) {
      mbar_init(smem_u32(&bars[s]), 32 * NP);   // producer threads' arrivals (+ TMA bytes)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  build_halo_tables<T::NT>(p, goff, gtab, vlo, n0, shift, 0, chw);
  // padding and unused band positions are +0.0 in every stage, once per tile
  for (int s = 0; s < ST; s++) {
    float4 *xz = reinterpret_cast<float4 *>(stages + s * stage_floats + WFLOATS);
    for (int i = tid; i < xfloats / 4; i += T::NT) xz[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();  // barriers initialised, tables and zeros visible

  const int chunk_begin = split * p.chunks_per_split;
  const int chunk_end = min(p.nchunks, chunk_begin + p.chunks_per_split);
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

  if (wid >= NCW) {
    // ---------------- producer warp(s) ----------------
    const int pt0 = (wid - NCW) * 32 + lane;  // producer thread index
    const float *xtile = p.x + (long long)n0 * chw;
    const bool tma = p.w_tma != 0;
    for (int chunk = chunk_begin; chunk < chunk_end; chunk++) {
      const int i = chunk - chunk_begin;
      const int s = i % ST;
      const int k = i / ST;
      const uint32_t full = smem_u32(&bars[s]);
      if (k > 0) named_bar_sync(1 + s, T::NT);  // every consumer is done with the stage's previous chunk
      float *wst = stages + s * stage_floats;
      const int c0 = chunk * BC;
      const int cvalid = min(BC, p.C - c0);
      if (p.w_tma == 2) {
        // the family's chunk is all C channels (BC == C): the tile's filter rows
        // are one contiguous block of the caller's tensor -> one bulk copy
        if (pt0 == 0) {
          const uint32_t bytes = 4u * (uint32_t)min(BM, p.M - m0) * WROW;
          mbar_expect_tx_only(full, bytes);
          bulk_copy_g2s(smem_u32(wst), p.w + (long long)m0 * WROW, bytes, full);
        }
      } else if (tma) {
        if (pt0 == 0) {
          mbar_expect_tx_only(full, WFLOATS * 4);
          tma_load_2d(smem_u32(wst), &wmap, c0 * TAPS, m0, full);
        }
      } else {
        const int ctv = cvalid * TAPS;
        const float *wsrc = p.w + (long long)m0 * p.C * TAPS + (long long)c0 * TAPS;
        for (int m = 0; m < BM && m0 + m < p.M; m++)
          for (int ct = pt0; ct < ctv; ct += 32 * NP)
            cp_async4(wst + m * WROW + ct, wsrc + (long long)m * p.C * TAPS + ct);
      }
      stage_halo_chunk<BC, false>(p, goff, gtab, wst + WFLOATS, xtile + (long long)c0 * hw, cvalid, hw, pt0, 32 * NP);
      cp_async_mbar_arrive_noinc(full);  // the arrive fires when this thread's copies have landed
    }
    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!p.cluster) return;
    // split-C through DSMEM: the producer warp takes part in the tile reduction
    // (its first cluster barrier orders it after the consumers' tile writes)
    cluster_reduce_tile<BM, SEG * RX, T::NT>(p, stages, m0, s0 * RX);
    return;
  }

  // ---------------- consumer warps ----------------
  const int wm = wid / WP, wp = wid - (wid / WP) * WP;
  const int sraw = s0 + wp * 32 + lane;
  const bool seg_ok = sraw < p.segs;
  const int sg = seg_ok ? sraw : p.segs - 1;
  const int R = sg / nb;
  const int b = sg - R * nb;
  const int n = R / p.Ho;
  const int oy = R - n * p.Ho;
  const int pix_base = shift + ((n - n0) * p.Hp + (oy - oy0) * S) * p.RS + b * RX * S;

  float2 acc[RM / 2][RX];
#pragma unroll
  for (int i = 0; i < RM / 2; i++)
#pragma unroll
    for (int j = 0; j < RX; j++) acc[i][j] = make_float2(0.0f, 0.0f);

  for (int chunk = chunk_begin; chunk < chunk_end; chunk++) {
    const int i = chunk - chunk_begin;
    const int s = i % ST;
    mbar_wait(smem_u32(&bars[s]), (i / ST) & 1, p.spin_limit);
    const float *wst = stages + s * stage_floats;
    const float *xc = wst + WFLOATS + pix_base;
    const float *wc = wst + (wm * RM) * WROW;
    const int cvalid = min(BC, p.C - chunk * BC);
    constexpr int YU = HF <= 3 ? HF : 1;
#pragma unroll 1
    for (int c = 0; c < cvalid; c++) {
#pragma unroll YU
      for (int yy = 0; yy < HF; yy++) {
        const float *xr = xc + yy * p.RS;
        float px[PXN];
#pragma unroll
        for (int q = 0; q < PXN; q++) px[q] = xr[q];
#pragma unroll
        for (int xx = 0; xx < WF; xx++) {
          const float *wt = wc + yy * WF + xx;
          float2 w2[RM / 2];
#pragma unroll
          for (int r = 0; r < RM / 2; r++) w2[r] = make_float2(wt[(2 * r) * WROW], wt[(2 * r + 1) * WROW]);
#pragma unroll
          for (int r = 0; r < RM / 2; r++)
#pragma unroll
            for (int j = 0; j < RX; j++) {
              const float xv = px[j * S + xx];
              acc[r][j] = __ffma2_rn(w2[r], make_float2(xv, xv), acc[r][j]);
            }
        }
      }
      xc += p.XCS;
      wc += TAPS;
    }
    if (chunk + ST < chunk_end) named_bar_arrive(1 + s, T::NT);  // release the stage for refill
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (p.cluster) {
    // split-C through DSMEM (reduce = 2; the planner allows it when RX divides
    // Wo, so the tile's segments are the contiguous output pixels
    // [s0*RX, (s0+SEG)*RX)): park the accumulators as a [BM][SEG*RX] tile in
    // this CTA's (drained) stage memory, then sum the splits' tiles in
    // ascending rank order — the order stage2_sum_kernel uses, bitwise equal
    // to partial planes
    float *tile = stages;
    const int col = (wp * 32 + lane) * RX;
    named_bar_sync(15, NCW * 32);  // every consumer is past its last stage read before the tile overlays them
#pragma unroll
    for (int r = 0; r < RM; r++)
#pragma unroll
      for (int j = 0; j < RX; j++)
        tile[(wm * RM + r) * (SEG * RX) + col + j] = (r & 1) ? acc[r >> 1][j].y : acc[r >> 1][j].x;
    cluster_reduce_tile<BM, SEG * RX, T::NT>(p, tile, m0, s0 * RX);
    return;
  }
  if (!seg_ok) return;
  float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : p.y;
  const long long pix0 = (long long)n * p.M * p.HoWo + (long long)oy * p.Wo + b * RX;
  const int jmax = min(RX, p.Wo - b * RX);
#pragma unroll
  for (int r = 0; r < RM; r++) {
    const int m = m0 + wm * RM + r;
    if (m >= p.M) break;
    float *row = dst + pix0 + (long long)m * p.HoWo;
#pragma unroll
    for (int j = 0; j < RX; j++)
      if (j < jmax) row[j] = (r & 1) ? acc[r >> 1][j].y : acc[r >> 1][j].x;
  }
}

}  // namespace b2c
