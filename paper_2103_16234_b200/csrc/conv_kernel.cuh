// Direct fp32 convolution for sm_100a (B200) — the hot path of cuConv
// (arXiv 2103.16234) re-engineered for Blackwell.
//
// Reference semantics: convkit twostage.conv_twostage (twostage.py:208-239) /
// reference.conv_naive (reference.py:58-83): cross-correlation over NCHW fp32,
// virtual zero padding (tensor.py:112-123), any stride (conv_naive), output
// [n][m][ho][wo].
//
// One template serves two roles:
//   * FUSED (STRICT=false): the paper's per-filter-row channel dot products
//     (its stage 1) and the cross-row sum (its stage 2) both reduced in
//     registers in one pass — no partial-sum planes, no im2col.  Accumulation
//     is FFMA2 (fma.rn.f32x2: two output channels per instruction with a
//     scalar-broadcast pixel operand).  Per output the order is "channels
//     ascending, filter taps row-major inside each channel" within each of
//     `splits` contiguous channel ranges; the range partials (splits > 1) are
//     combined in ascending range order by the tile's last-arriving CTA
//     (deterministic, no atomics on data).
//   * STAGE 1 (STRICT=true, HF=WF=1, blockIdx.z = filter row k): the paper's
//     scalar_prods kernel — channel dot products with separately rounded
//     multiply and add (FMUL+FADD), +0.0 start, channels ascending: bitwise
//     equal to the reference's _run_block (twostage.py:101-115).
//
// Tiling (B200-first, not the paper's one-filter-row-per-block mapping):
//   CTA = BM output channels x BP flattened output pixels (n, y, x order).
//   Thread = RM=16 channels x RP=4 pixels; a thread's pixels are strided by
//   NTP so a warp's lanes touch consecutive pixels (conflict-free shared loads,
//   coalesced stores), and all lanes of a warp share their 16 channels (weight
//   loads are warp-wide broadcasts, LDS.128).
//   Input halo: per channel, the tile's receptive field is staged as a band of
//   "virtual rows" of the zero-padded image stack (row V = n*Hp + padded_y), so
//   a tile may span image boundaries (7x7/14x14 planes) with no re-layout.
//   Out-of-plane elements are staged as +0.0 and multiplied like real data, so
//   0*inf = nan exactly as in the reference.  Filters are staged transposed,
//   [c][tap][m], straight from [m][c][hf][wf].  Global->shared movement is
//   cp.async (4-byte) double-buffered over BC-channel chunks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace b2c {

struct KParams {
  const float *x;
  const float *w;
  float *y;
  float *partials;   // split-C partial planes: [split][n][m][ho][wo]
  long long part_stride;  // elements per partial plane (N*M*Ho*Wo)
  int N, C, H, W, M;
  int S;             // stride
  int HF, WF;        // filter extent handled by THIS launch (1x1 for stage 1)
  int PH, PW;        // padding of the full filter
  int Ho, Wo, HoWo;
  int Hp;            // H + 2*PH: virtual-row period of one image
  int Q;             // N*Ho*Wo
  int RS;            // shared-memory row stride (floats), == W (mod 4) so rows stay 16B-congruent
  int RC;            // staged columns per row: (Wo-1)*S + WF
  int ROWS;          // staged virtual rows per channel
  int XCS;           // shared-memory channel stride (floats), multiple of 4, >= ROWS*RS + 3
  int vec_ok;        // H*W % 4 == 0 and x 16B-aligned: 16-byte cp.async groups allowed
  int vec_out;       // pointwise kernels: Ho*Wo % 4 == 0 and y (and partials) 16B-aligned: float4 stores
  int mtiles;        // ceil(M/BM)
  int ptiles;        // ceil(Q/BP) (pointwise kernels: work items = mtiles * ptiles * splits)
  int nchunks;       // ceil(C/BC)
  int splits;        // channel ranges reduced separately (blockIdx.y)
  int chunks_per_split;
  int w_ctaps;       // taps between consecutive channels in w (hf*wf of the full filter)
  int wf_full;       // wf of the full filter (stage 1 decodes k -> (yf, xf))
  long long y_tap_stride;  // stage 1: elements between partial planes of consecutive k
  int strict_tap_major;    // stage 1: blockIdx.z selects the filter row
  unsigned long long *trace;  // optional per-CTA (smid, t_start, t_tables, t_loop, t_end) records
  unsigned long long mRS, mHp, mHoWo, mWo;  // exact division magics: floor(2^44/d) + 1 (see fdiv)
  int pdl;                    // launched with programmatic dependent launch
  int cluster;                // split-C partials reduced through DSMEM: the splits of a tile form one cluster
  int nb;                     // row-segment kernel (conv_row.cuh): segments per output row
  int segs;                   // row-segment kernel: N*Ho*nb segments
  int w_tma;                  // warp-specialised row kernel: filter tiles by 2-D TMA (tensor map argument)
  unsigned long long spin_limit;  // mbarrier wait bound (ns) before __trap; 0 = unbounded (watchdog_ns())
  int qp;                     // packed pointwise (kind 9): row pitch of the packed pixels x'[C][qp], qp = Q rounded up to 4
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// floor(x / d) via a host-computed magic m = floor(2^44/d) + 1 (fdiv_magic).
// Exact for 0 <= x < 2^20 and 1 <= d < 2^24: m = 2^44/d + e with 0 < e <= 1,
// so x*m/2^44 = x/d + x*e/2^44 with x*e/2^44 < 2^-24 < 1/d, which never
// carries past the next integer; x*m < 2^20 * (2^44 + 1) fits 64 bits.  The
// planner keeps every divided quantity below 2^20 (fdiv_range_ok).
constexpr int kFdivShift = 44;
constexpr long long kFdivLimit = 1LL << 20;
__host__ __device__ __forceinline__ unsigned long long fdiv_magic(int d) {
  return ((1ULL << kFdivShift) / (unsigned long long)d) + 1ULL;
}
__device__ __forceinline__ int fdiv(int x, unsigned long long m) {
  return (int)(((unsigned long long)(unsigned)x * m) >> kFdivShift);
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ void cp_async4(float *smem_dst, const float *gmem_src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16(float *smem_dst, const float *gmem_src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// --- split-C reduction inside a thread-block cluster ---------------------------
// The `splits` CTAs of one output tile (blockIdx.y = channel range) launch as
// one cluster (dims 1 x splits x 1).  Each CTA has parked its accumulator tile
// [BM][BP] (row = output channel, column = output pixel) at the base of its
// shared memory; after a cluster barrier, rank r sums slice r of the tile over
// ranks 0..splits-1 in ascending order (every add rounded, +0.0 start: the
// sum stage2_sum_kernel forms from partial planes, so results are bitwise
// identical) and stores it.  No partial planes in HBM, no second kernel.
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(unsigned local_addr, unsigned rank) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote)
               : "memory");
  return v;
}

// Store elements [lo, hi) of a shared-memory tile [BM][BP] (row = output
// channel, column = output pixel q0 + col) to `dst` (y layout): consecutive
// threads take consecutive pixels, so a warp writes one contiguous run per
// image (coalesced for any H*W, unlike per-thread register tiles).
template <int BM, int BP, int NT>
__device__ __forceinline__ void store_tile_coalesced(const KParams &p, const float *tile, float *dst, int m0, int q0,
                                                     int lo, int hi) {
  const int hw = p.HoWo;
  const int n0 = q0 / hw;
  const int r0 = q0 - n0 * hw;
  for (int i = lo + (int)threadIdx.x; i < hi; i += NT) {
    const int row = i / BP;
    const int col = i - row * BP;
    const int m = m0 + row;
    if (m >= p.M || q0 + col >= p.Q) continue;
    const int rel = r0 + col;  // < hw + BP < 2^20
    const int dn = fdiv(rel, p.mHoWo);
    dst[(long long)(n0 + dn) * p.M * hw + (long long)m * hw + (rel - dn * hw)] = tile[i];
  }
}

template <int BM, int BP, int NT>
__device__ __forceinline__ void cluster_reduce_tile(const KParams &p, float *tile, int m0, int q0) {
  cluster_barrier();
  constexpr int F4 = BM * BP / 4;
  const int S = p.splits;
  const int per = (F4 + S - 1) / S;
  const int lo = (int)cluster_rank() * per;
  const int hi = min(F4, lo + per);
  const unsigned tile_sa = (unsigned)__cvta_generic_to_shared(tile);
  const int hw = p.HoWo;
  // 16-byte stores when 4 consecutive pixels always share an image and y is aligned
  const bool vec = (hw & 3) == 0 && (reinterpret_cast<uintptr_t>(p.y) & 15) == 0;
  for (int i = lo + (int)threadIdx.x; i < hi; i += NT) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < S; s++) {
      const float4 v = ld_dsmem_f4(tile_sa + 16u * (unsigned)i, (unsigned)s);
      a.x = __fadd_rn(a.x, v.x);
      a.y = __fadd_rn(a.y, v.y);
      a.z = __fadd_rn(a.z, v.z);
      a.w = __fadd_rn(a.w, v.w);
    }
    const int row = i / (BP / 4);
    const int q = q0 + (i - row * (BP / 4)) * 4;
    const int m = m0 + row;
    if (m >= p.M || q >= p.Q) continue;
    if (vec) {
      const int n = q / hw;
      *reinterpret_cast<float4 *>(p.y + (long long)n * p.M * hw + (long long)m * hw + (q - n * hw)) = a;
    } else {
      // slice i of this CTA's own tile is read by this CTA only: park the sum there
      *reinterpret_cast<float4 *>(tile + 4 * i) = a;
    }
  }
  if (!vec) {
    __syncthreads();
    store_tile_coalesced<BM, BP, NT>(p, tile, p.y, m0, q0, 4 * lo, 4 * hi);
  }
  cluster_barrier();  // keep this CTA's tile alive until every rank has read it
}

// ---- halo staging, shared by the direct kernels ---------------------------------
// A tile's receptive field is a band of ROWS "virtual rows" (row V = n*Hp +
// padded y) of RC columns, staged per channel at shared position
// shift + r*RS + col (RS == W mod 4, so every row is 16-byte congruent with its
// global row).  goff[pos] = global element offset relative to image n0 channel
// 0 (-1: zero padding, -2: unused slot); gtab[G] = offset of an aligned run of
// 4 data elements for 16-byte group G, -1 for a mixed group (element-wise
// copies), -3 for an all-unused group.  Built once per tile, reused for every
// channel chunk.  Ends with a barrier (gtab reads goff).
template <int NT>
__device__ __forceinline__ void build_halo_tables(const KParams &p, int *goff, int *gtab, int vlo, int n0, int shift,
                                                  int tap_x, long long chw) {
  for (int pos = threadIdx.x; pos < p.XCS; pos += NT) {
    const int rel = pos - shift;
    int g = -2;
    if (rel >= 0) {
      const int r = fdiv(rel, p.mRS);
      const int col = rel - r * p.RS;
      if (r < p.ROWS && col < p.RC) {
        const int vrel = vlo - n0 * p.Hp + r;  // virtual row relative to image n0 (< 2^20)
        const int dn = fdiv(vrel, p.mHp);
        const int n = n0 + dn;
        const int iy = vrel - dn * p.Hp - p.PH;
        const int ix = col + tap_x - p.PW;
        const bool ok = (n < p.N) && (iy >= 0) && (iy < p.H) && (ix >= 0) && (ix < p.W);
        g = ok ? (int)((long long)dn * chw + iy * p.W + ix) : -1;
      }
    }
    goff[pos] = g;
  }
  __syncthreads();
  const int ngroups = p.XCS >> 2;
  for (int G = threadIdx.x; G < ngroups; G += NT) {
    const int g0 = goff[4 * G], g1 = goff[4 * G + 1], g2 = goff[4 * G + 2], g3 = goff[4 * G + 3];
    int t = -1;
    if (p.vec_ok && g0 >= 0 && (g0 & 3) == 0 && g1 == g0 + 1 && g2 == g0 + 2 && g3 == g0 + 3) t = g0;
    else if (g0 == -2 && g1 == -2 && g2 == -2 && g3 == -2) t = -3;
    gtab[G] = t;
  }
}

// Stage BC channel planes of the band (channel stride XCS floats) from xsrc =
// &x[n0][c0][0][0]: 16-byte cp.async for aligned data runs, 4-byte copies and
// (ZERO) +0.0 stores of the padding elsewhere; channels >= cvalid are left
// untouched (never read).  Threads t0, t0 + tstride, ... of the CTA take part.
template <int BC, bool ZERO = true>
__device__ __forceinline__ void stage_halo_chunk(const KParams &p, const int *goff, const int *gtab, float *xs,
                                                 const float *xsrc, int cvalid, int hw, int t0, int tstride) {
  const int ngroups = p.XCS >> 2;
  for (int G = t0; G < ngroups; G += tstride) {
    const int t = gtab[G];
    if (t == -3) continue;
    float *dst = xs + 4 * G;
    if (t >= 0) {
      const float *src = xsrc + t;
#pragma unroll
      for (int c = 0; c < BC; c++) {
        if (c < cvalid) cp_async16(dst, src);
        dst += p.XCS;
        src += hw;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int g = goff[4 * G + k];
        float *d = dst + k;
        if (g >= 0) {
          const float *src = xsrc + g;
          for (int c = 0; c < cvalid; c++, d += p.XCS, src += hw) cp_async4(d, src);
        } else if (ZERO && g == -1) {
          for (int c = 0; c < cvalid; c++, d += p.XCS) *d = 0.0f;
        }
      }
    }
  }
}

// Filters w[m0+m][c0+c][tap] -> ws[(c*taps + tap)*(BM+4) + m] (transposed, so
// a thread's 16 output channels of one (channel, tap) are 4 LDS.128); wsrc =
// &w[m0][c0][tap0]; per_m = BC*taps; taps past ct_valid and channels past M
// are zero.
template <int NT, int BM>
__device__ __forceinline__ void stage_filter_chunk(const KParams &p, float *ws, const float *wsrc, int per_m, int taps,
                                                   int ct_valid, bool w_dense, int m0) {
  constexpr int WS = BM + 4;
  const int wtotal = BM * per_m;
  const int mstride = p.C * p.w_ctaps;
  for (int e = threadIdx.x; e < wtotal; e += NT) {
    const int m = e / per_m;
    const int ct = e - m * per_m;
    float *dst = ws + ct * WS + m;
    if (m0 + m < p.M && ct < ct_valid) {
      const int off = w_dense ? ct : (ct / taps) * p.w_ctaps + (ct % taps);
      cp_async4(dst, wsrc + m * mstride + off);
    } else {
      *dst = 0.0f;
    }
  }
}

// HF_T/WF_T/S_T == 0 -> taken from the runtime parameters (generic family).
// RP_ = output pixels per thread: 4 (64 accumulators, 2 CTAs of 256 threads per
// SM) or 8 (128 accumulators, 128-thread CTAs).  Per (channel, tap) a thread
// loads 16 filter values (4 LDS.128, warp-wide broadcast, 4 shared-memory
// wavefronts each) and RP pixels (1 wavefront each) for 8*RP FFMA2: at RP = 4
// that is 20 wavefronts per 64 FMA-pipe cycles of a warp, 80 % of the
// 128 B/clk shared-memory rate at the FFMA2 peak with four warps per SMSP
// (the measured ceiling of the 3x3 family, ~68 % FMA-pipe active); RP = 8
// needs 24 per 128 cycles (75 % at peak).
template <int HF_T, int WF_T, int S_T, int BM, int BP, int BC, bool STRICT, int RP_ = 4>
struct ConvTile {
  static constexpr int RM = 16;
  static constexpr int RP = RP_;
  static constexpr int NTP = BP / RP;
  static constexpr int NMG = BM / RM;
  static constexpr int NT = NMG * NTP;
  static constexpr int WS = BM + 4;  // weight row stride: keeps LDS.128 alignment, spreads banks
  // target 16 resident warps per SM at <= 128 registers per thread
  static constexpr int MIN_BLOCKS = RP_ == 4 ? (NT >= 512 ? 1 : 512 / NT) : (NT >= 256 ? 1 : 256 / NT);
  static_assert(BM % RM == 0, "BM must be a multiple of 16");
  static_assert(NTP % 32 == 0, "a warp must share one channel group");
};

template <int HF_T, int WF_T, int S_T, int BM, int BP, int BC, bool STRICT, int RP_ = 4>
__global__ void __launch_bounds__(ConvTile<HF_T, WF_T, S_T, BM, BP, BC, STRICT, RP_>::NT,
                                  ConvTile<HF_T, WF_T, S_T, BM, BP, BC, STRICT, RP_>::MIN_BLOCKS)
    conv_direct_kernel(const KParams p) {
  using T = ConvTile<HF_T, WF_T, S_T, BM, BP, BC, STRICT, RP_>;
  constexpr int RM = T::RM, RP = T::RP, NTP = T::NTP, NT = T::NT, WS = T::WS;
  const int hf = HF_T ? HF_T : p.HF;
  const int wf = WF_T ? WF_T : p.WF;
  const int S = S_T ? S_T : p.S;
  const int taps = hf * wf;

  extern __shared__ __align__(16) float smem[];
  // [goff: XCS ints][gtab: XCS/4 ints][stage 0: X (BC*XCS) | W (BC*taps*WS)][stage 1: ...]
  int *goff = reinterpret_cast<int *>(smem);
  int *gtab = goff + p.XCS;
  const int ngroups = p.XCS >> 2;
  const int xfloats = BC * p.XCS;
  const int stage_floats = xfloats + BC * taps * WS;
  float *stage0 = smem + p.XCS + ((ngroups + 3) & ~3);

  const int tid = threadIdx.x;
  const unsigned long long t_start = p.trace ? global_ns() : 0ull;
  const int mg = tid / NTP;
  const int tp = tid - mg * NTP;
  const int tile = blockIdx.x;
  const int mt = tile % p.mtiles;
  const int pt = tile / p.mtiles;
  const int m0 = mt * BM;
  const int q0 = pt * BP;
  const int split = blockIdx.y;

  // filter row handled by this launch slice (stage 1); zero for the fused path
  int tap_y = 0, tap_x = 0, w_tap0 = 0;
  if (p.strict_tap_major) {
    const int k = blockIdx.z;
    tap_y = k / p.wf_full;
    tap_x = k - tap_y * p.wf_full;
    w_tap0 = k;
  }

  // ---- tile origin in virtual-row space -----------------------------------
  const int n0 = q0 / p.HoWo;  // q0 may exceed 2^20: exact hardware division once per CTA
  const int oy0 = fdiv(q0 - n0 * p.HoWo, p.mWo);
  const int vlo = n0 * p.Hp + oy0 * S + tap_y;
  const long long chw = (long long)p.C * p.H * p.W;
  const int hw = p.H * p.W;
  // shift so that shared position == global offset (mod 4) along rows: the
  // interior of every row can then move as 16-byte groups
  const int shift = (((vlo - n0 * p.Hp - p.PH) * p.W + tap_x - p.PW) % 4 + 4) % 4;

  build_halo_tables<NT>(p, goff, gtab, vlo, n0, shift, tap_x, chw);
  // ---- per-thread output pixels: shared-memory offsets of their windows ----
  const long long trace_cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  int pix_off[RP];
#pragma unroll
  for (int j = 0; j < RP; j++) {
    const int qr = min(q0 + j * NTP + tp, p.Q - 1) - n0 * p.HoWo;  // relative to image n0 (< 2^20)
    const int dn = fdiv(qr, p.mHoWo);
    const int rem = qr - dn * p.HoWo;
    const int oy = fdiv(rem, p.mWo);
    const int ox = rem - oy * p.Wo;
    pix_off[j] = shift + (dn * p.Hp + (oy - oy0) * S) * p.RS + ox * S;
  }
  __syncthreads();  // tables visible
  if (p.trace && tid == 0) {
    p.trace[5 * trace_cta] = smid();
    p.trace[5 * trace_cta + 1] = t_start;
    p.trace[5 * trace_cta + 2] = global_ns();
  }

  const float *xtile = p.x + (long long)n0 * chw;
  const bool w_dense = (p.w_ctaps == taps);  // fused: filter taps of a channel are contiguous
  auto load_chunk = [&](int chunk, float *stage) {
    const int c0 = chunk * BC;
    const int cvalid = min(BC, p.C - c0);
    stage_halo_chunk<BC>(p, goff, gtab, stage, xtile + (long long)c0 * hw, cvalid, hw, threadIdx.x, NT);
    stage_filter_chunk<NT, BM>(p, stage + xfloats, p.w + ((long long)m0 * p.C + c0) * p.w_ctaps + w_tap0, BC * taps,
                               taps, cvalid * taps, w_dense, m0);
  };

  // ---- accumulators -------------------------------------------------------
  float2 acc2[RM / 2][RP];  // fused: channel pairs (2i, 2i+1)
  float accs[STRICT ? RM : 1][STRICT ? RP : 1];
  if (STRICT) {
#pragma unroll
    for (int i = 0; i < (STRICT ? RM : 1); i++)
#pragma unroll
      for (int j = 0; j < (STRICT ? RP : 1); j++) accs[i][j] = 0.0f;
  } else {
#pragma unroll
    for (int i = 0; i < RM / 2; i++)
#pragma unroll
      for (int j = 0; j < RP; j++) acc2[i][j] = make_float2(0.0f, 0.0f);
  }

  // ---- main loop: double-buffered channel chunks of this split --------------
  // Programmatic dependent launch: everything above (tables, addressing) overlaps
  // the previous kernel's tail; inputs are read only after it has completed.
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int chunk_begin = split * p.chunks_per_split;
  const int chunk_end = min(p.nchunks, chunk_begin + p.chunks_per_split);
  if (chunk_begin < chunk_end) {
    load_chunk(chunk_begin, stage0);
    cp_async_commit();
  }
  for (int chunk = chunk_begin; chunk < chunk_end; chunk++) {
    const int buf = (chunk - chunk_begin) & 1;
    float *cur = stage0 + buf * stage_floats;
    if (chunk + 1 < chunk_end) {
      load_chunk(chunk + 1, stage0 + (buf ^ 1) * stage_floats);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    const int cvalid = min(BC, p.C - chunk * BC);
    // strength-reduced shared addresses: one base per output pixel, one for
    // this warp's 16 filter columns; advanced by a channel plane per step
    const float *xcur[RP];
#pragma unroll
    for (int j = 0; j < RP; j++) xcur[j] = cur + pix_off[j];
    const float *wcur = cur + xfloats + mg * RM;
    const int wstep = taps * WS;
    constexpr int CUNROLL = (HF_T == 1 && WF_T == 1) ? 2 : 1;  // 1x1: two channels per trip
#pragma unroll CUNROLL
    for (int c = 0; c < cvalid; c++) {
#pragma unroll 1
      for (int yy = 0; yy < hf; yy++) {
        const int roff = yy * p.RS;
#pragma unroll
        for (int xx = 0; xx < wf; xx++) {
          const float *wt = wcur + (yy * wf + xx) * WS;
          float wv[RM];
#pragma unroll
          for (int i = 0; i < RM; i += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(wt + i);
            wv[i] = v.x; wv[i + 1] = v.y; wv[i + 2] = v.z; wv[i + 3] = v.w;
          }
          float xv[RP];
#pragma unroll
          for (int j = 0; j < RP; j++) xv[j] = xcur[j][roff + xx];
          if (STRICT) {
#pragma unroll
            for (int i = 0; i < (STRICT ? RM : 1); i++)
#pragma unroll
              for (int j = 0; j < (STRICT ? RP : 1); j++)
                accs[i][j] = __fadd_rn(accs[i][j], __fmul_rn(xv[j], wv[i]));
          } else {
#pragma unroll
            for (int i = 0; i < RM / 2; i++)
#pragma unroll
              for (int j = 0; j < RP; j++)
                acc2[i][j] = __ffma2_rn(make_float2(wv[2 * i], wv[2 * i + 1]), make_float2(xv[j], xv[j]),
                                        acc2[i][j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < RP; j++) xcur[j] += p.XCS;
      wcur += wstep;
    }
    __syncthreads();
  }

  auto acc_at = [&](int i, int j) -> float {
    if (STRICT) return accs[STRICT ? i : 0][STRICT ? j : 0];
    return (i & 1) ? acc2[i >> 1][j].y : acc2[i >> 1][j].x;
  };

  if (p.trace && tid == 0) p.trace[5 * trace_cta + 3] = global_ns();
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  auto trace_end = [&]() {
    if (p.trace && tid == 0) p.trace[5 * trace_cta + 4] = global_ns();
  };
  // ---- epilogue ---------------------------------------------------------------
  float *yout = p.y;
  if (p.strict_tap_major) yout += (long long)blockIdx.z * p.y_tap_stride;
  long long out_off[RP];
  bool pix_ok[RP];
#pragma unroll
  for (int j = 0; j < RP; j++) {
    const int q = q0 + j * NTP + tp;
    pix_ok[j] = q < p.Q;
    const int qq = pix_ok[j] ? q : 0;
    const int n = qq / p.HoWo;
    out_off[j] = (long long)n * p.M * p.HoWo + (qq - n * p.HoWo);
  }
  const long long plane = p.HoWo;

  if (p.cluster) {  // split-C through DSMEM (cluster_reduce_tile)
    cp_async_wait<0>();
    __syncthreads();  // the tile overwrites the halo tables and pipeline stages
#pragma unroll
    for (int i = 0; i < RM; i++)
#pragma unroll
      for (int j = 0; j < RP; j++) smem[(mg * RM + i) * BP + j * NTP + tp] = acc_at(i, j);
    cluster_reduce_tile<BM, BP, NT>(p, smem, m0, q0);
    trace_end();
    return;
  }
  // splits == 1: fully overwrite y.  splits > 1: this channel range's partial
  // goes to plane `split` of the workspace (y layout); stage2_sum_kernel then
  // adds the planes in ascending order (deterministic, no atomics).
  float *dst = p.splits > 1 ? p.partials + (long long)split * p.part_stride : yout;
#pragma unroll
  for (int i = 0; i < RM; i++) {
    const int m = m0 + mg * RM + i;
    if (m >= p.M) break;
#pragma unroll
    for (int j = 0; j < RP; j++)
      if (pix_ok[j]) dst[out_off[j] + (long long)m * plane] = acc_at(i, j);
  }
  trace_end();
}

// Stage 2 (twostage.py:175-205): y = +0.0 + p_0 + p_1 + ... + p_{k-1}, every
// add rounded (FADD, never contracted).  HBM-bound streaming kernel.  `vec`:
// total % 4 == 0 and both pointers 16-byte aligned (decided by the launcher;
// a view at an odd float offset takes the scalar loop).
__global__ void __launch_bounds__(256) stage2_sum_kernel(const float *__restrict__ partials, float *__restrict__ y,
                                                         long long total, int taps, int pdl, int vec) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // partials come from the previous grid
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (vec) {
    const long long total4 = total >> 2;
    const float4 *p4 = reinterpret_cast<const float4 *>(partials);
    float4 *y4 = reinterpret_cast<float4 *>(y);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += stride) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k = 0; k < taps; k++) {
        const float4 v = __ldcs(p4 + (long long)k * total4 + i);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
      y4[i] = acc;
    }
  } else {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      float acc = 0.0f;
      for (int k = 0; k < taps; k++) acc = __fadd_rn(acc, __ldcs(partials + (long long)k * total + i));
      y[i] = acc;
    }
  }
}

}  // namespace b2c
