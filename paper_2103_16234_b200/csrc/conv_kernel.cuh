// Direct fp32 convolution for sm_100a (B200) — the hot path of cuConv
// (arXiv 2103.16234) re-engineered for Blackwell.
//
// Reference semantics: convkit twostage.conv_twostage (twostage.py:208-239) /
// reference.conv_naive (reference.py:58-83): cross-correlation over NCHW fp32,
// virtual zero padding (tensor.py:112-123), any stride (conv_naive), output
// [n][m][ho][wo].
//
// One template serves three roles:
//   * FUSED (STRICT=false): the paper's per-filter-row dot products (stage 1)
//     and the cross-row sum (stage 2) both reduced in registers in one pass —
//     no workspace, no im2col.  Accumulation uses FFMA2 (fma.rn.f32x2, two
//     output channels per instruction, scalar-broadcast pixel operand).  The
//     per-output order is "c ascending, then (yf,xf) row-major" for every tile
//     plan, so results are bitwise independent of the plan / GPU count.
//   * STAGE 1 (STRICT=true, HF=WF=1, launched once per filter row k via
//     blockIdx.z): the paper's scalar_prods kernel — each output of filter row
//     k is a channel dot product with separately rounded multiply and add
//     (FMUL+FADD), +0.0 start, channels ascending: bitwise equal to the
//     reference's _run_block (twostage.py:101-115).
//
// Tiling (B200-first, not the paper's one-filter-row-per-block mapping):
//   CTA = BM output channels x BP flattened output pixels (n, y, x order).
//   Thread = RM=16 channels x RP=4 pixels, pixels strided by NTP so a warp's
//   lanes touch consecutive pixels (conflict-free shared loads, coalesced
//   stores) and all lanes of a warp share their 16 channels (the weight loads
//   are warp-wide broadcasts, LDS.128).
//   Input halo: the tile's receptive field is staged per channel as a band of
//   "virtual rows" of the zero-padded image stack (row V = n*Hp + padded_y),
//   so tiles may span image boundaries (small 7x7/14x14 planes) without any
//   re-layout.  Out-of-plane elements are staged as +0.0 and multiplied like
//   real data, so 0*inf = nan exactly as in the reference.
//   Filters are staged transposed, [c][tap][m], straight from [m][c][hf][wf].
//   Global->shared movement is cp.async (4-byte, zero-fill), double-buffered
//   over BC-channel chunks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace b2c {

struct KParams {
  const float *x;
  const float *w;
  float *y;
  int N, C, H, W, M;
  int S;             // stride
  int HF, WF;        // filter extent handled by THIS launch (1x1 for stage 1)
  int PH, PW;        // padding of the full filter
  int Ho, Wo, HoWo;
  int Hp;            // H + 2*PH: virtual-row period of one image
  int Q;             // N*Ho*Wo
  int RS;            // shared-memory row stride (floats)
  int ROWS;          // virtual rows staged per channel
  int XCS;           // shared-memory channel stride (floats), multiple of 4
  int tile_elems;    // ROWS*RS
  int mtiles;        // ceil(M/BM)
  int nchunks;       // ceil(C/BC)
  int w_ctaps;       // taps between consecutive channels in w (hf*wf of the full filter)
  int wf_full;       // wf of the full filter (stage 1 decodes k -> (yf, xf))
  long long y_tap_stride;  // stage 1: elements between partial planes of consecutive k
  int strict_tap_major;    // stage 1: blockIdx.z selects the filter row
};

__device__ __forceinline__ void cp_async4(float *smem_dst, const float *gmem_src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// HF_T/WF_T/S_T == 0 -> taken from the runtime parameters (generic family).
template <int HF_T, int WF_T, int S_T, int BM, int BP, int BC, bool STRICT>
struct ConvTile {
  static constexpr int RM = 16;
  static constexpr int RP = 4;
  static constexpr int NTP = BP / RP;
  static constexpr int NMG = BM / RM;
  static constexpr int NT = NMG * NTP;
  static constexpr int WS = BM + 4;  // weight row stride: keeps LDS.128 alignment, spreads banks
  static_assert(BM % RM == 0, "BM must be a multiple of 16");
  static_assert(NTP % 32 == 0, "a warp must share one channel group");
};

template <int HF_T, int WF_T, int S_T, int BM, int BP, int BC, bool STRICT>
__global__ void __launch_bounds__(ConvTile<HF_T, WF_T, S_T, BM, BP, BC, STRICT>::NT,
                                  (ConvTile<HF_T, WF_T, S_T, BM, BP, BC, STRICT>::NT >= 512 ? 1 : 2))
    conv_direct_kernel(const KParams p) {
  using T = ConvTile<HF_T, WF_T, S_T, BM, BP, BC, STRICT>;
  constexpr int RM = T::RM, RP = T::RP, NTP = T::NTP, NT = T::NT, WS = T::WS;
  const int hf = HF_T ? HF_T : p.HF;
  const int wf = WF_T ? WF_T : p.WF;
  const int S = S_T ? S_T : p.S;
  const int taps = hf * wf;

  extern __shared__ __align__(16) float smem[];
  // [goff table: tile_elems ints][stage 0: X (BC*XCS) | W (BC*taps*WS)][stage 1: ...]
  int *goff = reinterpret_cast<int *>(smem);
  const int goff_floats = (p.tile_elems + 3) & ~3;
  const int xfloats = BC * p.XCS;
  const int stage_floats = xfloats + BC * taps * WS;
  float *stage0 = smem + goff_floats;

  const int tid = threadIdx.x;
  const int mg = tid / NTP;
  const int tp = tid - mg * NTP;
  const int mt = blockIdx.x % p.mtiles;
  const int pt = blockIdx.x / p.mtiles;
  const int m0 = mt * BM;
  const int q0 = pt * BP;

  // filter row handled by this launch slice (stage 1); zero for the fused path
  int tap_y = 0, tap_x = 0, w_tap0 = 0;
  float *yout = p.y;
  if (p.strict_tap_major) {
    const int k = blockIdx.z;
    tap_y = k / p.wf_full;
    tap_x = k - tap_y * p.wf_full;
    w_tap0 = k;
    yout += (long long)k * p.y_tap_stride;
  }

  // ---- tile origin in virtual-row space -----------------------------------
  const int n0 = q0 / p.HoWo;
  const int oy0 = (q0 - n0 * p.HoWo) / p.Wo;
  const int vlo = n0 * p.Hp + oy0 * S + tap_y;
  const long long chw = (long long)p.C * p.H * p.W;
  const float *xtile = p.x + (long long)n0 * chw;
  const int hw = p.H * p.W;

  // ---- per-element global offsets of the halo band (same for every channel)
  for (int idx = tid; idx < p.tile_elems; idx += NT) {
    const int r = idx / p.RS;
    const int col = idx - r * p.RS;
    const int v = vlo + r;
    const int n = v / p.Hp;
    const int iy = v - n * p.Hp - p.PH;
    const int ix = col + tap_x - p.PW;
    const bool ok = (n < p.N) && (iy >= 0) && (iy < p.H) && (ix >= 0) && (ix < p.W);
    goff[idx] = ok ? (int)((long long)(n - n0) * chw + iy * p.W + ix) : -1;
  }

  // ---- per-thread output pixels ---------------------------------------------
  int pix_off[RP];
  long long out_off[RP];
  bool pix_ok[RP];
#pragma unroll
  for (int j = 0; j < RP; j++) {
    const int q = q0 + j * NTP + tp;
    pix_ok[j] = q < p.Q;
    const int qq = pix_ok[j] ? q : q0;
    const int n = qq / p.HoWo;
    const int rem = qq - n * p.HoWo;
    const int oy = rem / p.Wo;
    const int ox = rem - oy * p.Wo;
    pix_off[j] = ((n - n0) * p.Hp + (oy - oy0) * S) * p.RS + ox * S;
    out_off[j] = (long long)n * p.M * p.HoWo + rem;
  }
  __syncthreads();  // goff table visible

  auto load_chunk = [&](int chunk, float *stage) {
    const int c0 = chunk * BC;
    float *xs = stage;
    float *ws = stage + xfloats;
    const float *xsrc = xtile + (long long)c0 * hw;
    const int cvalid = min(BC, p.C - c0);
    for (int idx = tid; idx < p.tile_elems; idx += NT) {
      const int g = goff[idx];
      float *dst = xs + idx;
      if (g >= 0) {
#pragma unroll
        for (int c = 0; c < BC; c++)
          if (c < cvalid) cp_async4(dst + c * p.XCS, xsrc + (long long)c * hw + g);
      } else {
#pragma unroll
        for (int c = 0; c < BC; c++)
          if (c < cvalid) dst[c * p.XCS] = 0.0f;
      }
    }
    const int per_m = BC * taps;
    const int wtotal = BM * per_m;
    for (int e = tid; e < wtotal; e += NT) {
      const int m = e / per_m;
      const int ct = e - m * per_m;
      const int c = ct / taps;
      const int t = ct - c * taps;
      float *dst = ws + ct * WS + m;
      if (m0 + m < p.M && c < cvalid)
        cp_async4(dst, p.w + ((long long)(m0 + m) * p.C + c0 + c) * p.w_ctaps + w_tap0 + t);
      else
        *dst = 0.0f;
    }
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

  // ---- main loop: double-buffered channel chunks ----------------------------
  load_chunk(0, stage0);
  cp_async_commit();
  for (int chunk = 0; chunk < p.nchunks; chunk++) {
    float *cur = stage0 + (chunk & 1) * stage_floats;
    if (chunk + 1 < p.nchunks) {
      load_chunk(chunk + 1, stage0 + ((chunk + 1) & 1) * stage_floats);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    const int cvalid = min(BC, p.C - chunk * BC);
    const float *xs = cur;
    const float *wsm = cur + xfloats + mg * RM;
#pragma unroll 1
    for (int c = 0; c < cvalid; c++) {
      const float *xc = xs + c * p.XCS;
      const float *wc = wsm + c * taps * WS;
#pragma unroll
      for (int yy = 0; yy < hf; yy++) {
        const float *xrow = xc + yy * p.RS;
#pragma unroll
        for (int xx = 0; xx < wf; xx++) {
          const float *wt = wc + (yy * wf + xx) * WS;
          float wv[RM];
#pragma unroll
          for (int i = 0; i < RM; i += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(wt + i);
            wv[i] = v.x; wv[i + 1] = v.y; wv[i + 2] = v.z; wv[i + 3] = v.w;
          }
          float xv[RP];
#pragma unroll
          for (int j = 0; j < RP; j++) xv[j] = xrow[pix_off[j] + xx];
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
    }
    __syncthreads();
  }

  // ---- epilogue: fully overwrite y ------------------------------------------
  const long long plane = p.HoWo;
#pragma unroll
  for (int i = 0; i < RM; i++) {
    const int m = m0 + mg * RM + i;
    if (m >= p.M) break;
#pragma unroll
    for (int j = 0; j < RP; j++) {
      if (!pix_ok[j]) continue;
      float v;
      if (STRICT)
        v = accs[STRICT ? i : 0][STRICT ? j : 0];
      else
        v = (i & 1) ? acc2[i >> 1][j].y : acc2[i >> 1][j].x;
      yout[out_off[j] + (long long)m * plane] = v;
    }
  }
}

// Stage 2 (twostage.py:175-205): y = +0.0 + p_0 + p_1 + ... + p_{k-1}, every
// add rounded (FADD, never contracted).  HBM-bound streaming kernel.
__global__ void __launch_bounds__(256) stage2_sum_kernel(const float *__restrict__ partials, float *__restrict__ y,
                                                         long long total, int taps) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  if ((total & 3) == 0) {
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
