// Kernel instantiations, the B200 tile planner and launch helpers.
//
// The reference plans one filter row per block with <=1024 threads
// (execmodel.plan_launch, execmodel.py:73-98).  On B200 the planner instead
// picks, per (filter size, stride, channels, spatial size, batch), a kernel
// family (BM output channels x BP output pixels per CTA, BC channels per
// pipeline stage) by minimising an occupancy- and wave-quantisation-aware cost
// over the 148 SMs.  The reference plan is still computed and validated by the
// C ABI for the drop-in's RunStats / InvalidPlan contract (api.cpp).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>
#include <cstdio>

#include "conv1x1_vec.cuh"
#include "conv1x1_ws.cuh"
#include "conv1x1_tma.cuh"
#include "conv_kernel.cuh"
#include "conv_row.cuh"
#include "internal.h"

namespace b2c {

namespace {

struct Family {
  const char *name;
  int hf, wf, s;  // 0 = generic (runtime)
  int bm, bp, bc;
  bool strict;
  int threads;
  const void *kernel;
  int max_ctas_per_sm;  // from __launch_bounds__
  int kind;             // 0: conv_direct_kernel (halo staging), 1: conv1x1_vec_kernel, 2: its 4-byte variant,
                        // 3: conv_row_kernel (row segments, halo staging), 4: its warp-specialised
                        //    variant (producer warp, mbarrier ring, TMA filter tiles), 5: the
                        //    warp-specialised pointwise kernel (conv1x1_ws.cuh, any stride), 6: the
                        //    TMA-fed pointwise kernel (conv1x1_tma.cuh), 9: conv1x1_vec_kernel on
                        //    packed pixels (pack_pixels_kernel first)
  int stages;           // cp.async pipeline depth of kind 1
  int tm = 2;           // pointwise kernels: channel groups of 4 per thread (4: 16 channels x 8 pixels)
  int rx = 0;           // kind 3: outputs per row segment
};

#define B2C_FAMILY(NAME, HF, WF, S, BM, BP, BC, STRICT)                                                    \
  Family {                                                                                                 \
    NAME, HF, WF, S, BM, BP, BC, STRICT, ConvTile<HF, WF, S, BM, BP, BC, STRICT>::NT,                     \
        reinterpret_cast<const void *>(&conv_direct_kernel<HF, WF, S, BM, BP, BC, STRICT>),                \
        ConvTile<HF, WF, S, BM, BP, BC, STRICT>::MIN_BLOCKS, 0, 2                                          \
  }

// 16 channels x 8 pixels per thread (conv_kernel.cuh ConvTile, RP = 8)
#define B2C_FAMILY8(NAME, HF, WF, S, BM, BP, BC)                                                           \
  Family {                                                                                                 \
    NAME, HF, WF, S, BM, BP, BC, false, ConvTile<HF, WF, S, BM, BP, BC, false, 8>::NT,                    \
        reinterpret_cast<const void *>(&conv_direct_kernel<HF, WF, S, BM, BP, BC, false, 8>),             \
        ConvTile<HF, WF, S, BM, BP, BC, false, 8>::MIN_BLOCKS, 0, 2                                        \
  }

#define B2C_VEC1X1(NAME, WM, WP, BC)                                                                       \
  Family {                                                                                                 \
    NAME, 1, 1, 1, Vec1x1Tile<WM, WP, BC>::BM, Vec1x1Tile<WM, WP, BC>::BP, BC, false,                      \
        Vec1x1Tile<WM, WP, BC>::NT, reinterpret_cast<const void *>(&conv1x1_vec_kernel<WM, WP, BC, true>), \
        Vec1x1Tile<WM, WP, BC>::MIN_BLOCKS, 1, Vec1x1Tile<WM, WP, BC>::STAGES                              \
  }
// 16 channels x 8 pixels per thread (TM = 4): 128 accumulators, 4-warp CTAs
#define B2C_VEC1X1W(NAME, WM, WP, BC)                                                                      \
  Family {                                                                                                 \
    NAME, 1, 1, 1, Vec1x1Tile<WM, WP, BC, 4>::BM, Vec1x1Tile<WM, WP, BC, 4>::BP, BC, false,                \
        Vec1x1Tile<WM, WP, BC, 4>::NT,                                                                     \
        reinterpret_cast<const void *>(&conv1x1_vec_kernel<WM, WP, BC, true, 4>),                          \
        Vec1x1Tile<WM, WP, BC, 4>::MIN_BLOCKS, 1, Vec1x1Tile<WM, WP, BC, 4>::STAGES, 4                     \
  }
// packed-pixel variants (kind 9): pack_pixels_kernel, then the 16-byte kernel on x'[C][qp]
#define B2C_PK1X1(NAME, WM, WP, BC, TM)                                                                    \
  Family {                                                                                                 \
    NAME, 1, 1, 1, Vec1x1Tile<WM, WP, BC, TM>::BM, Vec1x1Tile<WM, WP, BC, TM>::BP, BC, false,              \
        Vec1x1Tile<WM, WP, BC, TM>::NT,                                                                    \
        reinterpret_cast<const void *>(&conv1x1_vec_kernel<WM, WP, BC, true, TM, true>),                    \
        Vec1x1Tile<WM, WP, BC, TM>::MIN_BLOCKS, 9, Vec1x1Tile<WM, WP, BC, TM>::STAGES, TM                  \
  }
// 4-byte staging variant for planes with H*W % 4 != 0 (kind 2)
#define B2C_SCA1X1(NAME, WM, WP, BC)                                                                       \
  Family {                                                                                                 \
    NAME, 1, 1, 1, Vec1x1Tile<WM, WP, BC>::BM, Vec1x1Tile<WM, WP, BC>::BP, BC, false,                      \
        Vec1x1Tile<WM, WP, BC>::NT, reinterpret_cast<const void *>(&conv1x1_vec_kernel<WM, WP, BC, false>),\
        Vec1x1Tile<WM, WP, BC>::MIN_BLOCKS, 2, Vec1x1Tile<WM, WP, BC>::STAGES                              \
  }

// row-segment kernel (kind 3): 16 channels x RX outputs of one row per thread
#define B2C_ROW(NAME, HF, WF, S, RX, WM, WP, BC, MINB)                                                    \
  Family {                                                                                                 \
    NAME, HF, WF, S, RowTile<HF, WF, S, RX, WM, WP, BC, MINB>::BM,                                         \
        RowTile<HF, WF, S, RX, WM, WP, BC, MINB>::SEG * RX, BC, false,                                     \
        RowTile<HF, WF, S, RX, WM, WP, BC, MINB>::NT,                                                      \
        reinterpret_cast<const void *>(&conv_row_kernel<HF, WF, S, RX, WM, WP, BC, MINB>), MINB, 3, 2, 2, RX \
  }

// warp-specialised row-segment kernel (kind 4): ST-stage mbarrier ring, TMA filters
#define B2C_ROWWS(NAME, HF, WF, S, RX, WM, WP, BC, ST)                                                    \
  Family {                                                                                                 \
    NAME, HF, WF, S, RowWsTile<HF, WF, S, RX, WM, WP, BC, ST>::BM,                                         \
        RowWsTile<HF, WF, S, RX, WM, WP, BC, ST>::SEG * RX, BC, false,                                     \
        RowWsTile<HF, WF, S, RX, WM, WP, BC, ST>::NT,                                                      \
        reinterpret_cast<const void *>(&conv_row_ws_kernel<HF, WF, S, RX, WM, WP, BC, ST>),                \
        RowWsTile<HF, WF, S, RX, WM, WP, BC, ST>::MIN_BLOCKS, 4, ST, 2, RX                                  \
  }

// ... with NP producer warps
#define B2C_ROWWSP2(NAME, HF, WF, S, RX, WM, WP, BC, ST)                                                  \
  Family {                                                                                                 \
    NAME, HF, WF, S, RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, 2>::BM,                                      \
        RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, 2>::SEG * RX, BC, false,                                  \
        RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, 2>::NT,                                                   \
        reinterpret_cast<const void *>(&conv_row_ws_kernel<HF, WF, S, RX, WM, WP, BC, ST, 2>),             \
        RowWsTile<HF, WF, S, RX, WM, WP, BC, ST, 2>::MIN_BLOCKS, 4, ST, 2, RX                               \
  }

// warp-specialised pointwise kernel (kind 5)
#define B2C_PW1X1WS(NAME, WM, WP, BC, ST)                                                                   \
  Family {                                                                                                 \
    NAME, 1, 1, 1, Pw1x1WsTile<WM, WP, BC, ST>::BM, Pw1x1WsTile<WM, WP, BC, ST>::BP, BC, false,            \
        Pw1x1WsTile<WM, WP, BC, ST>::NT, reinterpret_cast<const void *>(&conv1x1_ws_kernel<WM, WP, BC, ST>), \
        Pw1x1WsTile<WM, WP, BC, ST>::MIN_BLOCKS, 5, ST, 4                                                   \
  }

// TMA-fed pointwise kernel (kind 6)
#define B2C_PW1X1TMA(NAME, WM, WP, BC, ST)                                                                  \
  Family {                                                                                                 \
    NAME, 1, 1, 1, Pw1x1TmaTile<WM, WP, BC, ST>::BM, Pw1x1TmaTile<WM, WP, BC, ST>::BP, BC, false,          \
        Pw1x1TmaTile<WM, WP, BC, ST>::NT, reinterpret_cast<const void *>(&conv1x1_tma_kernel<WM, WP, BC, ST>), \
        Pw1x1TmaTile<WM, WP, BC, ST>::MIN_BLOCKS, 6, ST, 2                                                  \
  }

const Family kFamilies[] = {
    // fused FFMA2 families
    B2C_FAMILY("fused_1x1s1_m16", 1, 1, 1, 16, 512, 16, false),
    B2C_FAMILY("fused_1x1s1_m32", 1, 1, 1, 32, 256, 16, false),
    B2C_FAMILY("fused_1x1s1_m64", 1, 1, 1, 64, 256, 16, false),
    B2C_FAMILY("fused_1x1s1_m128", 1, 1, 1, 128, 256, 16, false),
    B2C_FAMILY("fused_1x1s2_m64", 1, 1, 2, 64, 256, 16, false),
    B2C_FAMILY("fused_1x1s2_m128", 1, 1, 2, 128, 256, 16, false),
    B2C_FAMILY("fused_3x3s1_m32", 3, 3, 1, 32, 256, 8, false),
    B2C_FAMILY("fused_3x3s1_m32p128", 3, 3, 1, 32, 128, 8, false),  // small tiles: latency-bound batch-1 layers
    B2C_FAMILY("fused_3x3s1_m64p128", 3, 3, 1, 64, 128, 8, false),
    B2C_FAMILY("fused_3x3s1_m64", 3, 3, 1, 64, 256, 8, false),
    B2C_FAMILY("fused_3x3s1_m128", 3, 3, 1, 128, 256, 8, false),
    B2C_FAMILY8("fused_3x3s1_m64r8", 3, 3, 1, 64, 256, 8),
    B2C_FAMILY8("fused_3x3s1_m32r8", 3, 3, 1, 32, 256, 8),
    B2C_FAMILY8("fused_3x3s1_m64r8p512", 3, 3, 1, 64, 512, 8),
    B2C_FAMILY8("fused_3x3s1_m128r8", 3, 3, 1, 128, 256, 8),
    B2C_FAMILY8("fused_3x3s2_m64r8", 3, 3, 2, 64, 256, 8),
    B2C_FAMILY8("fused_3x3s2_m128r8", 3, 3, 2, 128, 256, 8),
    B2C_FAMILY8("fused_5x5s1_m64r8", 5, 5, 1, 64, 256, 4),
    B2C_FAMILY8("fused_5x5s1_m32r8", 5, 5, 1, 32, 256, 4),
    B2C_FAMILY8("fused_7x7s2_m32r8", 7, 7, 2, 32, 256, 4),
    B2C_FAMILY8("fused_7x7s2_m64r8", 7, 7, 2, 64, 256, 4),
    B2C_FAMILY("fused_7x7s2_m32", 7, 7, 2, 32, 256, 4, false),
    B2C_FAMILY("fused_7x7s2_m64p128", 7, 7, 2, 64, 128, 4, false),
    B2C_FAMILY("fused_3x3s2_m64", 3, 3, 2, 64, 256, 8, false),
    B2C_FAMILY("fused_3x3s2_m128", 3, 3, 2, 128, 256, 8, false),
    B2C_FAMILY("fused_5x5s1_m32", 5, 5, 1, 32, 256, 4, false),
    B2C_FAMILY("fused_5x5s1_m32p128", 5, 5, 1, 32, 128, 4, false),
    B2C_FAMILY("fused_5x5s1_m64", 5, 5, 1, 64, 256, 4, false),
    B2C_FAMILY("fused_5x5s1_m128", 5, 5, 1, 128, 256, 4, false),
    B2C_FAMILY("fused_7x7s2_m64", 7, 7, 2, 64, 256, 4, false),
    B2C_FAMILY("fused_generic_m64", 0, 0, 0, 64, 256, 4, false),
    B2C_FAMILY("fused_generic_m32", 0, 0, 0, 32, 256, 4, false),
    // pointwise 16-byte families (1x1, stride 1, no padding, H*W % 4 == 0)
    B2C_VEC1X1("fused_1x1v_m32", 1, 4, 16),
    B2C_VEC1X1("fused_1x1v_m32p128", 1, 2, 16),
    B2C_VEC1X1("fused_1x1v_m64", 2, 4, 16),
    B2C_VEC1X1("fused_1x1v_m64p128", 2, 2, 16),
    B2C_VEC1X1("fused_1x1v_m128", 4, 2, 16),
    B2C_VEC1X1("fused_1x1v_m32b32", 1, 4, 32),
    B2C_VEC1X1("fused_1x1v_m64b32", 2, 4, 32),
    B2C_VEC1X1("fused_1x1v_m128b32", 4, 2, 32),
    B2C_VEC1X1W("fused_1x1w_m64", 1, 4, 16),
    B2C_VEC1X1W("fused_1x1w_m128", 2, 2, 16),
    B2C_VEC1X1W("fused_1x1w_m256", 4, 1, 16),
    B2C_VEC1X1W("fused_1x1w_m128p256", 2, 4, 16),
    // pointwise on packed pixels (7x7 planes, strided projection shortcuts)
    B2C_PK1X1("fused_1x1pk_m64", 2, 4, 16, 2),
    B2C_PK1X1("fused_1x1pk_m64b32", 2, 4, 32, 2),
    B2C_PK1X1("fused_1x1pk_m128", 4, 2, 16, 2),
    B2C_PK1X1("fused_1x1pkw_m64", 1, 4, 16, 4),
    B2C_PK1X1("fused_1x1pkw_m128", 2, 2, 16, 4),
    // pointwise, 4-byte pixel staging (1x1, stride 1, no padding, any H*W)
    // (and strided 1x1, e.g. ResNet projection shortcuts)
    B2C_SCA1X1("fused_1x1s_m32", 1, 4, 16),
    B2C_SCA1X1("fused_1x1s_m64", 2, 4, 16),
    B2C_SCA1X1("fused_1x1s_m64p128", 2, 2, 16),
    B2C_SCA1X1("fused_1x1s_m128", 4, 2, 16),
    // paper-faithful stage 1 (strict FMUL+FADD, one filter row per blockIdx.z)
    B2C_FAMILY("stage1_strict_m32", 1, 1, 1, 32, 256, 16, true),
    B2C_FAMILY("stage1_strict_m64", 1, 1, 1, 64, 256, 16, true),
    // row-segment families (conv_row.cuh)
    B2C_ROW("fused_3x3s1_row7_m64", 3, 3, 1, 7, 4, 1, 8, 3),
    B2C_ROW("fused_3x3s1_row7_m64w2", 3, 3, 1, 7, 4, 2, 8, 1),
    B2C_ROW("fused_3x3s1_row7_m128", 3, 3, 1, 7, 8, 1, 8, 1),
    B2C_ROW("fused_3x3s1_row7_m32", 3, 3, 1, 7, 2, 2, 8, 3),
    B2C_ROW("fused_3x3s2_row7_m64", 3, 3, 2, 7, 4, 1, 8, 3),
    B2C_ROW("fused_3x3s2_row7_m128", 3, 3, 2, 7, 8, 1, 8, 1),
    B2C_ROW("fused_5x5s1_row7_m64", 5, 5, 1, 7, 4, 1, 4, 3),
    B2C_ROW("fused_5x5s1_row7_m32", 5, 5, 1, 7, 2, 2, 4, 3),
    B2C_ROW("fused_7x7s2_row7_m64", 7, 7, 2, 7, 4, 1, 4, 2),
    B2C_ROWWS("fused_3x3s1_rws7_m64", 3, 3, 1, 7, 4, 1, 8, 3),
    B2C_ROWWSP2("fused_3x3s1_rws7_m64p2", 3, 3, 1, 7, 4, 1, 8, 3),
    B2C_ROWWSP2("fused_3x3s1_rws7_m64c12st2p2", 3, 3, 1, 7, 4, 1, 12, 2),
    B2C_ROWWS("fused_3x3s1_rws7_m64w2", 3, 3, 1, 7, 4, 2, 8, 4),
    B2C_ROWWS("fused_3x3s1_rws7_m32", 3, 3, 1, 7, 2, 2, 8, 3),
    B2C_ROWWS("fused_3x3s1_rws7_m128", 3, 3, 1, 7, 8, 1, 8, 3),
    B2C_ROWWS("fused_3x3s2_rws7_m64", 3, 3, 2, 7, 4, 1, 8, 3),
    B2C_ROWWS("fused_3x3s2_rws7_m128", 3, 3, 2, 7, 8, 1, 8, 3),
    B2C_ROWWSP2("fused_3x3s2_rws7_m128p2", 3, 3, 2, 7, 8, 1, 8, 3),
    B2C_ROWWSP2("fused_3x3s2_rws7_m64p2", 3, 3, 2, 7, 4, 1, 8, 3),
    B2C_ROWWSP2("fused_3x3s2_rws7_m64c4p2", 3, 3, 2, 7, 4, 1, 4, 3),
    B2C_ROWWS("fused_5x5s1_rws7_m64", 5, 5, 1, 7, 4, 1, 4, 3),
    B2C_ROWWSP2("fused_5x5s1_rws7_m64p2", 5, 5, 1, 7, 4, 1, 4, 3),
    B2C_ROWWS("fused_5x5s1_rws7_m32", 5, 5, 1, 7, 2, 2, 4, 3),
    B2C_ROWWS("fused_7x7s2_rws7_m64", 7, 7, 2, 7, 4, 1, 4, 2),
    // stride 2 on small planes: the band is ~2x the output rows, so 4-channel stages keep 2 CTAs per SM
    B2C_ROWWS("fused_3x3s2_rws7_m64c4", 3, 3, 2, 7, 4, 1, 4, 3),
    B2C_ROWWS("fused_3x3s2_rws7_m128c4", 3, 3, 2, 7, 8, 1, 4, 3),
    // single-chunk layers (ResNet conv1, C = 3): one stage, two CTAs per SM
    B2C_ROWWS("fused_7x7s2_rws7_m64st1", 7, 7, 2, 7, 4, 1, 4, 1),
    B2C_ROWWS("fused_7x7s2_rws7_m32st1", 7, 7, 2, 7, 2, 2, 4, 1),
    // 3-channel stages (ResNet conv1): the filter rows of a tile are one contiguous bulk copy
    B2C_ROWWS("fused_7x7s2_rws7_m64c3", 7, 7, 2, 7, 4, 1, 3, 1),
    B2C_ROWWSP2("fused_7x7s2_rws7_m64c3p2", 7, 7, 2, 7, 4, 1, 3, 1),
    B2C_ROWWS("fused_7x7s2_rws7_m32c3", 7, 7, 2, 7, 2, 2, 3, 1),
    // persistent warp-specialised pointwise families (conv1x1_ws.cuh)
    B2C_PW1X1WS("fused_1x1ws_m64", 4, 2, 16, 4),
    B2C_PW1X1WS("fused_1x1ws_m128", 8, 1, 16, 4),
    // TMA-fed pointwise families (conv1x1_tma.cuh)
    B2C_PW1X1TMA("fused_1x1t_m64", 2, 4, 16, 3),
    B2C_PW1X1TMA("fused_1x1t_m128", 4, 2, 16, 3),
    B2C_PW1X1TMA("fused_1x1t_m64p128", 2, 2, 16, 3),
};
constexpr int kNumFamilies = sizeof(kFamilies) / sizeof(kFamilies[0]);

int g_sm_count = -1;
std::mutex g_mu;
bool g_attr_done[kNumFamilies][64] = {};
std::unordered_map<long long, int> g_cluster_ok;  // (family, splits, device) -> cluster launch feasible

int sm_count_of(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_sm_count > 0) return g_sm_count;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
  g_sm_count = n;
  return n;
}

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

// Rows of the virtual padded image stack needed by the worst tile.
int max_tile_rows(const Geom &g, int hf_eff, int bp) {
  const long long tiles = cdiv(g.Q, bp);
  int worst = 0;
  for (long long t = 0; t < tiles; t++) {
    const long long qa = t * bp;
    const long long qb = std::min<long long>(qa + bp, g.Q) - 1;
    const long long na = qa / g.HoWo, nb = qb / g.HoWo;
    const long long ya = (qa - na * g.HoWo) / g.Wo, yb = (qb - nb * g.HoWo) / g.Wo;
    const long long rows = (nb * g.Hp + yb * g.S) - (na * g.Hp + ya * g.S) + hf_eff;
    worst = (int)std::max<long long>(worst, rows);
  }
  return worst;
}

// conv_row_ws_kernel shared layout: [barriers: 128 B][goff: XCS ints][gtab: XCS/4]
// padded to 128 B, then the stages (also where a DSMEM split-C tile is parked).
long long ws_tile_offset(int xcs) { return 128 + ((4LL * (xcs + (xcs >> 2)) + 127) & ~127LL); }

// Row-segment kernel: rows of the virtual padded image stack spanned by the
// worst tile of `seg` segments (nb segments per output row).
int max_tile_rows_seg(const Geom &g, int nb, int seg) {
  const long long segs = (long long)g.N * g.Ho * nb;
  const long long tiles = cdiv(segs, seg);
  int worst = 0;
  for (long long t = 0; t < tiles; t++) {
    const long long ra = t * seg / nb;
    const long long rb = (std::min<long long>((t + 1) * seg, segs) - 1) / nb;
    const long long va = (ra / g.Ho) * g.Hp + (ra % g.Ho) * g.S;
    const long long vb = (rb / g.Ho) * g.Hp + (rb % g.Ho) * g.S;
    worst = (int)std::max<long long>(worst, vb - va + g.HF);
  }
  return worst;
}

// Row stride of the row-segment kernel's band: >= rc, spreading the 32
// segment origins of a warp over the 32 banks (scalar pixel loads: one
// wavefront when all origins differ mod 32).  Stride 1: == W (mod 4), so every
// band row stays 16-byte congruent with its global row (16-byte staging).
// Stride >= 2: consecutive output rows are S band rows apart, and with RS == W
// (mod 4) and W % 4 == 0 the origins crowd into a few banks (5-way on ResNet
// 28->14), so any residue is allowed (rows then stage by 4-byte copies), the
// congruent one winning ties.  Scored on the first warps of a sample of tiles.
int pick_row_stride(const Geom &g, int rc, int nb, int rx, int seg) {
  const long long segs = (long long)g.N * g.Ho * nb;
  const long long tiles = cdiv(segs, seg);
  const int congruent = rc + (((g.W - rc) % 4) + 4) % 4;
  const int step = g.S == 1 ? 4 : 1;
  int best_rs = congruent, best_score = INT_MAX;
  for (int rs = g.S == 1 ? congruent : rc; rs < congruent + 64; rs += step) {
    int score = 0;
    for (long long t = 0; t < std::min<long long>(tiles, 16); t++) {
      const long long tt = t * std::max<long long>(1, tiles / 16);
      const long long s0 = tt * seg;
      const long long r0 = s0 / nb;
      const long long v0 = (r0 / g.Ho) * g.Hp + (r0 % g.Ho) * g.S;
      for (int w = 0; w < seg / 32; w++) {
        int cnt[32] = {0};
        int worst = 0;
        for (int l = 0; l < 32; l++) {
          const long long sg = std::min(s0 + 32 * w + l, segs - 1);
          const long long r = sg / nb, b = sg - r * nb;
          const long long v = (r / g.Ho) * g.Hp + (r % g.Ho) * g.S;
          const int bank = (int)(((v - v0) * rs + b * rx * g.S) % 32);
          worst = std::max(worst, ++cnt[bank]);
        }
        score += worst;
      }
    }
    score = 2 * score + ((rs - congruent) % 4 != 0 ? 1 : 0);  // ties: keep 16-byte staging
    if (score < best_score) {
      best_score = score;
      best_rs = rs;
    }
  }
  return best_rs;
}

struct Candidate {
  int family = -1;
  TileChoice tc;
  double cost = 1e300;
};

// Relative time of one launch in "FMA-equivalents at full SM rate".  Models
// wave quantisation over the SMs, the per-SM warp count needed to saturate
// the FMA pipes, halo/filter staging, a fixed per-CTA prologue and the split-C
// partial traffic.  (Coefficients fitted on B200 timings of the BASELINE
// layers.)
double model_cost(const Geom &g, const TileChoice &tc, int taps, bool stage1, int sms, int max_blocks) {
  // the halo-staged kernel on a 1x1 filter issues 4 LDS.128 + 4 LDS.32 per 32
  // FFMA2 against the pointwise kernels' 4 LDS.128 (measured: the pointwise
  // families win every 1x1 layer with H*W % 4 == 0 they can run, tuned_plans.json)
  double lds_penalty = (!stage1 && tc.kind == 0 && taps == 1) ? 1.25 : 1.0;
  // row segments: the FMA pipe, not the shared-memory crossbar, bounds them
  if (tc.kind == 3) lds_penalty = 0.85;
  if (tc.kind == 4) lds_penalty = 0.8;  // no CTA-wide barriers in the channel loop
  // persistent pointwise: measured on par with the 16-byte pointwise families on
  // stride-1 planes, ahead on strided / 4-byte-staged ones (profiles/ab/r2_pointwise_ws_ab.txt)
  if (tc.kind == 5) lds_penalty = (g.S == 1 && (long long)g.H * g.W % 4 == 0) ? 1.15 : 0.9;
  if (tc.kind == 6) lds_penalty = 0.95;  // no per-thread staging, no CTA-wide barrier
  const double fma = (double)tc.bm * tc.bp * taps * tc.bc * tc.chunks_per_split * (stage1 ? 2.0 : 1.0) * lds_penalty;
  const double per_elem = (tc.kind == 1 || tc.kind == 9 || (tc.kind == 5 && g.S == 1 && (long long)g.H * g.W % 4 == 0) || ((long long)g.H * g.W % 4 == 0 && (tc.kind == 0 || tc.kind >= 3))) ? 2.0 : 6.0;  // 16-byte groups vs 4-byte copies
  const double loads = (per_elem * tc.tile_elems + 4.0 * tc.bm * taps) * tc.bc * tc.chunks_per_split;
  const double fixed = 250000.0 + 12.0 * tc.tile_elems;
  const double split_io = tc.splits > 1 ? (double)tc.bm * tc.bp * 24.0 : 0.0;  // partial store per CTA
  const double work = fma + loads + fixed + split_io;
  const long long ctas = tc.grid * tc.splits * tc.grid_z;
  const int occ = std::max(1, std::min(max_blocks, tc.occupancy));
  const double warps = tc.threads / 32.0;
  auto eff = [&](int k) { return std::min(1.0, k * warps / 12.0); };
  double t;
  if (tc.kind == 5) {  // persistent: one CTA per SM walks the items, no per-item pipeline fill
    t = (fma + loads + split_io) * (double)cdiv(ctas, sms) + fixed;
  } else if (ctas <= (long long)sms * occ) {
    const int k = (int)cdiv(ctas, sms);
    t = work * k / eff(k);
  } else {
    const double waves = (double)cdiv(ctas, (long long)sms * occ);
    t = waves * work * occ / eff(occ);
  }
  double reduce = 0.0;  // stage-2 style sum of the split planes: launch + 2*(splits+1) plane passes
  if (tc.splits > 1)
    reduce = 1.5e6 + 2.0 * (tc.splits + 1) * (double)g.N * g.M * g.HoWo * 4.0 * 168.0 / 40.0 / sms;
  return t + reduce + 2.0e6;  // launch + ramp
}

// packed pointwise (kind 9): bytes of x'[C][qp] at the start of the workspace (partials follow)
long long packed_bytes(const Geom &g) { return (4LL * g.C * ((g.Q + 3) & ~3LL) + 255) & ~255LL; }

bool evaluate(const Geom &g, int fam_id, bool stage1, int sms, int forced_splits, bool allow_split,
              Candidate *out) {
  const Family &f = kFamilies[fam_id];
  const int hf_eff = stage1 ? 1 : g.HF;
  const int wf_eff = stage1 ? 1 : g.WF;
  const int taps = hf_eff * wf_eff;
  TileChoice base;
  base.family = fam_id;
  base.bm = f.bm;
  base.bp = f.bp;
  base.bc = f.bc;
  base.threads = f.threads;
  base.kind = f.kind;
  if (f.kind == 9 && !allow_split) return false;  // needs a workspace for the packed pixels
  if (f.kind == 1 || f.kind == 2 || f.kind == 5 || f.kind == 6 || f.kind == 9) {
    base.rs = g.W;
    base.rows = 1;
    base.tile_elems = f.bp;
    base.xcs = f.bp;
    const long long mtiles = cdiv(g.M, f.bm);
    base.grid = mtiles * cdiv(g.Q, f.bp);
    base.grid_z = 1;
    const int nchunks = (int)cdiv(g.C, f.bc);
    Candidate best;
    const int auto_opts[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
    const int forced_opts[] = {forced_splits};
    const int *opts = forced_splits > 0 ? forced_opts : auto_opts;
    const int nopts = forced_splits > 0 ? 1 : (int)(sizeof(auto_opts) / sizeof(int));
    for (int oi = 0; oi < nopts; oi++) {
      const int sp = opts[oi];
      if (sp > 1 && !allow_split) break;
      if (sp > nchunks) {
        if (forced_splits > 0) return false;
        break;
      }
      TileChoice tc = base;
      tc.chunks_per_split = (int)cdiv(nchunks, sp);
      tc.splits = (int)cdiv(nchunks, tc.chunks_per_split);
      if (tc.splits != sp && forced_splits <= 0) continue;
      tc.stages = f.stages;
      long long smem = 4LL * f.stages * ((long long)f.bc * f.bp + (long long)f.bc * (f.bm + 4));
      if (f.kind == 2) smem = std::max(smem, 4LL * f.bm * f.bp);  // epilogue transposes the tile in smem
      if (f.kind == 5)  // barriers | ST x (filter tile | pixel tile)
        smem = 128 + 4LL * f.stages * ((long long)f.bm * f.bc + (long long)f.bc * f.bp);
      if (f.kind == 6)  // barriers | ST x (filter tile [BM][BC+4] | two pixel boxes [BC][BP])
        smem = 128 + 4LL * f.stages * ((long long)f.bm * (f.bc + 4) + 2LL * f.bc * f.bp);
      if (smem > 226 * 1024) return false;
      tc.smem_bytes = (int)smem;
      const int by_smem = std::max(1, (int)((228LL * 1024) / (smem + 1024)));
      tc.occupancy = std::max(1, std::min({f.max_ctas_per_sm, by_smem, 2048 / f.threads}));
      tc.ws_bytes = tc.splits > 1 ? 4LL * tc.splits * g.N * g.M * g.HoWo : 0;
      tc.cost = model_cost(g, tc, 1, false, sms, tc.occupancy) * ((f.kind == 1 || f.kind == 9) && f.tm == 2 ? 1.12 : 1.0);
      if (f.kind == 9) {  // + the packing pass: read the (strided) input rows, write x'[C][qp]
        const long long qp = (g.Q + 3) & ~3LL;
        tc.ws_bytes += packed_bytes(g);
        const double moved = 4.0 * g.C * ((double)g.N * g.Ho * (g.S == 1 ? g.H / (double)g.Ho : 1.0) * g.W + qp);
        tc.cost += 1.5e6 + 0.03 * moved;
      }
      if (f.kind >= 5) tc.stages = f.stages;
      if (tc.cost < best.cost) {
        best.family = fam_id;
        best.tc = tc;
        best.cost = tc.cost;
      }
    }
    if (best.family < 0) return false;
    *out = best;
    return true;
  }
  long long ptiles;
  if (f.kind == 3 || f.kind == 4) {
    const int nb = (int)cdiv(g.Wo, f.rx);
    const long long segs = (long long)g.N * g.Ho * nb;
    const int seg = f.bp / f.rx;
    if (segs + seg >= INT_MAX) return false;
    const int rc = (nb * f.rx - 1) * g.S + g.WF;
    base.rs = pick_row_stride(g, rc, nb, f.rx, seg);
    base.rows = max_tile_rows_seg(g, nb, seg);
    base.tile_elems = rc * base.rows;
    ptiles = cdiv(segs, seg);
  } else {
    const int rc = (g.Wo - 1) * g.S + wf_eff;
    base.rs = rc + (((g.W - rc) % 4) + 4) % 4;  // == W (mod 4): rows stay 16B-congruent with global rows
    base.rows = max_tile_rows(g, hf_eff, f.bp);
    base.tile_elems = rc * base.rows;
    ptiles = cdiv(g.Q, f.bp);
  }
  const long long positions = (long long)base.rs * base.rows + 3;
  if (positions > kFdivLimit || (long long)g.Hp + base.rows >= kFdivLimit) return false;
  base.xcs = (int)((positions + 3) & ~3LL);
  // relative offsets inside a tile must fit int32 (goff table)
  const long long imgs = cdiv(f.bp, g.HoWo) + 2;
  if (imgs * (long long)g.C * g.H * g.W >= INT_MAX) return false;
  const long long mtiles = cdiv(g.M, f.bm);
  base.grid = mtiles * ptiles;
  base.grid_z = stage1 ? g.HF * g.WF : 1;
  const int nchunks = (int)cdiv(g.C, f.bc);

  Candidate best;
  const int auto_opts[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
  const int forced_opts[] = {forced_splits};
  const int *opts = forced_splits > 0 ? forced_opts : auto_opts;
  const int nopts = forced_splits > 0 ? 1 : (int)(sizeof(auto_opts) / sizeof(int));
  for (int oi = 0; oi < nopts; oi++) {
    const int sp = opts[oi];
    if (sp > 1 && (stage1 || !allow_split)) break;
    if (sp > nchunks) {
      if (forced_splits > 0) return false;
      break;
    }
    TileChoice tc = base;
    tc.chunks_per_split = (int)cdiv(nchunks, sp);
    tc.splits = (int)cdiv(nchunks, tc.chunks_per_split);
    if (tc.splits != sp && forced_splits <= 0) continue;  // duplicate of a smaller split
    tc.stages = tc.chunks_per_split > 1 ? 2 : 1;
    const long long stage_floats = (long long)f.bc * tc.xcs + (long long)f.bc * taps * (f.bm + 4);
    const long long tables = tc.xcs + (((tc.xcs >> 2) + 3) & ~3);
    long long smem = 4LL * (tables + tc.stages * stage_floats);
    if (f.kind == 4) {  // conv_row_ws_kernel layout: barriers | tables | ST x (filter tile | band)
      tc.stages = f.stages;
      const long long wfloats = (long long)f.bm * f.bc * taps;
      const long long xfl = ((long long)f.bc * tc.xcs + 31) & ~31LL;
      smem = ws_tile_offset(tc.xcs) + 4LL * f.stages * (wfloats + xfl);
    }
    if (smem > 226 * 1024) return best.family >= 0 ? (*out = best, true) : false;
    tc.smem_bytes = (int)smem;
    const int by_smem = std::max(1, (int)((228LL * 1024) / (smem + 1024)));
    const int by_threads = 2048 / f.threads;
    tc.occupancy = std::max(1, std::min({f.max_ctas_per_sm, by_smem, by_threads}));
    tc.ws_bytes = tc.splits > 1 ? 4LL * tc.splits * g.N * g.M * g.HoWo : 0;
    tc.cost = model_cost(g, tc, taps, stage1, sms, tc.occupancy);
    if (tc.cost < best.cost) {
      best.family = fam_id;
      best.tc = tc;
      best.cost = tc.cost;
    }
  }
  if (best.family < 0) return false;
  *out = best;
  return true;
}

}  // namespace

// mbarrier watchdog of the tensor-core kernels: B2C_WATCHDOG_MS > 0 makes a
// stalled wait trap after that long (the test suite sets it so a protocol bug
// cannot hang the GPU); default 0 = unbounded waits (preemption-safe).
unsigned long long watchdog_ns() {
  static const unsigned long long ns = [] {
    const char *e = std::getenv("B2C_WATCHDOG_MS");
    const long long ms = e ? std::atoll(e) : 0;
    return ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
  }();
  return ns;
}

bool pdl_enabled() {
#ifdef B2C_DEV
  static const bool on = std::getenv("B2C_NO_PDL") == nullptr;
#else
  static const bool on = true;
#endif
  return on;
}

// Split-C through DSMEM clusters is opt-in (B2C_CLUSTER=1): measured on B200 it
// loses to partial planes + stage 2 (C2 26.1 vs 29.9 TFLOP/s; 4e-1x1 65.9 vs
// 45.8 us) because cross-CTA DSMEM reads run at ~20 B/clk per SM, so parking a
// 32-64 KB tile costs more than the L2-resident partial planes.
bool cluster_reduce_enabled() {
#ifdef B2C_DEV
  static const bool on = std::getenv("B2C_CLUSTER") != nullptr;
#else
  static const bool on = false;
#endif
  return on;
}

// Resident CTAs per SM of a kernel at a given dynamic shared memory size
// (cached per family, size and device).
int resident_ctas(int family, const void *kernel, int threads, int smem, int dev) {
  static std::unordered_map<long long, int> cache;
  const long long key = (((long long)family * 64 + dev) << 20) + smem;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, (size_t)smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cache[key] = n;
  return n;
}

const char *family_name(int id) {
  if (id < 0 || id >= kNumFamilies) return "invalid";
  return kFamilies[id].name;
}

int num_families() { return kNumFamilies; }

// Every quantity the kernels divide with fdiv (pixel offsets within an image
// plus one tile, virtual rows within an image plus a tile's band) stays below
// 2^20, where the magic division is exact (conv_kernel.cuh).
bool fdiv_range_ok(const Geom &g) {
  return (long long)g.HoWo + 4096 < kFdivLimit && (long long)g.Hp + 4096 < kFdivLimit;
}

bool family_matches(int fam_id, const Geom &g, bool stage1) {
  if (fam_id < 0 || fam_id >= kNumFamilies) return false;
  if (!fdiv_range_ok(g)) return false;
  const Family &f = kFamilies[fam_id];
  if (f.strict != stage1) return false;
  if (f.kind == 1)
    return g.HF == 1 && g.WF == 1 && g.S == 1 && g.PH == 0 && g.PW == 0 && ((long long)g.H * g.W) % 4 == 0;
  if (f.kind == 2)
    return g.HF == 1 && g.WF == 1 && g.PH == 0 && g.PW == 0 && (g.S != 1 || ((long long)g.H * g.W) % 4 != 0) &&
           (long long)g.N * g.C * g.H * g.W < (1LL << 31);
  if (f.kind == 9)  // where the 16-byte kernel cannot read x in place; fdiv-exact pixel indices
    return !stage1 && g.HF == 1 && g.WF == 1 && g.PH == 0 && g.PW == 0 &&
           (g.S != 1 || ((long long)g.H * g.W) % 4 != 0) && g.Q + 4 < kFdivLimit && g.C <= 65535;
  if (stage1) return g.S == 1;
  if (f.kind == 3 || f.kind == 4)
    return f.hf == g.HF && f.wf == g.WF && f.s == g.S && (long long)g.N * g.Ho * g.Wo < (1LL << 30);
  if (f.kind == 6)  // TMA boxes: 16-byte global strides, a tile spans at most two images
    return g.HF == 1 && g.WF == 1 && g.S == 1 && g.PH == 0 && g.PW == 0 && ((long long)g.H * g.W) % 4 == 0 &&
           g.C % 4 == 0 && g.HoWo >= f.bp && g.N < (1 << 30);
  if (f.kind == 5)  // gather offsets relative to a tile's first image stay in int32
    return g.HF == 1 && g.WF == 1 && g.PH == 0 && g.PW == 0 &&
           (cdiv(f.bp, g.HoWo) + 2) * (long long)g.C * g.H * g.W < INT_MAX;
  if (f.hf == 0) return true;  // generic
  return f.hf == g.HF && f.wf == g.WF && f.s == g.S;
}

int device_sm_count(int device) { return sm_count_of(device); }

bool family_has_cluster_epilogue(int fam_id) {
  return fam_id >= 0 && fam_id < kNumFamilies && !kFamilies[fam_id].strict &&
         (kFamilies[fam_id].kind < 3 || kFamilies[fam_id].kind == 4);
}

// Measured plans ("find" results of tools/autotune.py, registered at import by
// the Python package): exact (shape, engine) -> (family, splits).
struct TunedKey {
  int v[11];
  bool operator==(const TunedKey &o) const { return std::memcmp(v, o.v, sizeof(v)) == 0; }
};
struct TunedHash {
  size_t operator()(const TunedKey &k) const {
    size_t h = 1469598103934665603ULL;
    for (int x : k.v) h = (h ^ (size_t)(unsigned)x) * 1099511628211ULL;
    return h;
  }
};
struct TunedPlan {
  int family = -1, splits = 0, reduce = 0;
};
std::unordered_map<TunedKey, TunedPlan, TunedHash> g_tuned;
std::mutex g_tuned_mu;

TunedKey tuned_key(const Geom &g, bool stage1) {
  return TunedKey{{g.N, g.C, g.H, g.W, g.M, g.HF, g.WF, g.S, g.PH, g.PW, stage1 ? 1 : 0}};
}

void register_tuned(const Geom &g, bool stage1, int family, int splits, int reduce) {
  std::lock_guard<std::mutex> lk(g_tuned_mu);
  TunedPlan t;
  t.family = family;
  t.splits = splits;
  t.reduce = reduce;
  g_tuned[tuned_key(g, stage1)] = t;
}

// Planner: returns false if no family can run the geometry.
namespace {
bool plan_tiles_core(const Geom &g, bool stage1, int device, int forced_family, int forced_splits, bool allow_split,
                     bool allow_vec, TileChoice *out, int *tuned_reduce, bool need_cluster) {
  const int sms = sm_count_of(device);
  Candidate best;
  if (forced_family < 0 && forced_splits <= 0) {
    TunedPlan t;
    {
      std::lock_guard<std::mutex> lk(g_tuned_mu);
      auto it = g_tuned.find(tuned_key(g, stage1));
      if (it != g_tuned.end()) t = it->second;
    }
    if (t.family >= 0 && (allow_split || t.splits <= 1) && (allow_vec || (kFamilies[t.family].kind != 1 && kFamilies[t.family].kind != 6)) &&
        (!need_cluster || family_has_cluster_epilogue(t.family)) &&
        family_matches(t.family, g, stage1) &&
        evaluate(g, t.family, stage1, sms, t.splits, allow_split, &best)) {
      *out = best.tc;
      *tuned_reduce = t.reduce;
      return true;
    }
  }
  if (forced_family >= 0) {
    if (!family_matches(forced_family, g, stage1)) return false;
    if (!evaluate(g, forced_family, stage1, sms, forced_splits, allow_split, &best)) return false;
    *out = best.tc;
    return true;
  }
  for (int pass = 0; pass < 2 && best.family < 0; pass++) {
    for (int i = 0; i < kNumFamilies; i++) {
      const Family &f = kFamilies[i];
      if (!family_matches(i, g, stage1)) continue;
      if (!allow_vec && (f.kind == 1 || f.kind == 6)) continue;  // need 16-byte aligned operands
      if (need_cluster && !family_has_cluster_epilogue(i)) continue;
      const bool generic = (f.hf == 0) && !stage1;
      if ((pass == 0) == generic) continue;  // specialised families first
      Candidate c;
      if (!evaluate(g, i, stage1, sms, forced_splits, allow_split, &c)) continue;
      if (c.cost < best.cost * 0.999 ||
          (c.cost <= best.cost * 1.001 && best.family >= 0 && kFamilies[i].bm > kFamilies[best.family].bm))
        best = c;
    }
  }
  if (best.family < 0) return false;
  *out = best.tc;
  return true;
}
}  // namespace

// Split-C reduction mode: forced by the caller, else the tuned plan's, else
// partial planes + stage 2 (B2C_CLUSTER=1 makes DSMEM clusters the default).
// Clusters hold at most 16 CTAs and need the tile [BM][BP] in shared memory.
bool plan_tiles(const Geom &g, bool stage1, int device, int forced_family, int forced_splits, bool allow_split,
                bool allow_vec, TileChoice *out, int forced_reduce) {
  int tuned_reduce = 0;
  if (!plan_tiles_core(g, stage1, device, forced_family, forced_splits, allow_split, allow_vec, out, &tuned_reduce,
                       forced_reduce == 2 && forced_family < 0))
    return false;
  int r = 0;
  if (out->splits > 1 && !stage1) {
    r = forced_reduce > 0 ? forced_reduce : (tuned_reduce > 0 ? tuned_reduce : (cluster_reduce_enabled() ? 2 : 1));
    // row-segment tiles are contiguous output pixels only when RX divides Wo
    const bool seg_contig = kFamilies[out->family].kind != 4 || g.Wo % kFamilies[out->family].rx == 0;
    if (r == 2 && (out->splits > 16 || !family_has_cluster_epilogue(out->family) || !seg_contig)) {
      if (forced_reduce == 2) return false;
      r = 1;
    }
  }
  out->reduce = r;
  if (r == 2) {
    // the parked tile starts at shared offset 0, except in conv_row_ws_kernel,
    // which parks it in its stage memory behind the barriers and halo tables
    const long long tile_bytes = 4LL * out->bm * out->bp + (kFamilies[out->family].kind == 4 ? ws_tile_offset(out->xcs) : 0);
    if (tile_bytes > 226 * 1024) {
      if (forced_reduce == 2) return false;
      out->reduce = 1;
    } else {
      out->smem_bytes = (int)std::max<long long>(out->smem_bytes, tile_bytes);
    }
  }
  return true;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda),
// resolved once; nullptr if the driver lacks it.
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn tensor_map_encoder() {
  static const EncodeFn encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeFn>(fn);
  }();
  return encode;
}

// 2-D tensor map of the filter bank viewed as [M][C*hf*wf] (row-major, fp32)
// for conv_row_ws_kernel's per-stage TMA tile {BC*hf*wf, BM}.  false when TMA
// cannot address it (row pitch not a multiple of 16 bytes, unaligned base, a
// box dimension above 256): the kernel then stages filters by cp.async.
bool encode_filter_map(CUtensorMap *map, const Geom &g, const float *w, int bm, int bc, int extra_cols = 0) {
  const EncodeFn encode = tensor_map_encoder();
  const long long row = (long long)g.C * g.HF * g.WF;
  const int box0 = bc * g.HF * g.WF + extra_cols;
  if (!encode || (row * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(w) & 15) != 0 || box0 > 256 || bm > 256 ||
      (box0 * 4) % 16 != 0)
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)row, (cuuint64_t)g.M};
  const cuuint64_t strides[1] = {(cuuint64_t)(row * 4)};
  const cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)bm};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(w), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D tensor map of the input viewed as [N][C][H*W] for conv1x1_tma_kernel's
// pixel boxes {BP, BC, 1} (out-of-range pixels and channels zero-filled).
bool encode_input_map(CUtensorMap *map, const Geom &g, const float *x, int bp, int bc) {
  const EncodeFn encode = tensor_map_encoder();
  const long long hw = (long long)g.H * g.W;
  if (!encode || (hw * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0 || bp > 256 || bc > 256)
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)hw, (cuuint64_t)g.C, (cuuint64_t)g.N};
  const cuuint64_t strides[2] = {(cuuint64_t)(hw * 4), (cuuint64_t)(hw * 4 * g.C)};
  const cuuint32_t box[3] = {(cuuint32_t)bp, (cuuint32_t)bc, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(x), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_direct(const Geom &g, const TileChoice &tc, const float *x, const float *w, float *y,
                          bool stage1, long long y_tap_stride, void *workspace, cudaStream_t stream) {
  const Family &f = kFamilies[tc.family];
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 64 && !g_attr_done[tc.family][dev]) {
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, f.kernel);
      if (e != cudaSuccess) return e;
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      if (optin <= 0) optin = 227 * 1024;
      e = cudaFuncSetAttribute(f.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               optin - (int)fa.sharedSizeBytes);
      if (e != cudaSuccess) return e;
      // full shared-memory carveout: the planner's occupancy assumes 228 KB per SM
      e = cudaFuncSetAttribute(f.kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
      if (!f.strict) {  // split-C clusters of up to 16 CTAs (non-portable above 8)
        e = cudaFuncSetAttribute(f.kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
      }
      g_attr_done[tc.family][dev] = true;
    }
  }
  KParams p;
  std::memset(&p, 0, sizeof(p));
  p.x = x;
  p.w = w;
  p.y = y;
  p.N = g.N; p.C = g.C; p.H = g.H; p.W = g.W; p.M = g.M;
  p.S = g.S;
  p.HF = stage1 ? 1 : g.HF;
  p.WF = stage1 ? 1 : g.WF;
  p.PH = g.PH; p.PW = g.PW;
  p.Ho = g.Ho; p.Wo = g.Wo; p.HoWo = g.HoWo;
  p.Hp = g.Hp;
  p.Q = (int)g.Q;
  p.RS = tc.rs;
  p.RC = (g.Wo - 1) * g.S + (stage1 ? 1 : g.WF);
  CUtensorMap wmap;
  std::memset(&wmap, 0, sizeof(wmap));
  if (f.kind == 4 || f.kind == 5) p.w_tma = encode_filter_map(&wmap, g, w, tc.bm, tc.bc) ? 1 : 0;
  if (f.kind == 4 && g.C == tc.bc) {
    // one chunk holding every channel: each tile's filter rows are one contiguous
    // block, moved by a single bulk copy when 16-byte sized and aligned (conv1: C = 3)
    const long long row_bytes = 4LL * g.C * g.HF * g.WF;
    const bool aligned = (reinterpret_cast<uintptr_t>(w) & 15) == 0 && (tc.bm * row_bytes) % 16 == 0 &&
                         (g.M % tc.bm == 0 || ((g.M % tc.bm) * row_bytes) % 16 == 0);
    if (aligned) p.w_tma = 2;
  }
  CUtensorMap xmap;
  std::memset(&xmap, 0, sizeof(xmap));
  if (f.kind == 6 && !(encode_filter_map(&wmap, g, w, tc.bm, tc.bc, 4) && encode_input_map(&xmap, g, x, tc.bp, tc.bc)))
    return cudaErrorNotSupported;  // the planner only offers kind 6 where both maps encode
  p.spin_limit = watchdog_ns();
  if (f.kind == 3 || f.kind == 4) {
    p.nb = (int)cdiv(g.Wo, f.rx);
    p.segs = (int)((long long)g.N * g.Ho * p.nb);
    p.RC = (p.nb * f.rx - 1) * g.S + g.WF;
  }
  p.ROWS = tc.rows;
  p.XCS = tc.xcs;
  p.vec_ok = ((long long)g.H * g.W % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  p.mtiles = (int)cdiv(g.M, tc.bm);
  p.ptiles = (int)(tc.grid / p.mtiles);
  p.nchunks = (int)cdiv(g.C, tc.bc);
  p.splits = tc.splits;
  p.chunks_per_split = tc.splits > 1 ? tc.chunks_per_split : p.nchunks;
  if (tc.splits > 1) {
    if (!workspace) return cudaErrorInvalidValue;
    p.partials = reinterpret_cast<float *>(static_cast<char *>(workspace) + (f.kind == 9 ? packed_bytes(g) : 0));
    p.part_stride = (long long)g.N * g.M * g.HoWo;
  }
  p.w_ctaps = g.HF * g.WF;
  p.wf_full = g.WF;
  p.y_tap_stride = y_tap_stride;
  p.strict_tap_major = stage1 ? 1 : 0;
  p.mRS = fdiv_magic(tc.rs);
  p.mHp = fdiv_magic(g.Hp);
  p.mHoWo = fdiv_magic(g.HoWo);
  p.mWo = fdiv_magic(g.Wo);
  p.pdl = pdl_enabled() ? 1 : 0;
  if (f.kind == 9) {  // pack the (strided) pixels into x'[C][qp], then convolve x'
    if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15)) return cudaErrorInvalidValue;
    p.qp = (int)((g.Q + 3) & ~3LL);
    float *xp = static_cast<float *>(workspace);
    note_launch();
    pack_pixels_kernel<<<dim3((unsigned)cdiv(p.qp / 4, 256), (unsigned)g.C), 256, 0, stream>>>(p, x, xp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    p.x = xp;
  }
  dim3 grid((unsigned)tc.grid, (unsigned)tc.splits, (unsigned)tc.grid_z);
  // development tracing (-DB2C_DEV builds): per-CTA SM id and start/end globaltimer to a CSV file
#ifdef B2C_DEV
  const char *trace_file = std::getenv("B2C_TRACE_FILE");
#else
  const char *trace_file = nullptr;
#endif
  const long long nctas = tc.grid * tc.splits * tc.grid_z;
  unsigned long long *trace = nullptr;
  if (trace_file && cudaMalloc(&trace, sizeof(unsigned long long) * 5 * nctas) == cudaSuccess) p.trace = trace;
  // split-C through DSMEM: the splits of one output tile launch as a cluster
  // (at most 16 CTAs; the cluster must fit the GPU)
  int smem = tc.smem_bytes;
  if (!stage1 && !f.strict && tc.splits > 1 && tc.splits <= 16 && tc.reduce == 2) {
    const int tile_bytes = tc.bm * tc.bp * (int)sizeof(float) + (f.kind == 4 ? (int)ws_tile_offset(tc.xcs) : 0);
    const int csmem = std::max(smem, tile_bytes);
    const long long key = ((((long long)tc.family * 32 + tc.splits) * 64 + dev) << 18) + csmem;
    int ok = -1;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_cluster_ok.find(key);
      if (it != g_cluster_ok.end()) ok = it->second;
    }
    if (ok < 0) {
      cudaLaunchConfig_t qc = {};
      qc.gridDim = grid;
      qc.blockDim = dim3(tc.threads);
      qc.dynamicSmemBytes = (size_t)csmem;
      cudaLaunchAttribute ca[1];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = 1;
      ca[0].val.clusterDim.y = (unsigned)tc.splits;
      ca[0].val.clusterDim.z = 1;
      qc.attrs = ca;
      qc.numAttrs = 1;
      int nclusters = 0;
      ok = (cudaOccupancyMaxActiveClusters(&nclusters, f.kernel, &qc) == cudaSuccess && nclusters > 0) ? 1 : 0;
      cudaGetLastError();  // a refused query is not a launch error
      std::lock_guard<std::mutex> lk(g_mu);
      g_cluster_ok[key] = ok;
    }
    if (ok) {
      p.cluster = 1;
      smem = csmem;
    }
  }
  // pointwise kernels storing float4 outside a cluster: persistent grid of one
  // wave of resident CTAs walking the work items (conv1x1_vec.cuh)
  p.vec_out = (g.HoWo % 4 == 0) && ((reinterpret_cast<uintptr_t>(y) & 15) == 0) &&
              (tc.splits <= 1 || ((reinterpret_cast<uintptr_t>(p.partials) & 15) == 0));
  // Measured on B200 (profiles/ab/r2_persist_ab.txt): the persistent grid is
  // 2-9 % SLOWER than one work item per CTA on every ResNet-50 / GoogLeNet
  // pointwise layer — the hardware CTA scheduler balances the tail and keeps
  // the channel tiles of a pixel tile co-resident (L2 reuse) better than a
  // static item stride — so it stays a development option.
  bool persist = false;
#ifdef B2C_DEV
  if (const char *e = std::getenv("B2C_PERSIST")) persist = !p.cluster && (f.kind == 1 || (f.kind == 2 && p.vec_out)) && std::atoi(e);
  if (std::getenv("B2C_KIND2_TRANSPOSE")) p.vec_out = 0;
#endif
  if (f.kind == 5) {  // persistent: one CTA per SM walks the (split, tile) items
    grid = dim3((unsigned)std::max<long long>(1, std::min<long long>(tc.grid * tc.splits, sm_count_of(dev))), 1, 1);
  } else if (persist) {
    const long long items = tc.grid * tc.splits;
    const long long slots = (long long)sm_count_of(dev) * resident_ctas(tc.family, f.kernel, tc.threads, smem, dev);
    grid = dim3((unsigned)std::max<long long>(1, std::min(items, slots)), 1, 1);
  }
  void *args[] = {&p, &wmap, &xmap};  // the maps are read by kinds 4-6 only
  note_launch();
  cudaError_t err;
  if (p.pdl || p.cluster) {
    // programmatic dependent launch: this grid's prologue may overlap the tail of
    // the previous kernel on the stream (the kernel waits before reading inputs)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(tc.threads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      na++;
    }
    if (p.cluster) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = 1;
      attr[na].val.clusterDim.y = (unsigned)tc.splits;
      attr[na].val.clusterDim.z = 1;
      na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    err = cudaLaunchKernelExC(&cfg, f.kernel, args);
  } else {
    err = cudaLaunchKernel(f.kernel, grid, dim3(tc.threads), args, (size_t)smem, stream);
  }
  if (err == cudaSuccess && tc.splits > 1 && !stage1 && !p.cluster)
    err = launch_stage2(p.partials, y, p.part_stride, tc.splits, dev, stream);
  if (trace) {
    std::vector<unsigned long long> h(5 * nctas);
    cudaStreamSynchronize(stream);
    cudaMemcpy(h.data(), trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(trace);
    if (FILE *fp = std::fopen(trace_file, "a")) {
      for (long long i = 0; i < nctas; i++)
        std::fprintf(fp, "%s,%lld,%llu,%llu,%llu,%llu,%llu\n", f.name, i, h[5 * i], h[5 * i + 1], h[5 * i + 2],
                     h[5 * i + 3], h[5 * i + 4]);
      std::fclose(fp);
    }
  }
  return err;
}

cudaError_t launch_stage2(const float *partials, float *y, long long total, int taps, int device,
                          cudaStream_t stream) {
  const int sms = sm_count_of(device);
  const int vec = (total % 4 == 0) &&
                  ((reinterpret_cast<uintptr_t>(partials) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  const long long work = vec ? total / 4 : total;
  long long blocks = std::min<long long>(cdiv(work, 256), (long long)sms * 8);
  if (blocks < 1) blocks = 1;
  note_launch();
  const int pdl = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, stage2_sum_kernel, partials, y, total, taps, pdl, vec);
}

}  // namespace b2c
