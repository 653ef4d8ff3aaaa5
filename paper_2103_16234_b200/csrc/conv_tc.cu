// Host side of the tcgen05 implicit-GEMM engine (conv_tc.cuh): tensor maps,
// tile planner and launch.  The tensor-map encoder is fetched from the driver
// through the runtime (cudaGetDriverEntryPoint), so libb2conv.so keeps linking
// only the static CUDA runtime.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <cstdio>

#include "conv_tc.cuh"
#include "internal.h"

namespace b2c {

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

const void *tc_kernel(int passes) {
  return passes == 3 ? reinterpret_cast<const void *>(&tc::conv_tc_kernel<3>)
                     : reinterpret_cast<const void *>(&tc::conv_tc_kernel<1>);
}

constexpr int kSmemBudget = 225 * 1024;  // dynamic smem per CTA incl. 1 KB alignment slack + barriers

}  // namespace

bool tc_flat(const Geom &g) { return g.HF == 1 && g.WF == 1 && g.S == 1 && g.PH == 0 && g.PW == 0; }

bool tc_supported(const Geom &g) {
  // chunk/tile indices and per-image offsets are 32-bit in the kernel's inner loops
  if ((long long)g.C * g.H * g.W >= (1LL << 31) || (long long)g.M * g.HoWo >= (1LL << 31)) return false;
  return true;  // the tensor-map encoder (needs a driver) is checked at launch
}

bool tc_needs_relayout(const Geom &g, const float *w) {
  return !(g.HF == 1 && g.WF == 1 && g.C % 4 == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0);
}

long long tc_workspace_bytes(const Geom &g) {
  const long long cp = (g.C + 3) / 4 * 4;
  return 4LL * g.HF * g.WF * g.M * cp;
}

bool plan_tc(const Geom &g, int passes, int forced_nf, int forced_xb, TcPlan *out) {
  if (!tc_supported(g)) return false;
  const bool flat = tc_flat(g);
  const int wo = flat ? g.HoWo : g.Wo;
  const int ho = flat ? 1 : g.Ho;
  // chunk shape: rc rows x xw columns (xw * rc = 32), least padded pixels, then widest
  int xw = 32;
  long long best_px = -1;
  for (int cand : {32, 16, 8}) {
    if (flat && cand != 32) break;
    if (forced_xb > 0 && cand != forced_xb) continue;
    const int rc = 32 / cand;
    const long long px = cdiv(wo, cand) * cand * cdiv(ho, rc) * rc;
    if (best_px < 0 || px < best_px) {
      best_px = px;
      xw = cand;
    }
  }
  if (best_px < 0) return false;
  const int rc = 32 / xw;
  const long long nchunks = (long long)g.N * cdiv(ho, rc) * cdiv(wo, xw);
  const long long ptiles = cdiv(nchunks, tc::TILE_P / 32);
  const int taps = g.HF * g.WF;
  const int cblocks = (int)cdiv(g.C, tc::BC);
  const int KB = cblocks * taps;
  const int sms = device_sm_count(0);
  TcPlan best;
  double best_cost = 1e300;
  for (int mt = 1; mt <= 64; mt++) {
    int nf = (int)cdiv(cdiv(g.M, mt), 16) * 16;
    if (nf > 256) continue;
    if (forced_nf > 0) nf = forced_nf;
    const int mtiles = (int)cdiv(g.M, nf);
    const long long stage = (long long)(tc::A_BYTES + nf * 64) * (passes == 3 ? 2 : 1);
    const int stages = (int)std::min<long long>(6, (kSmemBudget - 2048) / stage);
    if (stages < 2) continue;
    const long long ctas = ptiles * mtiles;
    // per-stage clocks: tensor (128 x nf x 8 UMMA ~ nf/2 clk, >= 16), smem and L2 feeds
    const double mma = passes * 2.0 * std::max(nf / 2.0, 16.0);
    const double l2 = (tc::A_BYTES + nf * 64) / 28.0;
    const double split = passes == 3 ? 2.0 * (tc::A_BYTES + nf * 64) / 128.0 : 0.0;
    const double t_cta = KB * std::max({mma, l2, split}) + 2500.0 + nf * 4.0;
    const double cost = (double)cdiv(ctas, sms) * t_cta;
    if (cost < best_cost) {
      best_cost = cost;
      best.xb = xw;
      best.nf = nf;
      best.mtiles = mtiles;
      best.stages = stages;
      best.stage_bytes = (int)stage;
      best.grid = ctas;
      best.passes = passes;
      best.flat = flat;
      best.nchunks = nchunks;
    }
    if (forced_nf > 0) break;
  }
  if (best.nf == 0) return false;
  int cols = 32;
  while (cols < best.nf) cols <<= 1;
  best.tmem_cols = cols;
  best.smem_bytes = best.stages * best.stage_bytes + 1024 /*align*/ + 256 /*barriers*/;
  best.cost = best_cost;
  *out = best;
  return true;
}

cudaError_t launch_tc(const Geom &g, const TcPlan &pl, const float *x, const float *w, float *y, void *workspace,
                      long long ws_bytes, cudaStream_t stream) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const float *wsrc = w;
  int cp = g.C;
  const int taps = g.HF * g.WF;
  if (tc_needs_relayout(g, w)) {
    cp = (g.C + 3) / 4 * 4;
    if (!workspace || ws_bytes < tc_workspace_bytes(g)) return cudaErrorInvalidValue;
    float *wp = static_cast<float *>(workspace);
    const long long total = (long long)taps * g.M * cp;
    const int blocks = (int)std::min<long long>(cdiv(total, 256), 4LL * device_sm_count(0));
    note_launch();
    tc::filter_relayout_kernel<<<blocks, 256, 0, stream>>>(w, wp, g.M, g.C, cp, taps);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    wsrc = wp;
  }

  tc::TcParams p;
  std::memset(&p, 0, sizeof(p));
  cuuint32_t ones[4] = {1, 1, 1, 1};
  const int rc = 32 / pl.xb;
  cuuint64_t wdim[3] = {(cuuint64_t)cp, (cuuint64_t)g.M, (cuuint64_t)taps};
  cuuint64_t wstr[2] = {(cuuint64_t)cp * 4, (cuuint64_t)cp * g.M * 4};
  cuuint32_t wbox[3] = {(cuuint32_t)tc::BC, (cuuint32_t)pl.nf, 1};
  CUresult r = enc(&p.wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(wsrc), wdim, wstr, wbox, ones,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;

  p.x = x;
  p.y = y;
  p.C = g.C;
  p.H = g.H;
  p.W = g.W;
  p.HW = g.H * g.W;
  p.S = g.S;
  p.flat = pl.flat ? 1 : 0;
  p.M = g.M;
  p.Wo = pl.flat ? g.HoWo : g.Wo;
  p.HoWo = g.HoWo;
  p.Ho = pl.flat ? 1 : g.Ho;
  p.xw = pl.xb;
  p.rc = rc;
  p.rgroups = (int)cdiv(p.Ho, rc);
  p.xblocks = (int)cdiv(p.Wo, pl.xb);
  p.nchunks = pl.nchunks;
  p.PH = g.PH;
  p.PW = g.PW;
  p.WF = g.WF;
  p.taps = taps;
  p.NF = pl.nf;
  p.mtiles = pl.mtiles;
  p.cblocks = (int)cdiv(g.C, tc::BC);
  p.stages = pl.stages;
  p.b_bytes = pl.nf * 64;
  p.stage_bytes = pl.stage_bytes;
  p.tmem_cols = pl.tmem_cols;
  // kind::tf32 instruction descriptor: D f32, A/B tf32, A MN-major (pixels), B K-major (filters)
  p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((uint32_t)(pl.nf >> 3) << 17) |
            ((uint32_t)(tc::TILE_P >> 4) << 24);
  p.spin_limit = 4000000000ull;  // 4 s

  const void *kern = tc_kernel(pl.passes);
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem_bytes);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pl.grid);
  cfg.blockDim = dim3(tc::THREADS);
  cfg.dynamicSmemBytes = (size_t)pl.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  // development dump (B2C_TC_DEBUG=path): timeout code, CTA-0 stage 0 and accumulator
  const char *dbg_file = std::getenv("B2C_TC_DEBUG");
  const size_t dbg_words = 16 + 65536 + 128 * 256;
  unsigned *dbg_host = nullptr;  // mapped pinned memory: readable even after a device trap
  if (dbg_file && cudaHostAlloc(reinterpret_cast<void **>(&dbg_host), dbg_words * 4, cudaHostAllocMapped) == cudaSuccess) {
    std::memset(dbg_host, 0, dbg_words * 4);
    cudaHostGetDevicePointer(reinterpret_cast<void **>(&p.dbg), dbg_host, 0);
  }
  void *args[] = {&p};
  note_launch();
  cudaError_t err = cudaLaunchKernelExC(&cfg, kern, args);
  if (p.dbg) {
    cudaError_t e2 = cudaStreamSynchronize(stream);
    dbg_host[1] = (unsigned)e2;
    if (FILE *fp = std::fopen(dbg_file, "wb")) {
      std::fwrite(dbg_host, 4, dbg_words, fp);
      std::fclose(fp);
    }
    if (e2 == cudaSuccess) cudaFreeHost(dbg_host);
    if (e2 != cudaSuccess) return e2;
  }
  return err;
}

}  // namespace b2c
