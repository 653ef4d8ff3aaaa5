// Host side of the tcgen05 implicit-GEMM engine (conv_tc.cuh): tile planner,
// per-call filter pre-tiling and launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <array>
#include <mutex>
#include <set>
#include <unordered_map>
#include <cstdio>

#include "conv_tc.cuh"
#include "internal.h"

namespace b2c {

namespace {

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

const void *tc_kernel(int passes, bool halo, int mh) {
  if (!halo && passes == 2) return reinterpret_cast<const void *>(&tc::conv_tc_kernel<2>);
  if (halo) {
    if (mh == 4)
      return passes == 3 ? reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<3, 4>)
           : passes == 2 ? reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<2, 4>)
                         : reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<1, 4>);
    if (mh == 2)
      return passes == 3 ? reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<3, 2>)
           : passes == 2 ? reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<2, 2>)
                         : reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<1, 2>);
    return passes == 3 ? reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<3, 1>)
         : passes == 2 ? reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<2, 1>)
                       : reinterpret_cast<const void *>(&tc::conv_tc_halo_kernel<1, 1>);
  }
  return passes == 3 ? reinterpret_cast<const void *>(&tc::conv_tc_kernel<3>)
                     : reinterpret_cast<const void *>(&tc::conv_tc_kernel<1>);
}

constexpr int kSmemBudget = 225 * 1024;  // dynamic smem per CTA incl. 1 KB alignment slack + barriers

}  // namespace

// 3xTF32 correction products as bf16 MMAs (halo mode).  Default on; B2C_TC_BF16CORR=0 disables.
bool bf16corr_enabled() {
#ifdef B2C_DEV
  static const bool on = [] {
    const char *e = std::getenv("B2C_TC_BF16CORR");
    return !(e && std::atoi(e) == 0);
  }();
#else
  static const bool on = true;
#endif
  return on;
}

bool tc_flat(const Geom &g) { return g.HF == 1 && g.WF == 1 && g.S == 1 && g.PH == 0 && g.PW == 0; }

bool tc_supported(const Geom &g) {
  // chunk/tile indices and per-image offsets are 32-bit in the kernel's inner loops
  if ((long long)g.C * g.H * g.W >= (1LL << 31) || (long long)g.M * g.HoWo >= (1LL << 31)) return false;
  return true;
}

long long tc_filter_bytes(const Geom &g, const TcPlan &pl) {
  const long long k = pl.kpack ? cdiv((long long)g.C * g.HF * g.WF, tc::BC) * tc::BC : cdiv(g.C, tc::BC) * tc::BC * g.HF * g.WF;
  const long long b = 4LL * k * (long long)pl.mtiles * pl.nf * pl.wplanes;
  return (b + 255) / 256 * 256;
}

long long tc_workspace_bytes(const Geom &g, const TcPlan &pl) {
  const long long partials = pl.splits > 1 ? 4LL * pl.splits * g.N * g.M * g.HoWo : 0;
  return tc_filter_bytes(g, pl) + partials;
}

// Measured plans (tools/autotune.py --engines tf32x3,tf32), registered at
// import by the Python package: exact (shape, passes) -> (mode, nf, splits).
namespace {
struct TcKey {
  int v[11];
  bool operator==(const TcKey &o) const { return std::memcmp(v, o.v, sizeof(v)) == 0; }
};
struct TcKeyHash {
  size_t operator()(const TcKey &k) const {
    size_t h = 1469598103934665603ULL;
    for (int x : k.v) h = (h ^ (size_t)(unsigned)x) * 1099511628211ULL;
    return h;
  }
};
std::unordered_map<TcKey, std::array<int, 4>, TcKeyHash> g_tc_tuned;
std::mutex g_tc_tuned_mu;
TcKey tc_key(const Geom &g, int passes) {
  return TcKey{{g.N, g.C, g.H, g.W, g.M, g.HF, g.WF, g.S, g.PH, g.PW, passes}};
}
}  // namespace

void register_tuned_tc(const Geom &g, int passes, int mode, int nf, int splits, int mh) {
  std::lock_guard<std::mutex> lk(g_tc_tuned_mu);
  g_tc_tuned[tc_key(g, passes)] = {mode, nf, splits, mh};
}

bool plan_tc(const Geom &g, int passes, int forced_nf, int forced_xb, int forced_splits, TcPlan *out,
             int forced_mode, int forced_mh) {
  if (!tc_supported(g)) return false;
  if (forced_nf <= 0 && forced_splits <= 0 && forced_mode <= 0 && forced_xb <= 0 && forced_mh <= 0) {
    std::array<int, 4> t{0, 0, 0, 0};
    bool hit = false;
    {
      std::lock_guard<std::mutex> lk(g_tc_tuned_mu);
      auto it = g_tc_tuned.find(tc_key(g, passes));
      if (it != g_tc_tuned.end()) {
        t = it->second;
        hit = true;
      }
    }
    if (hit && plan_tc(g, passes, t[1], 0, t[2], out, t[0], t[3])) return true;
  }
  const bool flat = tc_flat(g);
  const int wo = flat ? g.HoWo : g.Wo;
  const int ho = flat ? 1 : g.Ho;
  // gather mode: chunk shape rc rows x xw columns (xw * rc = 32), least padded pixels, then widest
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
  const int taps_geom = g.HF * g.WF;
  // K packing (gather mode): few input channels waste most of each 16-channel
  // k-block, so the reduction runs over (channel, tap) pairs instead
  const bool kpack = g.C < tc::BC && taps_geom > 1 && forced_mode != 2;
  const int taps = kpack ? 1 : taps_geom;
  const int cblocks = (int)cdiv((long long)g.C * (kpack ? taps_geom : 1), tc::BC);
  const int KB = cblocks * taps;
  const int sms = device_sm_count(0);
  // halo mode (stride 1): tiles over the flattened padded stack
  const bool halo_ok = g.S == 1 && forced_mode != 1 && !kpack;
  const long long Wp = (long long)g.W + 2 * g.PW, Hp = (long long)g.H + 2 * g.PH;

  TcPlan best;
  double best_cost = 1e300;
  // 3xTF32 accuracy: the tensor core accumulates with truncation, so the main
  // accumulator's error grows with its number of steps; keep <= 1152 products
  // (72 k-blocks of 16 channels) per split, the split partials being summed in
  // fp32 round-to-nearest (measured: within tol(K) up to K = 4608 with margin)
  const int max_kbps = passes == 3 ? 72 : 1 << 30;
  const double out_bytes = 4.0 * g.N * g.M * g.HoWo;
  const int planes = passes == 3 ? 2 : 1;
  // modes: 1 = gather; 2 / 3 / 4 = halo with 1 / 2 / 4 128-position M slices
  for (int mode = 1; mode <= 4; mode++) {
    const int mh = mode == 4 ? 4 : mode == 3 ? 2 : 1;
    if (forced_mode > 0 && (mode == 1) != (forced_mode == 1)) continue;
    if (forced_mh > 0 && mode >= 2 && mh != forced_mh) continue;  // halo M slices forced (1, 2 or 4)
    if (mode >= 2 && !halo_ok) continue;
    const long long halo = (tc::TILE_P * mh + (g.HF - 1) * Wp + (g.WF - 1) + 7) / 8 * 8;
    const long long ptiles = mode == 1 ? cdiv(nchunks, tc::TILE_P / 32) : cdiv((long long)g.N * Hp * Wp, tc::TILE_P * mh);
    for (int mt = 1; mt <= 64; mt++) {
      int nf = (int)cdiv(cdiv(g.M, mt), 16) * 16;
      if (nf > 256) continue;
      if (forced_nf > 0) nf = forced_nf;
      if (nf * mh * planes > 512) continue;  // TMEM: main (+ correction) accumulators of every M half
      const int mtiles = (int)cdiv(g.M, nf);
      const long long bstage = (long long)nf * 64 * planes;
      long long stage, smem_fixed;
      int stages, abufs = 0;
      if (mode == 1) {
        stage = (long long)tc::A_BYTES * planes + bstage;  // A + B (+ lo planes)
        smem_fixed = 0;
      } else {
        // filter ring (hi + lo) of `stages`; a ring of `abufs` staged halos,
        // deep enough that ~8 taps of work are in flight (1x1 layers: many
        // shallow channel blocks, 3x3/5x5: two suffice)
        stage = bstage;
        const long long abuf = halo * 64 * planes;
        abufs = (int)std::max<long long>(2, std::min<long long>(8, cdiv(8, taps)));
        while (abufs > 2 && abufs * abuf + 4 * stage > kSmemBudget - 2048) abufs--;
        smem_fixed = abufs * abuf;
      }
      stages = (int)std::min<long long>(mode == 1 ? 6 : 8, (kSmemBudget - 2048 - smem_fixed) / stage);
      if (smem_fixed + 2 * stage > kSmemBudget - 2048) continue;
      if (stages < 2) continue;
      static const int kAuto[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
      const int nopt = forced_splits > 0 ? 1 : (int)(sizeof(kAuto) / sizeof(int));
      for (int oi = 0; oi < nopt; oi++) {
        const int sp = forced_splits > 0 ? forced_splits : kAuto[oi];
        // halo mode splits whole channel blocks (all taps of a block in one CTA)
        const int units = mode == 1 ? KB : cblocks;
        if (sp > units) break;
        const int ups = (int)cdiv(units, sp);
        const int splits = (int)cdiv(units, ups);
        if (splits != sp && forced_splits <= 0) continue;  // duplicate of a smaller split
        const int kbps = mode == 1 ? ups : ups * taps;
        if (kbps > max_kbps && forced_splits <= 0 && !(mode >= 2 && ups == 1)) continue;
        const long long ctas = ptiles * mtiles * splits;
        // per-k-block clocks (B200 measurements): tensor issue ~95 clk per
        // 128x256x8 tf32 UMMA; gather mode adds a ~1.1-1.3k clk latency chain
        // per k-block, halo mode ~150 clk of barrier work per tap and one
        // double-buffered halo fill per channel block
        const bool bf16corr = passes == 3 && bf16corr_enabled();
        // tf32 MMA-equivalents per k-block and M half: 2 (main) [+ 4 tf32 or 2 bf16 corrections]
        const double mma_units = passes == 1 ? 2.0 : (bf16corr ? 4.0 : 6.0);
        const double mma = mma_units * mh * std::max(95.0 * nf / 256.0, 12.0);
        double t_cta;
        if (mode == 1) {
          t_cta = kbps * std::max(mma, passes == 3 ? 1300.0 : 1100.0);
        } else {
          // per tap: tensor issue, the L2 feed of the filter tile (~36 B/clk/SM
          // of the ~6.3 KB/clk chip L2 rate), ~150 clk of barrier work
          const double l2 = nf * 64.0 * planes / 36.0;  // hi (+ streamed lo) plane
          const double fill = 500.0 + halo * 10.0;  // measured ~2.4 clk per (position, 4-channel) item
          t_cta = ups * std::max(taps * (std::max(mma, l2) + 150.0), fill);
        }
        t_cta += 6000.0 + nf * 8.0;
        double cost = (double)cdiv(ctas, sms) * t_cta;
        if (splits > 1) cost += 4000.0 + 2.0 * (splits + 1) * out_bytes / (3.0e3 * sms / 148.0);  // stage-2 sum
        if (cost < best_cost) {
          best_cost = cost;
          best = TcPlan();
          best.xb = mode == 1 ? xw : 0;
          best.halo = mode >= 2 ? (int)halo : 0;
          best.mh = mh;
          best.abufs = abufs;
          best.wplanes = planes;  // filter lo plane streamed with the hi plane
          best.bf16corr = bf16corr;
          best.kpack = kpack;
          best.nf = nf;
          best.mtiles = mtiles;
          best.stages = stages;
          best.stage_bytes = (int)stage;
          best.grid = ctas;
          best.passes = passes;
          best.flat = flat;
          best.nchunks = mode == 1 ? nchunks : 0;
          best.splits = splits;
          best.kb_per_split = kbps;
          best.smem_bytes = (int)(stages * stage + smem_fixed) + 1024 /*align*/ + 512 /*barriers*/;
        }
      }
      if (forced_nf > 0) break;
    }
  }
  if (best.nf == 0) return false;
  int cols = 32;
  while (cols < best.nf * best.mh * (passes == 3 ? 2 : 1)) cols <<= 1;  // 3xTF32: main + correction
  best.tmem_cols = cols;
  best.cost = best_cost;
  *out = best;
  return true;
}

cudaError_t launch_tc(const Geom &g, const TcPlan &pl, const float *x, const float *w, float *y, void *workspace,
                      long long ws_bytes, cudaStream_t stream) {
  // K packing: filters [m][c][ky][kx] are already [m][k] with k = c*taps + tap,
  // so they pre-tile as a 1x1 layer over C*taps virtual channels
  const int taps = pl.kpack ? 1 : g.HF * g.WF;
  const int cvirt = pl.kpack ? g.C * g.HF * g.WF : g.C;
  const int cblocks = (int)cdiv(cvirt, tc::BC);
  const int Mp = pl.mtiles * pl.nf;
  if (!workspace || ws_bytes < tc_workspace_bytes(g, pl)) return cudaErrorInvalidValue;
  float *wt = static_cast<float *>(workspace);
  const int planes = pl.wplanes;
  // 3xTF32 in halo mode: correction products as bf16 MMAs (kernel PASSES 2) when the plan says so
  const int kpasses = (pl.passes == 3 && pl.bf16corr) ? 2 : pl.passes;
  if (kpasses == 2) {
    const long long total = (long long)cblocks * taps * Mp * tc::BC;
    const int blocks = (int)std::min<long long>(cdiv(total, 256), 8LL * device_sm_count(0));
    note_launch();
    tc::filter_tile_bf16corr_kernel<<<blocks, 256, 0, stream>>>(w, wt, g.M, cvirt, taps, pl.nf, pl.mtiles, cblocks);
  } else {
    const long long total = (long long)cblocks * taps * Mp * tc::BC * planes;
    const int blocks = (int)std::min<long long>(cdiv(total, 256), 8LL * device_sm_count(0));
    note_launch();
    tc::filter_tile_kernel<<<blocks, 256, 0, stream>>>(w, wt, g.M, cvirt, taps, pl.nf, pl.mtiles, cblocks, planes);
  }
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int rc = pl.xb > 0 ? 32 / pl.xb : 1;

  tc::TcParams p;
  std::memset(&p, 0, sizeof(p));
  p.wt = wt;
  p.Mp = Mp;
  const bool flat_chunks = pl.flat && pl.halo == 0;  // gather mode runs 1x1 over the flattened plane
  p.x = x;
  p.y = y;
  p.N = g.N;
  p.Hp = g.H + 2 * g.PH;
  p.Wp = g.W + 2 * g.PW;
  p.halo = pl.halo;
  p.mh = pl.mh;
  p.abufs = pl.abufs;
  p.C = g.C;
  p.H = g.H;
  p.W = g.W;
  p.HW = g.H * g.W;
  p.S = g.S;
  p.flat = flat_chunks ? 1 : 0;
  p.M = g.M;
  p.Wo = flat_chunks ? g.HoWo : g.Wo;
  p.HoWo = g.HoWo;
  p.Ho = flat_chunks ? 1 : g.Ho;
  p.xw = pl.xb > 0 ? pl.xb : 32;
  p.rc = rc;
  p.rgroups = (int)cdiv(p.Ho, rc);
  p.xblocks = (int)cdiv(p.Wo, p.xw);
  p.nchunks = pl.nchunks;
  p.PH = g.PH;
  p.PW = g.PW;
  p.WF = g.WF;
  p.taps = taps;
  p.kpack = pl.kpack ? 1 : 0;
  p.taps_full = g.HF * g.WF;
  p.NF = pl.nf;
  p.mtiles = pl.mtiles;
  p.cblocks = cblocks;
  p.stages = pl.stages;
  p.b_bytes = pl.nf * 64 * planes;
  p.stage_bytes = pl.stage_bytes;
  p.tmem_cols = pl.tmem_cols;
  p.splits = pl.splits;
  p.kb_per_split = pl.kb_per_split;
  if (pl.splits > 1) {
    p.partials = reinterpret_cast<float *>(static_cast<char *>(workspace) + tc_filter_bytes(g, pl));
    p.part_stride = (long long)g.N * g.M * g.HoWo;
  }
  // kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major
  p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(pl.nf >> 3) << 17) |
            ((uint32_t)(tc::TILE_P >> 4) << 24);
  p.spin_limit = watchdog_ns();
#ifdef B2C_DEV
  if (const char *m = std::getenv("B2C_TC_MODE")) p.mode = std::atoi(m);
#endif

  const void *kern = tc_kernel(kpasses, pl.halo > 0, pl.mh);
  // once per (kernel, device): allow the full opt-in shared memory, so launches
  // carry no attribute calls
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> attr_done;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!attr_done.count({kern, dev})) {
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, kern);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               std::max(pl.smem_bytes, optin - (int)fa.sharedSizeBytes));
      if (e != cudaSuccess) return e;
      attr_done.insert({kern, dev});
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(pl.grid / pl.splits), (unsigned)pl.splits);
  cfg.blockDim = dim3(tc::THREADS);
  cfg.dynamicSmemBytes = (size_t)pl.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  // development dump (-DB2C_DEV builds, B2C_TC_DEBUG=path): timeout code, CTA-0 stage 0 and accumulator
#ifdef B2C_DEV
  const char *dbg_file = std::getenv("B2C_TC_DEBUG");
#else
  const char *dbg_file = nullptr;
#endif
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
  // split-K: partial planes summed in ascending split order, fp32 round-to-nearest
  if (err == cudaSuccess && pl.splits > 1) {
    int dev = 0;
    cudaGetDevice(&dev);
    err = launch_stage2(p.partials, y, p.part_stride, pl.splits, dev, stream);
  }
  return err;
}

}  // namespace b2c
