// C ABI of the B200 forward-convolution engine (include/b2conv.h).
//
// Host-side responsibilities: the reference's preconditions and their order
// (twostage.py:73-79, 214-224), the reference planner's arithmetic for the
// drop-in RunStats / InvalidPlan contract (execmodel.py:73-128), the B200 tile
// plan cache, and host<->device staging for callers that hold host buffers.
#include "../../include/b2conv.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "internal.h"

namespace {

thread_local std::string t_last_error;
std::atomic<long long> g_launches{0};

b2c_status fail(b2c_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return st;
}

b2c_status cuda_fail(cudaError_t e, const char *what) {
  return fail(B2C_CUDA_ERROR, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

const char *kFieldNames[] = {"n", "c", "h", "w", "m", "hf", "wf", "stride", "pad_h", "pad_w"};

const int32_t *fields_of(const b2c_conv_desc *d) { return &d->n; }

b2c_status check_config(const b2c_conv_desc *d, int32_t *bad_field) {
  if (!d) return fail(B2C_INVALID_ARGUMENT, "null descriptor");
  const int32_t *f = fields_of(d);
  for (int i = 0; i < 8; i++) {
    if (f[i] < 1) {
      if (bad_field) *bad_field = i;
      return fail(B2C_INVALID_CONFIG, "%s: must be >= 1, got %d", kFieldNames[i], f[i]);
    }
  }
  for (int i = 8; i < 10; i++) {
    if (f[i] < 0) {
      if (bad_field) *bad_field = i;
      return fail(B2C_INVALID_CONFIG, "%s: must be >= 0, got %d", kFieldNames[i], f[i]);
    }
  }
  if ((long long)d->hf > (long long)d->h + 2LL * d->pad_h) {
    if (bad_field) *bad_field = 5;
    return fail(B2C_INVALID_CONFIG, "hf: filter height %d exceeds padded input height %lld", d->hf,
                (long long)d->h + 2LL * d->pad_h);
  }
  if ((long long)d->wf > (long long)d->w + 2LL * d->pad_w) {
    if (bad_field) *bad_field = 6;
    return fail(B2C_INVALID_CONFIG, "wf: filter width %d exceeds padded input width %lld", d->wf,
                (long long)d->w + 2LL * d->pad_w);
  }
  return B2C_OK;
}

b2c::Geom geom_of(const b2c_conv_desc *d) {
  b2c::Geom g;
  g.N = d->n; g.C = d->c; g.H = d->h; g.W = d->w; g.M = d->m;
  g.HF = d->hf; g.WF = d->wf; g.S = d->stride; g.PH = d->pad_h; g.PW = d->pad_w;
  g.Ho = (d->h + 2 * d->pad_h - d->hf) / d->stride + 1;
  g.Wo = (d->w + 2 * d->pad_w - d->wf) / d->stride + 1;
  g.HoWo = g.Ho * g.Wo;
  g.Hp = d->h + 2 * d->pad_h;
  g.Wp = d->w + 2 * d->pad_w;
  g.Q = (long long)g.N * g.HoWo;
  return g;
}

b2c_status check_sizes(const b2c::Geom &g) {
  const long long in = (long long)g.N * g.C * g.H * g.W;
  const long long out = (long long)g.N * g.M * g.HoWo;
  if (g.Q >= (1LL << 31) || (long long)g.N * g.Hp + g.Hp >= (1LL << 31) || in >= (1LL << 40) || out >= (1LL << 40))
    return fail(B2C_UNSUPPORTED, "problem too large for the engine's index arithmetic");
  return B2C_OK;
}

b2c_device_model default_device() { return b2c_device_model{32, 128, 1024, 4}; }

b2c_status check_device(const b2c_device_model *dev) {
  const int32_t *f = &dev->warp_width;
  const char *names[] = {"warp_width", "line_bytes", "max_threads_per_block", "element_bytes"};
  for (int i = 0; i < 4; i++)
    if (f[i] < 1) return fail(B2C_INVALID_CONFIG, "%s: must be >= 1, got %d", names[i], f[i]);
  if (dev->line_bytes % dev->element_bytes != 0)
    return fail(B2C_INVALID_CONFIG, "line_bytes: %d not a multiple of element size %d", dev->line_bytes,
                dev->element_bytes);
  return B2C_OK;
}

// --------------------------------------------------------------- plan cache
struct PlanKey {
  b2c_conv_desc d;
  int stage1;
  int device;
  int forced;
  int forced_splits;
  int allow_split;
  int allow_vec;
  int forced_reduce;
  bool operator==(const PlanKey &o) const {
    return std::memcmp(&d, &o.d, sizeof(d)) == 0 && stage1 == o.stage1 && device == o.device && forced == o.forced &&
           forced_splits == o.forced_splits && allow_split == o.allow_split && allow_vec == o.allow_vec &&
           forced_reduce == o.forced_reduce;
  }
};
struct PlanKeyHash {
  size_t operator()(const PlanKey &k) const {
    size_t h = 1469598103934665603ULL;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(&k);
    for (size_t i = 0; i < sizeof(PlanKey); i++) h = (h ^ p[i]) * 1099511628211ULL;
    return h;
  }
};
std::mutex g_plan_mu;
std::unordered_map<PlanKey, b2c::TileChoice, PlanKeyHash> g_plans;

b2c_status get_tiles(const b2c_conv_desc *d, const b2c::Geom &g, bool stage1, int forced, int forced_splits,
                     bool allow_split, b2c::TileChoice *tc, bool allow_vec = true, int forced_reduce = 0) {
  int device = 0;
  cudaGetDevice(&device);
  PlanKey key;
  std::memset(&key, 0, sizeof(key));
  key.d = *d;
  key.stage1 = stage1;
  key.device = device;
  key.forced = forced;
  key.forced_splits = forced_splits;
  key.allow_split = allow_split;
  key.allow_vec = allow_vec;
  key.forced_reduce = forced_reduce;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
      *tc = it->second;
      return B2C_OK;
    }
  }
  if (!b2c::plan_tiles(g, stage1, device, forced, forced_splits, allow_split, allow_vec, tc, forced_reduce)) {
    if (forced >= 0 || forced_splits > 0 || forced_reduce > 0)
      return fail(B2C_INVALID_PLAN, "tile family %d (%s) / split %d / reduce %d cannot run this configuration",
                  forced, forced >= 0 ? b2c::family_name(forced) : "auto", forced_splits, forced_reduce);
    return fail(B2C_UNSUPPORTED, "no kernel family fits this configuration (shared-memory halo too large)");
  }
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plans[key] = *tc;
  return B2C_OK;
}

void export_tiles(const b2c::TileChoice &tc, b2c_tile_plan *out) {
  out->family = tc.family;
  out->bm = tc.bm;
  out->bp = tc.bp;
  out->bc = tc.bc;
  out->threads = tc.threads;
  out->stages = tc.stages;
  out->smem_rows = tc.rows;
  out->smem_row_stride = tc.rs;
  out->smem_bytes = tc.smem_bytes;
  out->grid = tc.grid * tc.splits * tc.grid_z;
  out->splits = tc.splits;
  out->workspace_bytes = tc.ws_bytes;
  out->reduce = tc.reduce;
}

b2c_status resolve_plan(const b2c_conv_desc *d, const b2c_launch_plan *plan, const b2c_device_model *dev,
                        b2c_launch_plan *resolved) {
  if (plan) {
    b2c_status st = b2c_validate_plan(d, dev, plan);
    if (st != B2C_OK) return st;
    *resolved = *plan;
    return B2C_OK;
  }
  b2c_status st = b2c_plan_launch(d, dev, resolved);
  if (st != B2C_OK) return st;
  return b2c_validate_plan(d, dev, resolved);
}

// The reference's precondition order for conv_twostage / stage1_scalar_prods:
// stride (Unsupported) -> [shape checks done by the caller] -> plan -> workspace.
b2c_status twostage_preconditions(const b2c_conv_desc *d, const b2c_launch_plan *plan, const b2c_device_model *dev,
                                  int64_t workspace_limit, b2c_launch_plan *resolved) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (d->stride != 1)
    return fail(B2C_UNSUPPORTED, "two-stage convolution requires stride 1, got %d", d->stride);
  st = resolve_plan(d, plan, dev, resolved);
  if (st != B2C_OK) return st;
  const int64_t need = b2c_workspace_bytes(d);
  if (need > workspace_limit)
    return fail(B2C_WORKSPACE_EXCEEDED, "workspace of %lld bytes exceeds limit of %lld bytes", (long long)need,
                (long long)workspace_limit);
  return B2C_OK;
}

void fill_stats(const b2c_conv_desc *d, const b2c_launch_plan &p, bool stage2, b2c_run_stats *s) {
  if (!s) return;
  s->stage1_tasks_run = p.blocks;
  s->filter_row_global_loads = p.blocks;
  s->stage2_invoked = stage2 ? 1 : 0;
  s->workspace_bytes = stage2 ? b2c_workspace_bytes(d) : 0;
}

b2c_status run_stage1(const b2c_conv_desc *d, const b2c::Geom &g, const float *x, const float *w, float *out,
                      cudaStream_t stream) {
  b2c::TileChoice tc;
  b2c_status st = get_tiles(d, g, true, -1, 0, false, &tc);
  if (st != B2C_OK) return st;
  cudaError_t e = b2c::launch_direct(g, tc, x, w, out, true, (long long)g.N * g.M * g.HoWo, nullptr, stream);
  if (e != cudaSuccess) return cuda_fail(e, "stage-1 launch");
  return B2C_OK;
}

// ------------------------------------------------------ host staging cache
// slots: 0 x, 1 w, 2 y, 3 two-stage partial planes, 4 split-C partial planes
struct DeviceBuffers {
  void *ptr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t cap[5] = {0, 0, 0, 0, 0};
  cudaStream_t stream = nullptr;
};
thread_local std::unordered_map<int, DeviceBuffers> t_bufs;

b2c_status ensure(DeviceBuffers &b, int slot, size_t bytes) {
  if (bytes == 0) bytes = 4;
  if (b.cap[slot] >= bytes) return B2C_OK;
  if (b.ptr[slot]) cudaFree(b.ptr[slot]);
  b.ptr[slot] = nullptr;
  b.cap[slot] = 0;
  cudaError_t e = cudaMalloc(&b.ptr[slot], bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  b.cap[slot] = bytes;
  return B2C_OK;
}

b2c_status select_device(int32_t device, DeviceBuffers **out) {
  if (device >= 0) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  }
  int cur = 0;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  DeviceBuffers &b = t_bufs[cur];
  if (!b.stream) {
    e = cudaStreamCreateWithFlags(&b.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
  }
  *out = &b;
  return B2C_OK;
}

b2c_status sync_and_check(cudaStream_t s, const char *what) {
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, what);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  return B2C_OK;
}

}  // namespace

namespace b2c {
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace b2c

extern "C" {

int32_t b2c_abi_version(void) { return B2C_ABI_VERSION; }
const char *b2c_last_error(void) { return t_last_error.c_str(); }
const char *b2c_family_name(int32_t family) { return b2c::family_name(family); }
int32_t b2c_num_families(void) { return b2c::num_families(); }
int64_t b2c_launch_count(void) { return g_launches.load(); }
void b2c_reset_launch_count(void) { g_launches.store(0); }

b2c_status b2c_validate_config(const b2c_conv_desc *d, int32_t *bad_field) { return check_config(d, bad_field); }

b2c_status b2c_output_dims(const b2c_conv_desc *d, int32_t *ho, int32_t *wo) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (ho) *ho = (d->h + 2 * d->pad_h - d->hf) / d->stride + 1;
  if (wo) *wo = (d->w + 2 * d->pad_w - d->wf) / d->stride + 1;
  return B2C_OK;
}

int64_t b2c_workspace_bytes(const b2c_conv_desc *d) {
  if (!d) return -1;
  if (d->hf == 1 && d->wf == 1) return 0;
  const int64_t ho = (d->h + 2 * d->pad_h - d->hf) / d->stride + 1;
  const int64_t wo = (d->w + 2 * d->pad_w - d->wf) / d->stride + 1;
  return 4LL * d->hf * d->wf * d->n * d->m * ho * wo;
}

b2c_status b2c_plan_launch(const b2c_conv_desc *d, const b2c_device_model *dev, b2c_launch_plan *out) {
  if (!d || !out) return fail(B2C_INVALID_ARGUMENT, "null argument");
  if (d->stride != 1) return fail(B2C_UNSUPPORTED, "launch planning covers stride 1, got %d", d->stride);
  const b2c_device_model dm = dev ? *dev : default_device();
  b2c_status st = check_device(&dm);
  if (st != B2C_OK) return st;
  const int64_t ho = (d->h + 2 * d->pad_h - d->hf) / d->stride + 1;
  const int64_t wo = (d->w + 2 * d->pad_w - d->wf) / d->stride + 1;
  const int64_t work = (int64_t)d->n * ho * wo;
  const int64_t maxt = dm.max_threads_per_block, warp = dm.warp_width;
  const int64_t split = (work + maxt - 1) / maxt;
  int64_t threads = work < maxt ? work : maxt;
  threads = (threads + warp - 1) / warp * warp;
  if (threads > maxt) {
    // device limit not a warp multiple: largest warp multiple under it
    threads = maxt / warp * warp;
    if (threads < warp) threads = warp;
    if (threads > maxt) threads = maxt;
  }
  out->blocks = (int64_t)d->m * d->hf * d->wf * split;
  out->threads_per_block = (int32_t)threads;
  out->split_per_filter_row = (int32_t)split;
  out->dot_products_per_thread = (int32_t)((work + split * threads - 1) / (split * threads));
  return B2C_OK;
}

b2c_status b2c_validate_plan(const b2c_conv_desc *d, const b2c_device_model *dev, const b2c_launch_plan *p) {
  if (!d || !p) return fail(B2C_INVALID_ARGUMENT, "null argument");
  const b2c_device_model dm = dev ? *dev : default_device();
  const int64_t ho = (d->h + 2 * d->pad_h - d->hf) / d->stride + 1;
  const int64_t wo = (d->w + 2 * d->pad_w - d->wf) / d->stride + 1;
  const int64_t work = (int64_t)d->n * ho * wo;
  if (p->split_per_filter_row < 1)
    return fail(B2C_INVALID_PLAN, "split_per_filter_row must be >= 1, got %d", p->split_per_filter_row);
  const int64_t want_blocks = (int64_t)d->m * d->hf * d->wf * p->split_per_filter_row;
  if (p->blocks != want_blocks)
    return fail(B2C_INVALID_PLAN, "blocks %lld != m*hf*wf*split = %lld", (long long)p->blocks,
                (long long)want_blocks);
  if (p->threads_per_block < 1 || p->threads_per_block > dm.max_threads_per_block)
    return fail(B2C_INVALID_PLAN, "threads_per_block %d outside [1, %d]", p->threads_per_block,
                dm.max_threads_per_block);
  if (p->threads_per_block % dm.warp_width != 0)
    return fail(B2C_INVALID_PLAN, "threads_per_block %d not a multiple of warp width %d", p->threads_per_block,
                dm.warp_width);
  if (p->dot_products_per_thread < 1) return fail(B2C_INVALID_PLAN, "dot_products_per_thread must be >= 1");
  const long double covered = (long double)p->blocks * p->threads_per_block * p->dot_products_per_thread;
  const long double total = (long double)d->m * d->hf * d->wf * work;
  if (covered < total)
    return fail(B2C_INVALID_PLAN, "plan covers %.0Lf dot products, workload needs %.0Lf", covered, total);
  return B2C_OK;
}

b2c_status b2c_block_position_ranges(int64_t work, int64_t split, int64_t *lo_hi) {
  if (!lo_hi || split < 1) return fail(B2C_INVALID_ARGUMENT, "bad arguments");
  for (int64_t i = 0; i < split; i++) {
    lo_hi[2 * i] = i * work / split;
    lo_hi[2 * i + 1] = (i + 1) * work / split;
  }
  return B2C_OK;
}

b2c_status b2c_select_tiles(const b2c_conv_desc *d, int32_t engine, b2c_tile_plan *out) {
  if (!out) return fail(B2C_INVALID_ARGUMENT, "null argument");
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  if (engine == B2C_ENGINE_TWOSTAGE && d->stride != 1)
    return fail(B2C_UNSUPPORTED, "two-stage convolution requires stride 1, got %d", d->stride);
  if (out->reduce < 0 || out->reduce > 2) return fail(B2C_INVALID_ARGUMENT, "reduce must be 0, 1 or 2, got %d", out->reduce);
  b2c::TileChoice tc;
  st = get_tiles(d, g, engine == B2C_ENGINE_TWOSTAGE, out->family >= 0 ? out->family : -1,
                 out->splits > 0 ? out->splits : 0, true, &tc, true, out->reduce);
  if (st != B2C_OK) return st;
  export_tiles(tc, out);
  return B2C_OK;
}

b2c_status b2c_register_tuned_plan(const b2c_conv_desc *d, int32_t engine, int32_t family, int32_t splits,
                                   int32_t reduce) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  b2c::Geom g = geom_of(d);
  const bool stage1 = engine == B2C_ENGINE_TWOSTAGE;
  if (!b2c::family_matches(family, g, stage1))
    return fail(B2C_INVALID_PLAN, "family %d cannot run this configuration", family);
  if (reduce < 0 || reduce > 2) return fail(B2C_INVALID_ARGUMENT, "reduce must be 0, 1 or 2, got %d", reduce);
  if (reduce == 2 && !b2c::family_has_cluster_epilogue(family))
    return fail(B2C_INVALID_PLAN, "family %s has no DSMEM cluster reduction", b2c::family_name(family));
  b2c::register_tuned(g, stage1, family, splits, reduce);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plans.clear();  // cached plans may predate the registration
  return B2C_OK;
}

int32_t b2c_family_matches(const b2c_conv_desc *d, int32_t engine, int32_t family) {
  if (check_config(d, nullptr) != B2C_OK) return 0;
  return b2c::family_matches(family, geom_of(d), engine == B2C_ENGINE_TWOSTAGE) ? 1 : 0;
}

b2c_status b2c_conv2d_forward(const b2c_conv_desc *d, const float *x, const float *w, float *y, void *workspace,
                              int64_t workspace_size, const b2c_tile_plan *tiles, void *stream) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (!x || !w || !y) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  const int forced = (tiles && tiles->family >= 0) ? tiles->family : -1;
  const int forced_splits = (tiles && tiles->splits > 0) ? tiles->splits : 0;
  const int forced_reduce = (tiles && tiles->reduce > 0 && tiles->reduce <= 2) ? tiles->reduce : 0;
  b2c::TileChoice tc;
  st = get_tiles(d, g, false, forced, forced_splits, true, &tc, true, forced_reduce);
  if (st != B2C_OK) return st;
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                         reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(workspace)) & 15) == 0;
  const bool ws_ok = tc.ws_bytes == 0 || (workspace && workspace_size >= tc.ws_bytes);
  if (!ws_ok && (forced_splits > 1 || (forced >= 0 && tc.kind == 9)))
    return fail(B2C_INVALID_ARGUMENT, "plan %s split %d needs a %lld-byte workspace, %lld provided",
                b2c::family_name(tc.family), tc.splits, (long long)tc.ws_bytes, (long long)workspace_size);
  const bool needs_align = tc.kind == 1 || tc.kind == 6 || tc.kind == 9;
  if (needs_align && !aligned && forced >= 0)
    return fail(B2C_INVALID_ARGUMENT, "family %s needs 16-byte aligned x, w, y and workspace", b2c::family_name(forced));
  if (!ws_ok || (needs_align && !aligned)) {
    st = get_tiles(d, g, false, forced, ws_ok ? forced_splits : 0, ws_ok, &tc, aligned, forced_reduce);
    if (st != B2C_OK) return st;
  }
  cudaError_t e = b2c::launch_direct(g, tc, x, w, y, false, 0, workspace, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fused conv launch");
  return B2C_OK;
}

namespace {
b2c_status tc_plan_of(const b2c_conv_desc *d, const b2c::Geom &g, int32_t engine, int forced_nf, int forced_splits,
                      b2c::TcPlan *pl, int forced_mode = 0, int forced_mh = 0) {
  if (engine != B2C_ENGINE_TF32X3 && engine != B2C_ENGINE_TF32)
    return fail(B2C_INVALID_ARGUMENT, "engine %d is not a tensor-core engine", engine);
  if (forced_nf > 0 && (forced_nf % 16 != 0 || forced_nf > 256))
    return fail(B2C_INVALID_PLAN, "filters_per_tile must be a multiple of 16 in [16, 256], got %d", forced_nf);
  if (forced_splits < 0 || forced_splits > 64) return fail(B2C_INVALID_PLAN, "splits must be in [0, 64], got %d", forced_splits);
  if (forced_mode < 0 || forced_mode > 2) return fail(B2C_INVALID_PLAN, "mode must be 0, 1 or 2, got %d", forced_mode);
  if (forced_mh != 0 && forced_mh != 1 && forced_mh != 2 && forced_mh != 4)
    return fail(B2C_INVALID_PLAN, "m_halves must be 0, 1, 2 or 4, got %d", forced_mh);
  if (!b2c::plan_tc(g, engine == B2C_ENGINE_TF32X3 ? 3 : 1, forced_nf, 0, forced_splits, pl, forced_mode, forced_mh)) {
    if (forced_splits > 0 || forced_nf > 0 || forced_mode > 0 || forced_mh > 0)
      return fail(B2C_INVALID_PLAN, "forced tensor-core tile (filters %d, splits %d) cannot run this layer", forced_nf,
                  forced_splits);
    return fail(B2C_UNSUPPORTED, "layer too large for the tensor-core engine's 32-bit per-image offsets");
  }
  (void)d;
  return B2C_OK;
}
}  // namespace

b2c_status b2c_tc_select_tiles(const b2c_conv_desc *d, int32_t engine, b2c_tc_plan *out) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (!out) return fail(B2C_INVALID_ARGUMENT, "null plan");
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  b2c::TcPlan pl;
  if ((st = tc_plan_of(d, g, engine, out->filters_per_tile, out->splits, &pl, out->mode, out->m_halves)) != B2C_OK)
    return st;
  out->pixels_per_chunk = pl.xb;
  out->filters_per_tile = pl.nf;
  out->filter_tiles = pl.mtiles;
  out->stages = pl.stages;
  out->smem_bytes = pl.smem_bytes;
  out->tmem_columns = pl.tmem_cols;
  out->flattened = pl.flat ? 1 : 0;
  out->passes = pl.passes;
  out->grid = pl.grid;
  out->splits = pl.splits;
  out->workspace_bytes = b2c::tc_workspace_bytes(g, pl);
  out->mode = pl.halo > 0 ? 2 : 1;
  out->halo_positions = pl.halo;
  out->m_halves = pl.mh;
  out->bf16_corrections = pl.bf16corr ? 1 : 0;
  out->k_packed = pl.kpack ? 1 : 0;
  return B2C_OK;
}

b2c_status b2c_register_tuned_tc_plan(const b2c_conv_desc *d, int32_t engine, int32_t mode, int32_t filters_per_tile,
                                      int32_t splits, int32_t m_halves) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  b2c::Geom g = geom_of(d);
  b2c::TcPlan pl;
  if ((st = tc_plan_of(d, g, engine, filters_per_tile, splits, &pl, mode, m_halves)) != B2C_OK) return st;  // runnable
  b2c::register_tuned_tc(g, engine == B2C_ENGINE_TF32X3 ? 3 : 1, mode, filters_per_tile, splits, m_halves);
  return B2C_OK;
}

b2c_status b2c_conv2d_forward_tc(const b2c_conv_desc *d, const float *x, const float *w, float *y, void *workspace,
                                 int64_t workspace_size, int32_t engine, const b2c_tc_plan *tiles, void *stream) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (!x || !w || !y) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  b2c::TcPlan pl;
  if ((st = tc_plan_of(d, g, engine, tiles ? tiles->filters_per_tile : 0, tiles ? tiles->splits : 0, &pl,
                       tiles ? tiles->mode : 0, tiles ? tiles->m_halves : 0)) != B2C_OK)
    return st;
  if (!workspace || workspace_size < b2c::tc_workspace_bytes(g, pl))
    return fail(B2C_INVALID_ARGUMENT, "tensor-core engine needs a %lld-byte filter workspace, %lld provided",
                (long long)b2c::tc_workspace_bytes(g, pl), (long long)workspace_size);
  cudaError_t e = b2c::launch_tc(g, pl, x, w, y, workspace, workspace_size, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "tensor-core conv launch");
  return B2C_OK;
}

b2c_status b2c_stage1_scalar_prods(const b2c_conv_desc *d, const float *x, const float *w, float *partials,
                                   const b2c_launch_plan *plan, const b2c_device_model *dev,
                                   int64_t workspace_limit, void *stream, b2c_run_stats *stats) {
  b2c_launch_plan rp;
  b2c_status st = twostage_preconditions(d, plan, dev, workspace_limit, &rp);
  if (st != B2C_OK) return st;
  if (!x || !w || !partials) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  st = run_stage1(d, g, x, w, partials, (cudaStream_t)stream);
  if (st != B2C_OK) return st;
  if (stats) {
    fill_stats(d, rp, false, stats);
    stats->workspace_bytes = b2c_workspace_bytes(d);
  }
  return B2C_OK;
}

b2c_status b2c_stage2_sum(const b2c_conv_desc *d, const float *partials, float *y, void *stream,
                          b2c_run_stats *stats) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (!partials || !y) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  int device = 0;
  cudaGetDevice(&device);
  cudaError_t e = b2c::launch_stage2(partials, y, (long long)g.N * g.M * g.HoWo, g.HF * g.WF, device,
                                     (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "stage-2 launch");
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->stage2_invoked = 1;
  }
  return B2C_OK;
}

b2c_status b2c_conv_twostage(const b2c_conv_desc *d, const float *x, const float *w, float *y, float *workspace,
                             int64_t workspace_size, const b2c_launch_plan *plan, const b2c_device_model *dev,
                             int64_t workspace_limit, void *stream, b2c_run_stats *stats) {
  b2c_launch_plan rp;
  b2c_status st = twostage_preconditions(d, plan, dev, workspace_limit, &rp);
  if (st != B2C_OK) return st;
  if (!x || !w || !y) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  const bool one_by_one = d->hf == 1 && d->wf == 1;
  if (one_by_one) {
    // fused 1x1: stage 1 writes the output directly, no workspace (twostage.py:228-231)
    st = run_stage1(d, g, x, w, y, (cudaStream_t)stream);
    if (st != B2C_OK) return st;
  } else {
    const int64_t need = b2c_workspace_bytes(d);
    if (!workspace || workspace_size < need)
      return fail(B2C_INVALID_ARGUMENT, "workspace of %lld bytes required, %lld provided", (long long)need,
                  (long long)workspace_size);
    st = run_stage1(d, g, x, w, workspace, (cudaStream_t)stream);
    if (st != B2C_OK) return st;
    int device = 0;
    cudaGetDevice(&device);
    cudaError_t e = b2c::launch_stage2(workspace, y, (long long)g.N * g.M * g.HoWo, g.HF * g.WF, device,
                                       (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "stage-2 launch");
  }
  fill_stats(d, rp, !one_by_one, stats);
  return B2C_OK;
}

b2c_status b2c_conv_host(const b2c_conv_desc *d, const float *x_host, const float *w_host, float *y_host,
                         int32_t engine, const b2c_launch_plan *plan, const b2c_device_model *dev,
                         int64_t workspace_limit, int32_t device, b2c_run_stats *stats) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (engine < B2C_ENGINE_FUSED || engine > B2C_ENGINE_TF32)
    return fail(B2C_INVALID_ARGUMENT, "unknown engine %d", engine);
  const bool tensor_core = engine == B2C_ENGINE_TF32X3 || engine == B2C_ENGINE_TF32;
  if (!x_host || !w_host || !y_host) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c_launch_plan rp;
  if (engine == B2C_ENGINE_TWOSTAGE) {
    st = twostage_preconditions(d, plan, dev, workspace_limit, &rp);
    if (st != B2C_OK) return st;
  }
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  DeviceBuffers *b = nullptr;
  if ((st = select_device(device, &b)) != B2C_OK) return st;
  const size_t xb = sizeof(float) * (size_t)g.N * g.C * g.H * g.W;
  const size_t wb = sizeof(float) * (size_t)g.M * g.C * g.HF * g.WF;
  const size_t yb = sizeof(float) * (size_t)g.N * g.M * g.HoWo;
  const size_t wsb = engine == B2C_ENGINE_TWOSTAGE ? (size_t)b2c_workspace_bytes(d) : 0;
  size_t splitb = 0;
  if (engine == B2C_ENGINE_FUSED) {
    b2c::TileChoice tc;
    if ((st = get_tiles(d, g, false, -1, 0, true, &tc)) != B2C_OK) return st;
    splitb = (size_t)tc.ws_bytes;
  } else if (tensor_core) {
    b2c::TcPlan pl;
    if ((st = tc_plan_of(d, g, engine, 0, 0, &pl)) != B2C_OK) return st;
    splitb = (size_t)b2c::tc_workspace_bytes(g, pl);
  }
  if ((st = ensure(*b, 0, xb)) || (st = ensure(*b, 1, wb)) || (st = ensure(*b, 2, yb)) ||
      (wsb && (st = ensure(*b, 3, wsb))) || (splitb && (st = ensure(*b, 4, splitb))))
    return st;
  cudaError_t e = cudaMemcpyAsync(b->ptr[0], x_host, xb, cudaMemcpyHostToDevice, b->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(b->ptr[1], w_host, wb, cudaMemcpyHostToDevice, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "host-to-device copy");
  const float *dx = static_cast<const float *>(b->ptr[0]);
  const float *dw = static_cast<const float *>(b->ptr[1]);
  float *dy = static_cast<float *>(b->ptr[2]);
  if (engine == B2C_ENGINE_FUSED) {
    st = b2c_conv2d_forward(d, dx, dw, dy, splitb ? b->ptr[4] : nullptr, (int64_t)splitb, nullptr, b->stream);
    if (stats) std::memset(stats, 0, sizeof(*stats));
  } else if (tensor_core) {
    st = b2c_conv2d_forward_tc(d, dx, dw, dy, b->ptr[4], (int64_t)splitb, engine, nullptr, b->stream);
    if (stats) std::memset(stats, 0, sizeof(*stats));
  } else {
    st = b2c_conv_twostage(d, dx, dw, dy, static_cast<float *>(b->ptr[3]), (int64_t)wsb, &rp, dev,
                           workspace_limit, b->stream, stats);
  }
  if (st != B2C_OK) return st;
  e = cudaMemcpyAsync(y_host, dy, yb, cudaMemcpyDeviceToHost, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "device-to-host copy");
  return sync_and_check(b->stream, "convolution");
}

// Pipelined host-buffer path over a sequence of layers: slot i%3 holds layer
// i's device buffers; H2D copies (own stream), convolutions (own stream) and
// D2H copies (own stream) of consecutive layers overlap, ordered by events.
namespace {
struct Pipeline {
  static constexpr int kSlots = 6;  // in-flight layers: lets the H2D and D2H directions run ahead of each other (layer sizes alternate)
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t loaded[kSlots] = {}, computed[kSlots] = {}, drained[kSlots] = {};
  DeviceBuffers slot[kSlots];
  bool used[kSlots] = {};
};
thread_local std::unordered_map<int, Pipeline> t_pipes;

b2c_status pipeline_of(int32_t device, Pipeline **out) {
  if (device >= 0) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  }
  int cur = 0;
  cudaGetDevice(&cur);
  Pipeline &pl = t_pipes[cur];
  if (!pl.h2d) {
    cudaError_t e = cudaSuccess;
    for (cudaStream_t *st : {&pl.h2d, &pl.comp, &pl.d2h})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
    for (int i = 0; i < Pipeline::kSlots && e == cudaSuccess; i++) {
      for (cudaEvent_t *ev : {&pl.loaded[i], &pl.computed[i], &pl.drained[i]})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_fail(e, "pipeline setup");
  }
  *out = &pl;
  return B2C_OK;
}
}  // namespace

b2c_status b2c_conv_host_layers(int32_t count, const b2c_conv_desc *descs, const float *const *x_host,
                                const float *const *w_host, float *const *y_host, int32_t engine, int32_t device) {
  if (count < 0 || (count > 0 && (!descs || !x_host || !w_host || !y_host)))
    return fail(B2C_INVALID_ARGUMENT, "null layer arrays");
  if (engine != B2C_ENGINE_FUSED && engine != B2C_ENGINE_TF32X3 && engine != B2C_ENGINE_TF32)
    return fail(B2C_INVALID_ARGUMENT, "b2c_conv_host_layers runs the fused or tensor-core engines, got %d", engine);
  b2c_status st;
  for (int i = 0; i < count; i++) {
    if ((st = check_config(&descs[i], nullptr)) != B2C_OK) return st;
    if ((st = check_sizes(geom_of(&descs[i]))) != B2C_OK) return st;
    if (!x_host[i] || !w_host[i] || !y_host[i]) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer (layer %d)", i);
  }
  Pipeline *pl = nullptr;
  if ((st = pipeline_of(device, &pl)) != B2C_OK) return st;
  for (int i = 0; i < count; i++) {
    const b2c_conv_desc *d = &descs[i];
    const b2c::Geom g = geom_of(d);
    const int k = i % Pipeline::kSlots;
    DeviceBuffers &b = pl->slot[k];
    // the slot's previous layer must have drained before its buffers are reused
    if (pl->used[k]) {
      cudaError_t e = cudaEventSynchronize(pl->drained[k]);
      if (e != cudaSuccess) return cuda_fail(e, "pipeline drain");
    }
    const size_t xb = sizeof(float) * (size_t)g.N * g.C * g.H * g.W;
    const size_t wb = sizeof(float) * (size_t)g.M * g.C * g.HF * g.WF;
    const size_t yb = sizeof(float) * (size_t)g.N * g.M * g.HoWo;
    size_t wsb = 0;
    b2c::TileChoice tc;
    b2c::TcPlan tp;
    if (engine == B2C_ENGINE_FUSED) {
      if ((st = get_tiles(d, g, false, -1, 0, true, &tc)) != B2C_OK) return st;
      wsb = (size_t)tc.ws_bytes;
    } else {
      if ((st = tc_plan_of(d, g, engine, 0, 0, &tp)) != B2C_OK) return st;
      wsb = (size_t)b2c::tc_workspace_bytes(g, tp);
    }
    if ((st = ensure(b, 0, xb)) || (st = ensure(b, 1, wb)) || (st = ensure(b, 2, yb)) ||
        (wsb && (st = ensure(b, 4, wsb))))
      return st;
    cudaError_t e = cudaMemcpyAsync(b.ptr[0], x_host[i], xb, cudaMemcpyHostToDevice, pl->h2d);
    if (e == cudaSuccess) e = cudaMemcpyAsync(b.ptr[1], w_host[i], wb, cudaMemcpyHostToDevice, pl->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(pl->loaded[k], pl->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pl->comp, pl->loaded[k], 0);
    if (e != cudaSuccess) return cuda_fail(e, "host-to-device copy");
    const float *dx = static_cast<const float *>(b.ptr[0]);
    const float *dw = static_cast<const float *>(b.ptr[1]);
    float *dy = static_cast<float *>(b.ptr[2]);
    if (engine == B2C_ENGINE_FUSED)
      st = b2c_conv2d_forward(d, dx, dw, dy, wsb ? b.ptr[4] : nullptr, (int64_t)wsb, nullptr, pl->comp);
    else
      st = b2c_conv2d_forward_tc(d, dx, dw, dy, b.ptr[4], (int64_t)wsb, engine, nullptr, pl->comp);
    if (st != B2C_OK) return st;
    e = cudaEventRecord(pl->computed[k], pl->comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pl->d2h, pl->computed[k], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(y_host[i], dy, yb, cudaMemcpyDeviceToHost, pl->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(pl->drained[k], pl->d2h);
    if (e != cudaSuccess) return cuda_fail(e, "device-to-host copy");
    pl->used[k] = true;
  }
  for (cudaStream_t sv : {pl->h2d, pl->comp, pl->d2h})
    if ((st = sync_and_check(sv, "pipelined convolution")) != B2C_OK) return st;
  return B2C_OK;
}

b2c_status b2c_stage1_host(const b2c_conv_desc *d, const float *x_host, const float *w_host, float *partials_host,
                           const b2c_launch_plan *plan, const b2c_device_model *dev, int64_t workspace_limit,
                           int32_t device, b2c_run_stats *stats) {
  b2c_launch_plan rp;
  b2c_status st = twostage_preconditions(d, plan, dev, workspace_limit, &rp);
  if (st != B2C_OK) return st;
  if (!x_host || !w_host || !partials_host) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  if ((st = check_sizes(g)) != B2C_OK) return st;
  DeviceBuffers *b = nullptr;
  if ((st = select_device(device, &b)) != B2C_OK) return st;
  const size_t xb = sizeof(float) * (size_t)g.N * g.C * g.H * g.W;
  const size_t wb = sizeof(float) * (size_t)g.M * g.C * g.HF * g.WF;
  const size_t pb = sizeof(float) * (size_t)g.HF * g.WF * g.N * g.M * g.HoWo;
  if ((st = ensure(*b, 0, xb)) || (st = ensure(*b, 1, wb)) || (st = ensure(*b, 3, pb))) return st;
  cudaError_t e = cudaMemcpyAsync(b->ptr[0], x_host, xb, cudaMemcpyHostToDevice, b->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(b->ptr[1], w_host, wb, cudaMemcpyHostToDevice, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "host-to-device copy");
  st = run_stage1(d, g, static_cast<const float *>(b->ptr[0]), static_cast<const float *>(b->ptr[1]),
                  static_cast<float *>(b->ptr[3]), b->stream);
  if (st != B2C_OK) return st;
  e = cudaMemcpyAsync(partials_host, b->ptr[3], pb, cudaMemcpyDeviceToHost, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "device-to-host copy");
  if (stats) {
    fill_stats(d, rp, false, stats);
    stats->workspace_bytes = b2c_workspace_bytes(d);
  }
  return sync_and_check(b->stream, "stage 1");
}

b2c_status b2c_stage2_host(const b2c_conv_desc *d, const float *partials_host, float *y_host, int32_t device,
                           b2c_run_stats *stats) {
  b2c_status st = check_config(d, nullptr);
  if (st != B2C_OK) return st;
  if (!partials_host || !y_host) return fail(B2C_INVALID_ARGUMENT, "null tensor pointer");
  b2c::Geom g = geom_of(d);
  DeviceBuffers *b = nullptr;
  if ((st = select_device(device, &b)) != B2C_OK) return st;
  const size_t yb = sizeof(float) * (size_t)g.N * g.M * g.HoWo;
  const size_t pb = yb * (size_t)g.HF * g.WF;
  if ((st = ensure(*b, 2, yb)) || (st = ensure(*b, 3, pb))) return st;
  cudaError_t e = cudaMemcpyAsync(b->ptr[3], partials_host, pb, cudaMemcpyHostToDevice, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "host-to-device copy");
  st = b2c_stage2_sum(d, static_cast<const float *>(b->ptr[3]), static_cast<float *>(b->ptr[2]), b->stream, stats);
  if (st != B2C_OK) return st;
  e = cudaMemcpyAsync(y_host, b->ptr[2], yb, cudaMemcpyDeviceToHost, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "device-to-host copy");
  return sync_and_check(b->stream, "stage 2");
}

void *b2c_host_alloc(size_t bytes) {
  void *p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 4, cudaHostAllocPortable) != cudaSuccess) {
    fail(B2C_CUDA_ERROR, "cudaHostAlloc of %zu bytes failed", bytes);
    return nullptr;
  }
  return p;
}

void b2c_host_free(void *p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
