/*
 * b2conv — B200-native fp32 forward convolution (cuConv, arXiv 2103.16234),
 * C ABI.  Everything crossing this boundary is POD: int32/int64 scalars,
 * plain structs, raw float pointers and an opaque stream handle.  No C++ or
 * torch types appear here.
 *
 * The reference (convkit 0.1.0, /root/reference/pkg/src/convkit) has no FFI of
 * its own; it is pure Python.  Each entry point below names the reference
 * interface it replaces (file:line), and INTEGRATION.md shows the ctypes
 * binding a reference maintainer would add.
 *
 * Conventions
 *  - Tensors are NCHW fp32, C-contiguous: input [n][c][h][w], filters
 *    [m][c][hf][wf], output [n][m][ho][wo] with ho = (h+2ph-hf)/stride+1
 *    (configs.py:60-64).  Cross-correlation, no dilation/groups/bias.
 *  - `y` is always fully overwritten, never accumulated into.
 *  - Device entry points are asynchronous on `stream` (a cudaStream_t; NULL =
 *    legacy default stream) and never allocate.  *_host entry points take host
 *    buffers and are synchronous.
 *  - Errors: a b2c_status is returned and a thread-local message is available
 *    from b2c_last_error().  The Python layer maps statuses onto the
 *    reference's exception classes (errors.py:9-61) in the reference's
 *    precedence: Unsupported(stride) -> ShapeMismatch -> InvalidPlan ->
 *    WorkspaceExceeded (twostage.py:73-79, 214-224).
 *  - Determinism: every engine is deterministic run to run
 *    (no atomics on data).  Each output's summation order is a function of
 *    (c, hf, wf) for the paper-faithful two-stage engine — bitwise
 *    independent of any plan — of (c, hf, wf) and the split-C channel ranges
 *    for the fused engine (ranges = split count x the family's channels per
 *    pipeline chunk; otherwise independent of the kernel family and of the
 *    split-C reduction mode), and of (mode, splits) for the tensor-core
 *    engines.  Images are independent, so a batch sharded across GPUs is
 *    bitwise identical to the unsharded result when each shard keeps the
 *    global plan's channel ranges (sharding.shard_layer pins them).
 */
#ifndef B2CONV_H
#define B2CONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2C_ABI_VERSION 1

/* == ConvConfig without its name (configs.py:17-40). */
typedef struct {
  int32_t n, c, h, w, m, hf, wf, stride, pad_h, pad_w;
} b2c_conv_desc;

typedef enum {
  B2C_OK = 0,
  B2C_UNSUPPORTED = 1,         /* errors.Unsupported (errors.py:41-42)          */
  B2C_SHAPE_MISMATCH = 2,      /* errors.ShapeMismatch (errors.py:45-46)        */
  B2C_INVALID_PLAN = 3,        /* errors.InvalidPlan (errors.py:49-50)          */
  B2C_WORKSPACE_EXCEEDED = 4,  /* errors.WorkspaceExceeded (errors.py:53-61)    */
  B2C_INVALID_CONFIG = 5,      /* errors.InvalidConfig (errors.py:29-34)        */
  B2C_CUDA_ERROR = 6,          /* a CUDA runtime failure (no reference analogue) */
  B2C_INVALID_ARGUMENT = 7     /* null pointer / bad enum (no reference analogue) */
} b2c_status;

/* == execmodel.DeviceModel (execmodel.py:36-56). */
typedef struct {
  int32_t warp_width, line_bytes, max_threads_per_block, element_bytes;
} b2c_device_model;

/* == execmodel.LaunchPlan (execmodel.py:59-66). */
typedef struct {
  int64_t blocks;
  int32_t threads_per_block, split_per_filter_row, dot_products_per_thread;
} b2c_launch_plan;

/* == twostage.RunStats (twostage.py:48-55); counts follow the reference's
 * launch-plan arithmetic so the reference's stat tests hold. */
typedef struct {
  int64_t stage1_tasks_run;
  int32_t stage2_invoked;
  int64_t filter_row_global_loads;
  int64_t workspace_bytes;
} b2c_run_stats;

/* The B200 tile plan chosen by the planner (no reference analogue: the
 * reference's model has one filter row per block; this is the real grid). */
typedef struct {
  int32_t family;       /* kernel family id, see b2c_family_name()          */
  int32_t bm;           /* output channels per CTA                          */
  int32_t bp;           /* output pixels per CTA (flattened n,y,x)          */
  int32_t bc;           /* input channels per pipeline stage                */
  int32_t threads;      /* threads per CTA                                  */
  int32_t stages;       /* cp.async pipeline depth                          */
  int32_t smem_rows;    /* halo rows staged per channel                     */
  int32_t smem_row_stride;
  int32_t smem_bytes;   /* dynamic shared memory per CTA                    */
  int64_t grid;         /* CTAs per launch                                  */
  int32_t splits;       /* fused: channel ranges reduced separately (split-C);
                           on input to b2c_select_tiles / b2c_conv2d_forward,
                           > 0 forces the split                              */
  int64_t workspace_bytes; /* workspace the plan needs: split-C partial planes
                              (splits > 1) and, for the packed-pixel pointwise
                              families (fused_1x1pk*), the packed input
                              4*C*ceil4(N*Ho*Wo) bytes; 0 otherwise          */
  int32_t reduce;       /* split-C reduction (splits > 1): 1 = partial planes in
                           the workspace + a stage-2 sum kernel, 2 = inside a
                           thread-block cluster through DSMEM (one kernel; same
                           ascending-order sum, bitwise identical).  On input
                           0 = planner's choice, 1 / 2 force a mode.          */
} b2c_tile_plan;

typedef enum {
  B2C_ENGINE_FUSED = 0,    /* single-pass FFMA2 direct convolution, no workspace,
                              within tol(K) = 1e-5*max(1,K/4096) of conv_naive_f64 */
  B2C_ENGINE_TWOSTAGE = 1, /* paper-faithful stage 1 + stage 2 with the
                              reference's separate-rounding order: bitwise equal
                              to conv_naive / conv_twostage                      */
  B2C_ENGINE_TF32X3 = 2,   /* tcgen05 tensor-core implicit GEMM, 3xTF32 operand
                              splitting (fp32-class: within tol(K) like FUSED)   */
  B2C_ENGINE_TF32 = 3      /* tcgen05 implicit GEMM, plain TF32 operands
                              (its own tolerance: 5e-3 relative)                 */
} b2c_engine;

/* Tile plan of the tensor-core engines (no reference analogue). */
typedef struct {
  int32_t pixels_per_chunk; /* chunk width (32, 16, 8): a chunk is 32 output
                               pixels = (32/width) rows x width columns      */
  int32_t filters_per_tile; /* UMMA N: output channels per CTA                */
  int32_t filter_tiles;
  int32_t stages;           /* TMA/mbarrier pipeline depth                     */
  int32_t smem_bytes;
  int32_t tmem_columns;
  int32_t flattened;        /* 1x1 layers: pixels flattened over the plane     */
  int32_t passes;           /* 3 (3xTF32) or 1 (TF32)                          */
  int64_t grid;             /* CTAs (128 output pixels x filters_per_tile each,
                               times splits)                                  */
  int32_t splits;           /* split-K over (16-channel block, tap) k-blocks;
                               partial planes summed by a second launch      */
  int64_t workspace_bytes;  /* pre-tiled filters (4*ceil(c/16)*16*hf*wf*filter_tiles
                               *filters_per_tile*passes' planes, rounded up to
                               256) + split-K partials (4*splits*n*m*ho*wo
                               when splits > 1)                               */
  int32_t mode;             /* in/out: 0 = planner's choice (in), 1 = gather
                               (loaders re-gather the tap-shifted input per
                               tap, any stride), 2 = halo (stride 1: one staged
                               padded-input halo per channel block, taps are
                               descriptor offsets)                            */
  int32_t halo_positions;   /* out: staged positions per tile (mode 2)        */
  int32_t m_halves;         /* in/out: 128-pixel UMMA M slices per tile (mode 2:
                               1, 2 or 4, sharing each filter tile); on input
                               0 = planner's choice, 1/2/4 force it for halo
                               plans                                          */
  int32_t bf16_corrections; /* out: 3xTF32 correction products run as bf16
                               MMAs (K=16, twice the tf32 rate)               */
  int32_t k_packed;         /* out: mode 1 with few input channels: the
                               reduction runs over ceil(c*hf*wf/16) blocks of
                               16 (channel, tap) pairs                        */
} b2c_tc_plan;

/* ---------------------------------------------------------------- metadata */
int32_t b2c_abi_version(void);
const char *b2c_last_error(void);
const char *b2c_family_name(int32_t family);
int32_t b2c_num_families(void);
/* 1 if kernel family `family` can run `d` under `engine` (used to enumerate
 * tile plans in plan-independence tests). */
int32_t b2c_family_matches(const b2c_conv_desc *d, int32_t engine, int32_t family);
/* Number of CUDA kernel launches issued by this thread since the last reset
 * (instrumentation used by bench.py's gpu_launches). */
int64_t b2c_launch_count(void);
void b2c_reset_launch_count(void);

/* ------------------------------------------------------ shape / plan logic */
/* ConvConfig.__post_init__ (configs.py:42-54); on failure *bad_field receives
 * the index of the offending field in b2c_conv_desc order (n=0 .. pad_w=9). */
b2c_status b2c_validate_config(const b2c_conv_desc *d, int32_t *bad_field);
/* configs.output_dims (configs.py:60-64). */
b2c_status b2c_output_dims(const b2c_conv_desc *d, int32_t *ho, int32_t *wo);
/* twostage.workspace_bytes (twostage.py:36-45): 4*hf*wf*n*m*ho*wo, 0 for 1x1. */
int64_t b2c_workspace_bytes(const b2c_conv_desc *d);
/* execmodel.plan_launch (execmodel.py:73-98).  dev may be NULL (defaults). */
b2c_status b2c_plan_launch(const b2c_conv_desc *d, const b2c_device_model *dev, b2c_launch_plan *out);
/* execmodel.validate_plan (execmodel.py:101-123). */
b2c_status b2c_validate_plan(const b2c_conv_desc *d, const b2c_device_model *dev, const b2c_launch_plan *p);
/* execmodel.block_position_ranges (execmodel.py:126-128): writes 2*split
 * int64 values lo0,hi0,lo1,hi1,... */
b2c_status b2c_block_position_ranges(int64_t work, int64_t split, int64_t *lo_hi);
/* B200 tile planner for the given engine ("launch planner picks the tile shape
 * per (filter size, channels, spatial size, batch)").  If out->family >= 0 on
 * entry that family is forced (B2C_INVALID_PLAN if it cannot run d). */
b2c_status b2c_select_tiles(const b2c_conv_desc *d, int32_t engine, b2c_tile_plan *out);

/* Register a measured plan (tools/autotune.py "find" result) for an exact
 * shape: the planner then uses (family, splits, reduce) for it instead of its cost
 * model.  The Python package registers paper_2103_16234_b200/tuned_plans.json
 * at import. */
b2c_status b2c_register_tuned_plan(const b2c_conv_desc *d, int32_t engine, int32_t family, int32_t splits,
                                   int32_t reduce);

/* ------------------------------------------------- device-pointer compute */
/* Fused direct convolution (any stride >= 1, any padding).  Replaces the
 * compute of twostage.conv_twostage (twostage.py:208-239) and
 * reference.conv_naive (reference.py:58-83) for device-resident tensors.
 * `tiles` may be NULL (planner's choice) or carry a forced family / split /
 * reduction mode.  Layers with too few output tiles for 148 SMs are split over
 * channel ranges (split-C), reduced either (reduce = 1) through partial planes
 * in `workspace` (tiles.workspace_bytes from b2c_select_tiles,
 * splits*N*M*Ho*Wo*4 bytes) and a second launch that adds them in ascending
 * range order, or (reduce = 2) inside a thread-block cluster through DSMEM in
 * the same order (one launch).  Strided 1x1 layers and 1x1 layers on planes
 * with H*W % 4 != 0 may run the packed-pixel path: a first launch gathers the
 * pixels the layer reads into the head of `workspace`, the convolution reads
 * them from there.  With no (or too small a) workspace the planner picks an
 * unsplit, unpacked plan (a forced plan that needs one fails with
 * B2C_INVALID_ARGUMENT).  Per output, the summation order is a function of
 * (c, hf, wf, splits) only: both reductions give bitwise-identical results. */
b2c_status b2c_conv2d_forward(const b2c_conv_desc *d, const float *x, const float *w, float *y, void *workspace,
                              int64_t workspace_size, const b2c_tile_plan *tiles, void *stream);

/* Tensor-core forward convolution (engine B2C_ENGINE_TF32X3 or _TF32) for
 * device-resident tensors, any stride and padding.  Same semantics and
 * output as b2c_conv2d_forward (which it complements for the
 * large-channel layers, BASELINE.json north star "optional TF32 tcgen05
 * implicit-GEMM variant").  `workspace` receives the per-call pre-tiled
 * filters and the split-K partial planes (b2c_tc_select_tiles()
 * .workspace_bytes bytes).  `tiles` may be NULL (planner's choice) or force
 * filters_per_tile / splits (0 = planner's choice).  Returns
 * B2C_UNSUPPORTED for layers beyond its 32-bit per-image offsets. */
b2c_status b2c_conv2d_forward_tc(const b2c_conv_desc *d, const float *x, const float *w, float *y, void *workspace,
                                 int64_t workspace_size, int32_t engine, const b2c_tc_plan *tiles, void *stream);
/* The tensor-core planner's choice for d (B2C_UNSUPPORTED if not covered).
 * out->filters_per_tile / out->splits / out->mode / out->m_halves > 0 on entry
 * are forced. */
b2c_status b2c_tc_select_tiles(const b2c_conv_desc *d, int32_t engine, b2c_tc_plan *out);

/* Register a measured tensor-core plan (tools/autotune.py) for an exact shape:
 * the planner then uses (mode, filters_per_tile, splits, m_halves) for it.  The
 * Python package registers paper_2103_16234_b200/tuned_plans.json at import. */
b2c_status b2c_register_tuned_tc_plan(const b2c_conv_desc *d, int32_t engine, int32_t mode, int32_t filters_per_tile,
                                      int32_t splits, int32_t m_halves);

/* twostage.conv_twostage (twostage.py:208-239): preconditions in the
 * reference's order, then stage 1 (+ stage 2 unless 1x1) with the reference's
 * rounding order.  `plan` may be NULL (plan_launch default).  `workspace`
 * must hold b2c_workspace_bytes(d) bytes (may be NULL for 1x1). */
b2c_status b2c_conv_twostage(const b2c_conv_desc *d, const float *x, const float *w, float *y,
                             float *workspace, int64_t workspace_size, const b2c_launch_plan *plan,
                             const b2c_device_model *dev, int64_t workspace_limit, void *stream,
                             b2c_run_stats *stats);

/* twostage.stage1_scalar_prods (twostage.py:148-172): partials laid out
 * (k, n, m, ho, wo), k = yf*wf+xf; partials must hold 4*hf*wf*n*m*ho*wo bytes. */
b2c_status b2c_stage1_scalar_prods(const b2c_conv_desc *d, const float *x, const float *w, float *partials,
                                   const b2c_launch_plan *plan, const b2c_device_model *dev,
                                   int64_t workspace_limit, void *stream, b2c_run_stats *stats);

/* twostage.stage2_sum (twostage.py:175-205): y = +0 + sum_k partials[k]. */
b2c_status b2c_stage2_sum(const b2c_conv_desc *d, const float *partials, float *y, void *stream,
                          b2c_run_stats *stats);

/* --------------------------------------------------- host-buffer compute */
/* The drop-in for callers holding host (numpy) buffers: copies x and w to the
 * device, runs `engine`, copies y back, synchronises.  Device buffers are
 * cached per thread and grown on demand.  For B2C_ENGINE_TWOSTAGE the
 * reference preconditions, plan and workspace limit apply exactly as in
 * b2c_conv_twostage; for B2C_ENGINE_FUSED stride >= 1 is accepted and no
 * workspace is used.  device < 0 means the current device. */
b2c_status b2c_conv_host(const b2c_conv_desc *d, const float *x_host, const float *w_host, float *y_host,
                         int32_t engine, const b2c_launch_plan *plan, const b2c_device_model *dev,
                         int64_t workspace_limit, int32_t device, b2c_run_stats *stats);

/* A sequence of independent layers (e.g. one inference pass over a network's
 * convolutions) from host buffers: H2D copies, convolutions and D2H copies of
 * consecutive layers overlap on three streams (six device slots, event
 * ordered); synchronous on return.  Pinned host memory gives full PCIe
 * overlap.  engine: B2C_ENGINE_FUSED, _TF32X3 or _TF32.  The batched form of
 * b2c_conv_host for harness loops like the reference's run_bench
 * (bench.py:91-163), which convolves one layer after another. */
b2c_status b2c_conv_host_layers(int32_t count, const b2c_conv_desc *descs, const float *const *x_host,
                                const float *const *w_host, float *const *y_host, int32_t engine, int32_t device);

/* Host-buffer stage 1 / stage 2 (used by the drop-in stage1_scalar_prods /
 * stage2_sum). */
b2c_status b2c_stage1_host(const b2c_conv_desc *d, const float *x_host, const float *w_host,
                           float *partials_host, const b2c_launch_plan *plan, const b2c_device_model *dev,
                           int64_t workspace_limit, int32_t device, b2c_run_stats *stats);
b2c_status b2c_stage2_host(const b2c_conv_desc *d, const float *partials_host, float *y_host,
                           int32_t device, b2c_run_stats *stats);

/* FP32 roofline denominator: times an FFMA2 (fma.rn.f32x2) register-blocked
 * loop on every SM; returns TFLOP/s (CUDA events), the SM clock the probe ran
 * at (per-CTA clock64 cycles / globaltimer ns) and FMA/clk/SM = FMAs / (SMs x
 * wall time x clock), whose hardware ceiling is 128 (FP32 lanes per SM). */
b2c_status b2c_probe_fp32_peak(int32_t iters, double *tflops, double *fma_per_clk_per_sm, double *sm_mhz);

/* Pinned host memory helpers (so e2e callers can stage through page-locked
 * buffers without linking CUDA themselves). */
void *b2c_host_alloc(size_t bytes);
void b2c_host_free(void *p);

#ifdef __cplusplus
}
#endif

#endif /* B2CONV_H */
