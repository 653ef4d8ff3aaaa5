// Internal (non-ABI) declarations shared by api.cpp and conv_launch.cu.
#pragma once

#include <cuda_runtime.h>

namespace b2c {

// Full geometry of one convolution (derived from b2c_conv_desc).
struct Geom {
  int N, C, H, W, M, HF, WF, S, PH, PW;
  int Ho, Wo, HoWo, Hp, Wp;
  long long Q;  // N*Ho*Wo
};

struct TileChoice {
  int family = -1;
  int kind = 0;  // 0: halo-staged direct kernel, 1: 16-byte pointwise kernel
  int bm = 0, bp = 0, bc = 0, threads = 0, stages = 0;
  int rows = 0, rs = 0, xcs = 0, tile_elems = 0;
  int smem_bytes = 0;
  int occupancy = 0;
  long long grid = 0;   // output tiles (m-tiles x pixel tiles)
  int grid_z = 1;       // stage 1: filter rows
  int splits = 1;       // fused: channel ranges reduced separately
  int chunks_per_split = 0;
  long long ws_bytes = 0;  // workspace needed for splits > 1 (partial planes)
  int reduce = 0;          // splits > 1: 1 = partial planes + stage-2 kernel, 2 = DSMEM cluster reduction
  double cost = 0;
};

// Tensor-core implicit-GEMM plan (conv_tc.cu / conv_tc.cuh).
struct TcPlan {
  int xb = 0;        // gather mode: chunk width XW in output columns (32, 16 or 8; chunk = 32/XW rows)
  int halo = 0;      // halo mode (stride 1): staged positions per tile (0 = gather mode)
  int mh = 1;        // halo mode: 128-position M halves per tile
  int abufs = 0;     // halo mode: staged halo buffers (ring depth)
  int wplanes = 1;   // pre-tiled filter planes streamed from HBM/L2 (gather 3xTF32: hi + lo)
  bool bf16corr = false;
  bool kpack = false;     // gather mode: k-blocks over (channel, tap) pairs (few input channels)  // 3xTF32 halo mode: correction products as bf16 MMAs (K=16, twice the rate)
  int nf = 0;        // output channels per tile (UMMA N)
  int mtiles = 0;
  int stages = 0, stage_bytes = 0, smem_bytes = 0, tmem_cols = 0;
  int passes = 3;    // 3: 3xTF32 (fp32-class), 1: TF32
  bool flat = false; // 1x1: pixels flattened over the plane
  long long nchunks = 0;
  long long grid = 0;  // CTAs incl. splits
  int splits = 1, kb_per_split = 0;  // split-K over (channel block, tap) k-blocks
  double cost = 0;
};
bool tc_supported(const Geom &g);
bool tc_flat(const Geom &g);
long long tc_workspace_bytes(const Geom &g, const TcPlan &pl);
bool plan_tc(const Geom &g, int passes, int forced_nf, int forced_xb, int forced_splits, TcPlan *out,
             int forced_mode = 0, int forced_mh = 0);
long long tc_filter_bytes(const Geom &g, const TcPlan &pl);
void register_tuned_tc(const Geom &g, int passes, int mode, int nf, int splits, int mh = 0);
cudaError_t launch_tc(const Geom &g, const TcPlan &pl, const float *x, const float *w, float *y, void *workspace,
                      long long ws_bytes, cudaStream_t stream);

// split-C workspace: `splits` partial planes in the output layout, [split][n][m][ho][wo]

const char *family_name(int id);
int num_families();
bool family_matches(int fam_id, const Geom &g, bool stage1);
int device_sm_count(int device);
bool family_has_cluster_epilogue(int fam_id);
bool plan_tiles(const Geom &g, bool stage1, int device, int forced_family, int forced_splits, bool allow_split,
                bool allow_vec, TileChoice *out, int forced_reduce = 0);
cudaError_t launch_direct(const Geom &g, const TileChoice &tc, const float *x, const float *w, float *y,
                          bool stage1, long long y_tap_stride, void *workspace, cudaStream_t stream);
cudaError_t launch_stage2(const float *partials, float *y, long long total, int taps, int device,
                          cudaStream_t stream);
bool pdl_enabled();
unsigned long long watchdog_ns();
void register_tuned(const Geom &g, bool stage1, int family, int splits, int reduce = 0);
void note_launch();

}  // namespace b2c
