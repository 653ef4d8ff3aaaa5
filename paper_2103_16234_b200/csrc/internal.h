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
  double cost = 0;
};

// split-C workspace: `splits` partial planes in the output layout, [split][n][m][ho][wo]

const char *family_name(int id);
int num_families();
bool family_matches(int fam_id, const Geom &g, bool stage1);
int device_sm_count(int device);
bool plan_tiles(const Geom &g, bool stage1, int device, int forced_family, int forced_splits, bool allow_split,
                bool allow_vec, TileChoice *out);
cudaError_t launch_direct(const Geom &g, const TileChoice &tc, const float *x, const float *w, float *y,
                          bool stage1, long long y_tap_stride, void *workspace, cudaStream_t stream);
cudaError_t launch_stage2(const float *partials, float *y, long long total, int taps, int device,
                          cudaStream_t stream);
bool pdl_enabled();
void register_tuned(const Geom &g, bool stage1, int family, int splits);
void note_launch();

}  // namespace b2c
