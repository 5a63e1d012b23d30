// cone_kernels.cuh — sm_100a kernels of the cone-beam path.
//
//  K1  cone_bp_kernel   voxel-driven back-projection (projector.hpp:283-313)
//  K2  cone_fp_kernel   ray-driven forward projection (projector.hpp:264-281,
//                       130-152, 83-107, 66-78)
//  aux footprint_kernel plan-time sizing of K1's TMA box
//      pad_volume_kernel zero-bordered volume copy for K2's branch-free taps
#pragma once

#include "device_common.cuh"

namespace tgb {
namespace cone {

// ---- K1 tiling -----------------------------------------------------------
// A CTA owns a BX x BY column tile of the volume and K consecutive z voxels
// per column; every consumer thread owns one (x, y) column and keeps its K
// voxel sums in registers across all views.  Warp w covers x in [0, 16) and
// y in [2w, 2w+2) of the tile, so a warp's LDS addresses stay within ~24
// detector columns; box rows are padded to a pitch of 16 mod 32 words so
// the two half-warps land on disjoint banks when they straddle a row.
constexpr int BX = 16, BY = 16;
constexpr int NCONS = BX * BY;          // consumer threads (8 warps)
constexpr int NTHREADS = NCONS + 32;    // + one producer warp
constexpr int STAGES = 6;               // projection boxes in flight
constexpr int kMaxConstViews = 640;     // FP64 matrices per constant-bank upload (60 KB)
constexpr int MODE_FAST = 0, MODE_SLOW = 1, MODE_SKIP = 2;

struct BpArgs {
  int nx, ny, nz;           // slab extent
  int z0;                   // global z index of the slab's first slice
  double ox, oy, oz;        // volume origin (world, mm)
  double sx, sy, sz;        // voxel pitch
  int nu, nv;               // full detector
  int band_v0, band_rows;   // detector rows present in `sino`
  int n_views;              // views in this launch (constant slots bank_off..bank_off+n-1)
  int bank_off;             // first view's slot in the constant bank
  int view_base;            // first view's index in the TMA tensor / sino buffer
  int boxU, boxV;           // TMA box (elements)
  float sid2;               // SID^2: 1/w^2 = SID^2 / hz^2
  float scale;
  int accumulate;
  // -(0x4B400000 * 4 * BOXU) mod 2^32: the magic-floor bias of a row address,
  // passed at run time so ptxas cannot split it back out of the per-view base
  uint32_t magic_row_off;
  const float* sino;        // band buffer (slow path gathers)
  long long row_pitch;      // elements between detector rows
  long long view_pitch;     // elements between views
  float* vol;               // slab [nz][ny][nx]
};

// Footprint of a tile on one view: the detector box holding every tap the
// tile's voxels can touch, with one pixel of margin for fp32 rounding.
struct Footprint {
  int ub, vb, width, height;
  bool ok;   // every corner in front of the source and finite
  bool hit;  // overlaps the detector at all
};

}  // namespace cone
}  // namespace tgb
