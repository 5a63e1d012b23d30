// cone.cu — cone-beam plan, K1 back-projection, K2 forward projection and
// the host-buffer pipelines.  Reference: projector.hpp:264-313 (operators),
// pipelines.hpp:73-84 (FDK composition), geometry.hpp:126-178 (plan data).
#include <mutex>
#include <string>
#include <algorithm>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "cone_kernels.cuh"
#include "filter.cuh"

namespace tgb {
namespace cone {

// per-view projection matrices in FP64, row-major P = K[R|t] (12 doubles)
__constant__ double c_views[12 * kMaxConstViews];
static ConstBank g_bank;

// ---------------------------------------------------------------------------
// Footprint + local frame of one (tile, view), computed in FP64 by the
// producer warp (and, identically, by the plan-time sizing kernel).

__device__ __forceinline__ Footprint make_footprint(double umin, double umax, double vmin,
                                                    double vmax, bool ok, int nu, int nv) {
  Footprint f;
  ok = ok && fabs(umin) < 4.0e6 && fabs(umax) < 4.0e6 && fabs(vmin) < 4.0e6 && fabs(vmax) < 4.0e6;
  f.ok = ok;
  if (!ok) {
    f.ub = f.vb = f.width = f.height = 0;
    f.hit = true;
    return f;
  }
  const int u_lo = int(floor(umin)), u_hi = int(floor(umax));
  const int v_lo = int(floor(vmin)), v_hi = int(floor(vmax));
  // taps [u_lo, u_hi + 1] plus one pixel of margin each side; the box's
  // first column is rounded down to a multiple of 4 because TMA requires
  // 16-byte aligned inner coordinates
  f.ub = (u_lo - 1) & ~3;
  f.vb = v_lo - 1;
  f.width = u_hi + 3 - f.ub;
  f.height = v_hi - v_lo + 4;
  // every tap outside the detector contributes exactly zero
  f.hit = !(u_hi + 2 < 0 || f.ub > nu - 1 || v_hi + 2 < 0 || f.vb > nv - 1);
  return f;
}

// Tile extent in voxel indices (slab-local z) and its centre in world units.
struct Tile {
  int x0, x1, y0, y1, z0, z1;  // inclusive
  double xc, yc, zc;           // centre (mm)
};

__device__ __forceinline__ Tile make_tile(const BpArgs& a, int tx, int ty, int tz, int K) {
  Tile t;
  t.x0 = tx * BX;
  t.y0 = ty * BY;
  t.z0 = tz * K;
  t.x1 = min(t.x0 + BX, a.nx) - 1;
  t.y1 = min(t.y0 + BY, a.ny) - 1;
  t.z1 = min(t.z0 + K, a.nz) - 1;
  t.xc = a.ox + 0.5 * double(t.x0 + t.x1) * a.sx;
  t.yc = a.oy + 0.5 * double(t.y0 + t.y1) * a.sy;
  t.zc = a.oz + 0.5 * double(2 * a.z0 + t.z0 + t.z1) * a.sz;
  return t;
}

__device__ __forceinline__ void corner_uv(const double* P, const BpArgs& a, const Tile& t, int c,
                                          double& u, double& v, bool& ok) {
  const double x = a.ox + double((c & 1) ? t.x1 : t.x0) * a.sx;
  const double y = a.oy + double((c & 2) ? t.y1 : t.y0) * a.sy;
  const double z = a.oz + double(a.z0 + ((c & 4) ? t.z1 : t.z0)) * a.sz;
  const double hx = P[0] * x + P[1] * y + P[2] * z + P[3];
  const double hy = P[4] * x + P[5] * y + P[6] * z + P[7];
  const double hz = P[8] * x + P[9] * y + P[10] * z + P[11];
  ok = hz > 0.0;
  // the footprint only selects a box (with a one-pixel margin), so the
  // divide runs in fp32 on the FP64 homogeneous coordinates: no DDIV in the
  // producer's per-view critical path
  const float r = 1.0f / float(hz);
  u = double(float(hx) * r);
  v = double(float(hy) * r);
}

// plan-time: largest footprint over every (tile, view) that takes the fast path
__global__ void footprint_kernel(BpArgs a, int K, int tiles_x, int tiles_y, int tiles_z,
                                 const double* __restrict__ mats, int* __restrict__ need) {
  const long long n_tiles = (long long)tiles_x * tiles_y * tiles_z;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_tiles * a.n_views) return;
  const int view = int(idx / n_tiles);
  long long r = idx % n_tiles;
  const int tx = int(r % tiles_x);
  r /= tiles_x;
  const int ty = int(r % tiles_y), tz = int(r / tiles_y);
  const Tile t = make_tile(a, tx, ty, tz, K);
  const double* P = mats + 12 * view;
  double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
  bool ok = true;
  for (int c = 0; c < 8; ++c) {
    double u, v;
    bool okc;
    corner_uv(P, a, t, c, u, v, okc);
    ok = ok && okc;
    umin = fmin(umin, u);
    umax = fmax(umax, u);
    vmin = fmin(vmin, v);
    vmax = fmax(vmax, v);
  }
  const Footprint f = make_footprint(umin, umax, vmin, vmax, ok, a.nu, a.nv);
  if (f.ok && f.hit) {
    atomicMax(&need[0], f.width);
    atomicMax(&need[1], f.height);
  }
}

// ---------------------------------------------------------------------------
// K1: voxel-driven back-projection

// d = a * B + c as one IMAD the compiler cannot re-associate (keeps the
// per-view constant folded into c)
template <uint32_t B>
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "n"(B), "r"(c));
  return d;
}

// the four bilinear taps (row r: a0 a1, row r+1: b0 b1) at one shared
// address with immediate offsets
template <uint32_t ROWB>
__device__ __forceinline__ void lds_quad(uint32_t ad, float& a0, float& a1, float& b0, float& b1) {
  asm volatile(
      "ld.shared.f32 %0, [%4];\n\t"
      "ld.shared.f32 %1, [%4+4];\n\t"
      "ld.shared.f32 %2, [%4+%5];\n\t"
      "ld.shared.f32 %3, [%4+%6];"
      : "=f"(a0), "=f"(a1), "=f"(b0), "=f"(b1)
      : "r"(ad), "n"(ROWB), "n"(ROWB + 4));
}

template <uint32_t ROWB>
__device__ __forceinline__ void lds_quad_v(uint32_t ad, float& a0, float& a1, float& b0, float& b1) {
  asm volatile(
      "ld.volatile.shared.f32 %0, [%4];\n\t"
      "ld.volatile.shared.f32 %1, [%4+4];\n\t"
      "ld.volatile.shared.f32 %2, [%4+%5];\n\t"
      "ld.volatile.shared.f32 %3, [%4+%6];"
      : "=f"(a0), "=f"(a1), "=f"(b0), "=f"(b1)
      : "r"(ad), "n"(ROWB), "n"(ROWB + 4));
}

// zero-padded bilinear gather from global memory (slow path; projector.hpp:44-64)
__device__ __forceinline__ float bilinear_global(const BpArgs& a, const float* __restrict__ img,
                                                 float u, float v) {
  const float fu = floorf(u), fv = floorf(v);
  const int c0 = int(fu), r0 = int(fv);
  const float wu = u - fu, wv = v - fv;
  float acc = 0.0f;
#pragma unroll
  for (int dr = 0; dr < 2; ++dr) {
    const int r = r0 + dr;
    if (r < 0 || r >= a.nv) continue;
    const int rb = r - a.band_v0;
    if (rb < 0 || rb >= a.band_rows) continue;
    const float wr = dr ? wv : 1.0f - wv;
    const float* row = img + (long long)rb * a.row_pitch;
    if (c0 >= 0 && c0 < a.nu) acc += (1.0f - wu) * wr * __ldg(row + c0);
    if (c0 + 1 >= 0 && c0 + 1 < a.nu) acc += wu * wr * __ldg(row + c0 + 1);
  }
  return acc;
}

// K1 epilogue, per warp and without barriers: the warp holds 8 x 4 (x, y)
// columns of 4 * NB z-voxels (v4[b] = voxels 4b .. 4b+3 of this lane's
// column); each group of 4 x-neighbour lanes transposes its 4 x 4 blocks
// (x, z) through shuffles so that lane i of the group ends with the float4
// (x0 .. x0+3) of z-voxels i, i+4, i+8, ...: the volume is written
// (read-modify-written when accumulating) as coalesced float4 rows (north_star
// item 3).  Same per-voxel arithmetic as a scalar store: *o = acc ? *o + v : v.
// Kept out of line so that the view loop's register allocation is not
// disturbed by it (inlined, the loop measured 1% slower at c4).
template <int NB>
__device__ __noinline__ void k1_store(const BpArgs& a, const float4* v4, int lane, int gx4, int gy,
                                      int z0, int kmax) {
  const int gi = lane & 3;
  const bool row_ok = gy < a.ny;
  const bool vec = ((reinterpret_cast<uintptr_t>(a.vol) & 15) == 0) && ((a.nx & 3) == 0) &&
                   gx4 + 3 < a.nx;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const float v[4] = {v4[b].x, v4[b].y, v4[b].z, v4[b].w};
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    // round r: lane i sends v[(i - r) & 3] and receives lane ((i + r) & 3)'s
    // v[i], i.e. x = (i + r) & 3 at z = 4b + i
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int sj = (gi - r) & 3;
      const float send = sj == 0 ? v[0] : sj == 1 ? v[1] : sj == 2 ? v[2] : v[3];
      const float got = __shfl_sync(0xffffffffu, send, (lane & ~3) | ((gi + r) & 3));
      const int dj = (gi + r) & 3;
      t[0] = dj == 0 ? got : t[0];
      t[1] = dj == 1 ? got : t[1];
      t[2] = dj == 2 ? got : t[2];
      t[3] = dj == 3 ? got : t[3];
    }
    const int k = 4 * b + gi;
    if (!row_ok || k > kmax) continue;
    float* o = a.vol + ((long long)(z0 + k) * a.ny + gy) * a.nx + gx4;
    if (vec) {
      float4 val = make_float4(t[0], t[1], t[2], t[3]);
      if (a.accumulate) {
        const float4 old = *reinterpret_cast<const float4*>(o);
        val = make_float4(old.x + val.x, old.y + val.y, old.z + val.z, old.w + val.w);
      }
      *reinterpret_cast<float4*>(o) = val;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (gx4 + c < a.nx) o[c] = a.accumulate ? o[c] + t[c] : t[c];
    }
  }
}

// producer back-off between empty-barrier polls (c4 K1: 37.24 ms spinning,
// 37.12 / 36.83 / 36.63 / 36.51 / 36.59 ms at 32 / 128 / 512 / 2048 / 4096 ns)
#ifndef TG_K1_GEN_FMARM
#define TG_K1_GEN_FMARM 1
#endif

#ifndef TG_K1_GEN_PIPE
#define TG_K1_GEN_PIPE 1
#endif

#ifndef TG_K1_BACKOFF_NS
#define TG_K1_BACKOFF_NS 2048
#endif

// Per-stage header written by the producer: the view's projective map in a
// local frame, h = M (dx, dy, dz, 1) with (dx, dy, dz) the voxel's offset
// from the tile centre and the u / v rows already shifted by the box origin
// (u_row -= ub * w_row, v_row -= vb * w_row).  Built in FP64, so fp32
// consumers see small, well-conditioned numbers.
struct StageHdr {
  float4 U, V, W;
  int4 meta;  // ub, vb, mode, -
};

// 3 CTAs (24 consumer + 3 producer warps) per SM: 72 registers (the few
// spills sit in the per-view prologue and the partial-tile path, not in the
// fast loop) and a 6-stage ring (<= 72 KB of boxes per CTA).  Against 2 CTAs
// at 96 registers: 45.2 -> 41.9 ms at c4.  The general (calibrated) variant
// too since round 2's FFMA2 loop (no spills in its fast loop at 72): c4
// calibrated 55.73 -> 53.35 ms against 2 CTAs at 96 registers (80: 55.79;
// round 1's scalar loop spilled at 72, 891 vs 1043 GUPS).
template <int K, int BOXU, bool CIRC>
__global__ void __maxnreg__(72)
    cone_bp_kernel(const __grid_constant__ CUtensorMap tmap, const BpArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int box_elems = BOXU * a.boxV;
  // TMA needs 128-byte aligned shared destinations: pad the stage stride
  const int stage_elems = (box_elems + 31) & ~31;
  float* boxes = reinterpret_cast<float*>(smem);
  StageHdr* hdr = reinterpret_cast<StageHdr*>(boxes + STAGES * stage_elems);
  uint64_t* full = reinterpret_cast<uint64_t*>(hdr + STAGES);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  // programmatic dependent launch: the next K1 of a chunked pipeline may start
  // its view loop on the SMs this grid's tail leaves idle; it waits for this
  // grid before its epilogue touches the volume (no-ops without PDL)
  asm volatile("griddepcontrol.launch_dependents;");
  const Tile tile = make_tile(a, blockIdx.x, blockIdx.y, blockIdx.z, K);

  if (tid >= NCONS) {
    // ---------------- producer warp: footprint, frame, TMA per view --------
    // Four views at a time, one 8-lane group per view (lane c of a group
    // projects tile corner c; the group leader builds the frame and issues
    // the TMA once the view's stage is free): the FP64 corner / frame chain is
    // latency-bound, and one view per step left the consumers waiting on the
    // full barrier in ~13% of their stall samples.
    const int lane = tid & 31;
    const int g = lane >> 3, c = lane & 7;
    if (lane == 0) prefetch_tensor_map(&tmap);
    for (int it0 = 0; it0 < a.n_views; it0 += 4) {
      const int it = it0 + g;
      const bool has_view = it < a.n_views;
      const double* P = c_views + 12 * (a.bank_off + (has_view ? it : it0));
      double u = 0.0, v = 0.0;
      bool ok = true;
      corner_uv(P, a, tile, c, u, v, ok);
      double umin = u, umax = u, vmin = v, vmax = v;
#pragma unroll
      for (int off = 4; off >= 1; off >>= 1) {  // reduce over the group's 8 corner lanes
        umin = fmin(umin, __shfl_xor_sync(0xffffffffu, umin, off));
        umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, off));
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, off));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, off));
        ok = __shfl_xor_sync(0xffffffffu, int(ok), off) && ok;
      }
      if (c == 0 && has_view) {
        const int s = it % STAGES;
        const Footprint f = make_footprint(umin, umax, vmin, vmax, ok, a.nu, a.nv);
        int mode = MODE_SLOW;
        if (f.ok && !f.hit) mode = MODE_SKIP;
        else if (f.ok && f.width <= BOXU && f.height <= a.boxV) mode = MODE_FAST;
        // local frame: rows evaluated at the tile centre, u/v shifted to the box
        const double ub = mode == MODE_FAST ? double(f.ub) : 0.0;
        const double vb = mode == MODE_FAST ? double(f.vb) : 0.0;
        double hc[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
          hc[r] = P[4 * r] * tile.xc + P[4 * r + 1] * tile.yc + P[4 * r + 2] * tile.zc + P[4 * r + 3];
        StageHdr h;
        h.U = make_float4(float(P[0] - ub * P[8]), float(P[1] - ub * P[9]),
                          float(P[2] - ub * P[10]), float(hc[0] - ub * hc[2]));
        h.V = make_float4(float(P[4] - vb * P[8]), float(P[5] - vb * P[9]),
                          float(P[6] - vb * P[10]), float(hc[1] - vb * hc[2]));
        h.W = make_float4(float(P[8]), float(P[9]), float(P[10]), float(hc[2]));
        h.meta = make_int4(f.ub, f.vb, mode, 0);
        // the stage's previous view has been consumed
        if (it >= STAGES) mbar_wait_backoff(&empty[s], ((it / STAGES) - 1) & 1, TG_K1_BACKOFF_NS);
        hdr[s] = h;
        if (mode == MODE_FAST) {
          mbar_arrive_expect_tx(&full[s], uint32_t(box_elems * 4));
          tma_load_3d(boxes + s * stage_elems, &tmap, &full[s], f.ub, f.vb - a.band_v0,
                      a.view_base + it);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- consumers: one (x, y) column, K voxels each -------------
  const int w = tid >> 5, lane = tid & 31;
  // warp -> 8 x 4 (x, y) columns of the 16 x 16 tile (fewer bank conflicts
  // than 16 x 2: 1408 vs 1351 GUPS at c4; 4 x 8 measured equal)
  const int lx = (lane & 7) + 8 * (w & 1);
  const int ly = 4 * (w >> 1) + (lane >> 3);
  const int gx = tile.x0 + lx, gy = tile.y0 + ly;
  const int ix = min(gx, a.nx - 1), iy = min(gy, a.ny - 1);
  // offsets from the tile centre (exact small numbers)
  const float dx = float((double(ix) - 0.5 * double(tile.x0 + tile.x1)) * a.sx);
  const float dy = float((double(iy) - 0.5 * double(tile.y0 + tile.y1)) * a.sy);
  const float dz0 = float((double(tile.z0) - 0.5 * double(tile.z0 + tile.z1)) * a.sz);
  const float sz = float(a.sz);
  const int kmax = tile.z1 - tile.z0;  // clamp tail voxels into the tile
  const uint32_t box_base = smem_u32(boxes);
  constexpr uint32_t ROWB = BOXU * 4;
  constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23: t = M + floor(v) under round-down
  constexpr uint32_t MAGIC_BITS = 0x4B400000u;

  // accumulators as (k, k + K/2) pairs for the FP32x2 pipe
  float2 acc[K / 2];
#pragma unroll
  for (int k = 0; k < K / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
#define ACC(k) ((k) >= K / 2 ? acc[(k) - K / 2].y : acc[(k)].x)

  for (int it = 0; it < a.n_views; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const float4 U = hdr[s].U, V = hdr[s].V, W = hdr[s].W;
    const int mode = hdr[s].meta.z;
    const float un = fmaf(U.x, dx, fmaf(U.y, dy, U.w));
    const float vn = fmaf(V.x, dx, fmaf(V.y, dy, V.w));
    const float hz0 = fmaf(W.x, dx, fmaf(W.y, dy, W.w));
    if (mode == MODE_FAST) {
      const uint32_t sbase = box_base + uint32_t(s * stage_elems) * 4u;
      if (CIRC) {
        // P[0][2] == P[2][2] == 0: u and 1/w^2 are constant along z and v is
        // affine in z (SURVEY §7 hard part (b)).
        // MUFU reciprocal (~1 ulp; no IEEE slow path in the per-view prologue)
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(hz0));
        const float invw2 = r * r;  // SID^2 is applied in the epilogue
        const float u = un * r;
        const float fu = floorf(u);
        const float wu = u - fu;
        const float v0 = fmaf(V.z, dz0, vn) * r;
        const float dv = V.z * sz * r;
        // a.magic_row_off = -MAGIC_BITS * ROWB (run-time value: ptxas would
        // otherwise re-associate the constant out of the IMAD and re-add it
        // before every LDS — it does not fit the 24-bit immediate offset)
        const uint32_t cbase = sbase + uint32_t(int(fu)) * 4u + a.magic_row_off;
        // two updates per step on the packed FP32x2 pipe (FFMA2 / FADD2):
        // voxels k and k + K/2, whose v differ by the per-view constant
        // (K/2)·dv folded into the pair's base.  Per update: v, floor
        // (round-down magic add), one IMAD address, 4 LDS, three lerps, one FFMA.
        constexpr int H = K / 2;
        const float2 v02 = make_float2(v0, fmaf(float(H), dv, v0)), dv2 = make_float2(dv, dv);
        const float2 wu2 = make_float2(wu, wu), iw2 = make_float2(invw2, invw2);
        const float2 M2 = make_float2(MAGIC, MAGIC), nM2 = make_float2(-MAGIC, -MAGIC);
        // software pipeline: pair k+1's 8 LDS are issued before pair k's
        // lerps.  The loads are ld.volatile.shared (same LDS, same
        // wavefronts) so ptxas keeps this order instead of re-serialising
        // each pair behind its own loads (45.2 vs 47.3 ms at c4).
        struct Taps {
          float a0, a1, b0, b1, c0, c1, d0, d1;
          float2 wv;
        };
        auto fetch = [&](float2 vk, Taps& q) {
          const float2 t = __fadd2_rd(vk, M2);
          const float2 fl = __fadd2_rn(t, nM2);
          q.wv = __fadd2_rn(vk, make_float2(-fl.x, -fl.y));
          lds_quad_v<ROWB>(mad_u32<ROWB>(__float_as_uint(t.x), cbase), q.a0, q.a1, q.b0, q.b1);
          lds_quad_v<ROWB>(mad_u32<ROWB>(__float_as_uint(t.y), cbase), q.c0, q.c1, q.d0, q.d1);
        };
        auto blend = [&](const Taps& q, float2& acc2) {
          const float2 p0 = make_float2(q.a0, q.c0), p1 = make_float2(q.a1, q.c1);
          const float2 q0 = make_float2(q.b0, q.d0), q1 = make_float2(q.b1, q.d1);
          const float2 top = __ffma2_rn(wu2, __fadd2_rn(p1, make_float2(-p0.x, -p0.y)), p0);
          const float2 bot = __ffma2_rn(wu2, __fadd2_rn(q1, make_float2(-q0.x, -q0.y)), q0);
          const float2 mid = __ffma2_rn(q.wv, __fadd2_rn(bot, make_float2(-top.x, -top.y)), top);
          acc2 = __ffma2_rn(mid, iw2, acc2);
        };
        Taps tp[2];
        if (kmax == K - 1) {  // full tile (every tile when nz % K == 0)
          fetch(__ffma2_rn(make_float2(0.f, 0.f), dv2, v02), tp[0]);
#pragma unroll
          for (int k = 0; k < H; ++k) {
            if (k + 1 < H)
              fetch(__ffma2_rn(make_float2(float(k + 1), float(k + 1)), dv2, v02), tp[(k + 1) & 1]);
            blend(tp[k & 1], acc[k]);
          }
        } else {
          const float2 v00 = make_float2(v0, v0);
#pragma unroll
          for (int k = 0; k < H; ++k) {
            fetch(__ffma2_rn(make_float2(float(min(k, kmax)), float(min(k + H, kmax))), dv2, v00),
                  tp[0]);
            blend(tp[0], acc[k]);
          }
        }
      } else {
        // general calibrated matrices: the full projective map per voxel,
        // voxels k and k + K/2 as FP32x2 pairs.  Along a column the depth hz and
        // the u / v numerators are affine in k, so each is one FFMA2 from
        // per-view bases; the reciprocal is the MUFU approximation (~1 ulp: far
        // inside the parity tolerance); 1/w^2 = SID^2 r^2 with SID^2 folded into
        // the epilogue's scale (every mode accumulates r^2-weighted taps); full
        // tiles use compile-time voxel offsets (no clamp)
        constexpr int H = K / 2;
        const uint32_t base2 = sbase + a.magic_row_off + 0u - MAGIC_BITS * 4u;
        const float hzA = fmaf(W.z, dz0, hz0), hzS = W.z * sz;
        const float nuA = fmaf(U.z, dz0, un), nuS = U.z * sz;
        const float nvA = fmaf(V.z, dz0, vn), nvS = V.z * sz;
        const float2 hzA2 = make_float2(hzA, hzA), hzS2 = make_float2(hzS, hzS);
        const float2 nuA2 = make_float2(nuA, nuA), nuS2 = make_float2(nuS, nuS);
        const float2 nvA2 = make_float2(nvA, nvA), nvS2 = make_float2(nvS, nvS);
        const float2 M2 = make_float2(MAGIC, MAGIC), nM2 = make_float2(-MAGIC, -MAGIC);
        auto voxel_pair = [&](float2 kk, float2& acc2) {
          const float2 hz = __ffma2_rn(kk, hzS2, hzA2);
          float2 r;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(hz.x));
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(hz.y));
          const float2 u = __fmul2_rn(__ffma2_rn(kk, nuS2, nuA2), r);
          const float2 v = __fmul2_rn(__ffma2_rn(kk, nvS2, nvA2), r);
          const float2 tu = __fadd2_rd(u, M2), tv = __fadd2_rd(v, M2);
          const float2 fu = __fadd2_rn(tu, nM2), fv = __fadd2_rn(tv, nM2);
          const float2 wu = __fadd2_rn(u, make_float2(-fu.x, -fu.y));
          const float2 wv = __fadd2_rn(v, make_float2(-fv.x, -fv.y));
          const float2 iw = __fmul2_rn(r, r);
          float a0, a1, b0, b1, c0, c1, d0, d1;
          lds_quad<ROWB>(mad_u32<ROWB>(__float_as_uint(tv.x), base2 + __float_as_uint(tu.x) * 4u),
                         a0, a1, b0, b1);
          lds_quad<ROWB>(mad_u32<ROWB>(__float_as_uint(tv.y), base2 + __float_as_uint(tu.y) * 4u),
                         c0, c1, d0, d1);
          const float2 p0 = make_float2(a0, c0), p1 = make_float2(a1, c1);
          const float2 q0 = make_float2(b0, d0), q1 = make_float2(b1, d1);
          const float2 top = __ffma2_rn(wu, __fadd2_rn(p1, make_float2(-p0.x, -p0.y)), p0);
          const float2 bot = __ffma2_rn(wu, __fadd2_rn(q1, make_float2(-q0.x, -q0.y)), q0);
          const float2 mid = __ffma2_rn(wv, __fadd2_rn(bot, make_float2(-top.x, -top.y)), top);
          acc2 = __ffma2_rn(mid, iw, acc2);
        };
        struct GTaps {
          float a0, a1, b0, b1, c0, c1, d0, d1;
          float2 wu, wv, iw;
        };
        auto gfetch = [&](float2 kk, GTaps& q) {
          const float2 hz = __ffma2_rn(kk, hzS2, hzA2);
          float2 r;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(hz.x));
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(hz.y));
          const float2 nu = __ffma2_rn(kk, nuS2, nuA2), nv = __ffma2_rn(kk, nvS2, nvA2);
#if TG_K1_GEN_FMARM
          // floor of the exact product nu * r: t = RD(nu * r + M) in one FFMA
          // (round-down magic), the fraction as one FFMA against the floor.  It
          // can differ from floor(RN(nu * r)) only when the product lies within
          // half an ulp below an integer n: then the taps are (n - 1, n) with
          // weight RN(nu * r - (n - 1)) = 1 — the same bilinear value, and inside
          // the box's one-pixel margin (make_footprint)
          const float2 tu = __ffma2_rd(nu, r, M2), tv = __ffma2_rd(nv, r, M2);
          const float2 fu = __fadd2_rn(tu, nM2), fv = __fadd2_rn(tv, nM2);
          q.wu = __ffma2_rn(nu, r, make_float2(-fu.x, -fu.y));
          q.wv = __ffma2_rn(nv, r, make_float2(-fv.x, -fv.y));
#else
          const float2 u = __fmul2_rn(nu, r);
          const float2 v = __fmul2_rn(nv, r);
          const float2 tu = __fadd2_rd(u, M2), tv = __fadd2_rd(v, M2);
          const float2 fu = __fadd2_rn(tu, nM2), fv = __fadd2_rn(tv, nM2);
          q.wu = __fadd2_rn(u, make_float2(-fu.x, -fu.y));
          q.wv = __fadd2_rn(v, make_float2(-fv.x, -fv.y));
#endif
          q.iw = __fmul2_rn(r, r);
          lds_quad_v<ROWB>(mad_u32<ROWB>(__float_as_uint(tv.x), base2 + __float_as_uint(tu.x) * 4u),
                           q.a0, q.a1, q.b0, q.b1);
          lds_quad_v<ROWB>(mad_u32<ROWB>(__float_as_uint(tv.y), base2 + __float_as_uint(tu.y) * 4u),
                           q.c0, q.c1, q.d0, q.d1);
        };
        auto gblend = [&](const GTaps& q, float2& acc2) {
          const float2 p0 = make_float2(q.a0, q.c0), p1 = make_float2(q.a1, q.c1);
          const float2 q0 = make_float2(q.b0, q.d0), q1 = make_float2(q.b1, q.d1);
          const float2 top = __ffma2_rn(q.wu, __fadd2_rn(p1, make_float2(-p0.x, -p0.y)), p0);
          const float2 bot = __ffma2_rn(q.wu, __fadd2_rn(q1, make_float2(-q0.x, -q0.y)), q0);
          const float2 mid = __ffma2_rn(q.wv, __fadd2_rn(bot, make_float2(-top.x, -top.y)), top);
          acc2 = __ffma2_rn(mid, q.iw, acc2);
        };
        if (kmax == K - 1) {
#if TG_K1_GEN_PIPE
          // software pipeline as in the circular path: pair k+1's map and
          // loads are issued before pair k's lerps
          GTaps gq[2];
          gfetch(make_float2(0.f, float(H)), gq[0]);
#pragma unroll
          for (int k = 0; k < H; ++k) {
            if (k + 1 < H) gfetch(make_float2(float(k + 1), float(k + 1 + H)), gq[(k + 1) & 1]);
            gblend(gq[k & 1], acc[k]);
          }
#else
#pragma unroll
          for (int k = 0; k < H; ++k) voxel_pair(make_float2(float(k), float(k + H)), acc[k]);
#endif
        } else {
#pragma unroll
          for (int k = 0; k < H; ++k)
            voxel_pair(make_float2(float(min(k, kmax)), float(min(k + H, kmax))), acc[k]);
        }
      }
    } else if (mode == MODE_SLOW) {
      // absolute frame (ub = vb = 0): per-voxel checks against the reference
      const float* img = a.sino + (long long)(a.view_base + it) * a.view_pitch;
#pragma unroll
      for (int k = 0; k < K; ++k) {  // unrolled: acc[] must stay in registers
        const float dz = fmaf(float(min(k, kmax)), sz, dz0);
        const float hz = fmaf(W.z, dz, hz0);
        if (!(hz > 0.0f)) continue;  // behind the source (projector.hpp:302)
        const float u = fmaf(U.z, dz, un) / hz, v = fmaf(V.z, dz, vn) / hz;
        if (!(fabsf(u) < 4.0e6f) || !(fabsf(v) < 4.0e6f)) continue;
        ACC(k) += bilinear_global(a, img, u, v) * (1.0f / (hz * hz));  // SID^2 in the epilogue
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // the previous grid of the stream (PDL) has finished writing the volume
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the taps were weighted by 1/hz^2; 1/w^2 = SID^2 / hz^2 (projector.hpp:306)
  const float sc = a.scale * a.sid2;
  float4 v4[K / 4];
#pragma unroll
  for (int b = 0; b < K / 4; ++b)
    v4[b] = make_float4(ACC(4 * b) * sc, ACC(4 * b + 1) * sc, ACC(4 * b + 2) * sc, ACC(4 * b + 3) * sc);
  k1_store<K / 4>(a, v4, lane, tile.x0 + (lx & ~3), gy, tile.z0, kmax);
}

// ---------------------------------------------------------------------------
// K2: ray-driven forward projection

struct FpArgs {
  int nu, nv;
  int view0;
  int nx, ny, nz;
  double ox, oy, oz, sx, sy, sz;
  double step;                    // march_step: 0.5 * min pitch
  const double* __restrict__ geo;  // per view: source (3) + inverse block (9)
  // zero-bordered "quad" volume, +2 on each side: element (x, y, z) holds
  // (V[z][y][x], V[z][y+1][x], V[z][y][x+1], V[z][y+1][x+1]), so one
  // trilinear sample is two 16-byte gathers (slices z and z+1) and the two
  // x-lerps of a slice are one FP32x2 pair
  const float4* __restrict__ vq;
  // the same quads in y-fastest order (index y + x * nyp + z * nxp * nyp):
  // views whose rays run mostly along x gather from it, so the 8 u-lanes of
  // a warp (which then step along y) read neighbouring quads
  const float4* __restrict__ vqT;
  int nxp, nyp;                   // padded extents (x, y)
  // MAGIC_BITS * (sx + sy + nxp * nyp) mod 2^32 for the x- / y-fastest quads
  uint32_t mbias, mbias_t;
  float* out;                     // [n_views][nv][nu]
};

#define DADD __dadd_rn
#define DMUL __dmul_rn
#define DDIV __ddiv_rn

// projector.hpp:83-101 clip_ray in IEEE FP64 without contraction: the hit
// test and the sample count are bit-exact with the reference.
__device__ __forceinline__ bool clip_ray3(const FpArgs& a, const double o[3], const double d[3],
                                          double& t0, double& t1) {
  const double org[3] = {a.ox, a.oy, a.oz};
  const double sp[3] = {a.sx, a.sy, a.sz};
  const int n[3] = {a.nx, a.ny, a.nz};
  t0 = -1e300;
  t1 = 1e300;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double lo = DADD(org[ax], -sp[ax]);
    const double hi = DADD(org[ax], DMUL(double(n[ax]), sp[ax]));
    if (fabs(d[ax]) < 1e-12) {
      if (o[ax] <= lo || o[ax] >= hi) return false;
      continue;
    }
    double ta = DDIV(DADD(lo, -o[ax]), d[ax]);
    double tb = DDIV(DADD(hi, -o[ax]), d[ax]);
    if (ta > tb) {
      const double tt = ta;
      ta = tb;
      tb = tt;
    }
    t0 = (t0 < ta) ? ta : t0;
    t1 = (tb < t1) ? tb : t1;
  }
  return t1 > t0;
}

// projector.hpp:264-281 ray setup for detector pixel (iu, iv) of view `view`
// (d = M^-1 (iu, iv, 1), then (1/|d|) d) and its clip, in IEEE FP64 without
// contraction.  Shared by K2 and the sample-count diagnostic, so the count
// the test compares is the one the projector marches.
__device__ __forceinline__ bool cone_ray(const FpArgs& a, int iu, int iv, int view, double o[3],
                                         double d[3], double& t0, double& t1) {
  const double* g = a.geo + 12 * view;
  o[0] = g[0];
  o[1] = g[1];
  o[2] = g[2];
  const double* M = g + 3;
  const double X = double(iu), Y = double(iv);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    d[r] = DADD(DADD(DMUL(M[3 * r], X), DMUL(M[3 * r + 1], Y)), DMUL(M[3 * r + 2], 1.0));
  const double nn = DADD(DADD(DMUL(d[0], d[0]), DMUL(d[1], d[1])), DMUL(d[2], d[2]));
  const double s = DDIV(1.0, __dsqrt_rn(nn));
#pragma unroll
  for (int r = 0; r < 3; ++r) d[r] = DMUL(s, d[r]);
  return clip_ray3(a, o, d, t0, t1);
}

// projector.hpp:117,138: n = ceil((t1 - t0) / step)
__device__ __forceinline__ long long ray_sample_count(double span, double step) {
  return (long long)ceil(DDIV(span, step));
}

__device__ __forceinline__ float lerpf(float a, float b, float w) { return fmaf(w, b - a, a); }

// Grid: x = 32-pixel u tiles, y = views, z = 8-row v bands (slowest).  A band
// of detector rows sees only a z-slab of the volume through every view, so
// the CTAs resident at any time gather from an L2-sized working set instead
// of streaming the whole volume from HBM once per view.
// Each warp covers 8 u x 4 v pixels (its rays stay close together in 3D:
// fewer cache lines per gather than a 32-wide row of pixels).
// Occupancy: 6 CTAs/SM (40 registers; the spills sit in the FP64 ray setup)
// for the 8-row-band variant used while the volume's slices are small (c4:
// 442.7 -> 432.7 ms at 5 CTAs; 401.5 -> 399.2 ms at 6 once the march loop
// was trimmed to ~27 instructions per sample), 4 CTAs/SM (64 registers)
// for the 4-row-band variant of large volumes (c5: 5 CTAs measured 0.7% slower,
// 6 CTAs 6.5%; profiles/r1_k2_occupancy.txt).
template <int TU>
__global__ void __launch_bounds__(256, TU == 32 ? 6 : 4) cone_fp_kernel(const FpArgs a) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int WPR = TU / 8;  // 8 u x 4 v warps, TU / 8 of them per 4-row band
  const int iu = blockIdx.x * TU + (w % WPR) * 8 + (lane & 7);
  const int iv = blockIdx.z * (256 / TU) + (w / WPR) * 4 + (lane >> 3);
  const int vl = blockIdx.y;
  if (iu >= a.nu || iv >= a.nv) return;
  double o[3], d[3], t0, t1;
  // a missed ray's zero is stored with its warp's other results (one store
  // instruction per warp).  Register budget (40 at 6 CTAs/SM): only the FP64
  // anchor state, the running total and the layout bit live across chunks;
  // the layout, the fp32 steps, the output address are re-derived where used
  // (fewer spill reloads at each chunk anchor, profiles/r2_k2_traffic.txt).
  const bool hit = cone_ray(a, iu, iv, a.view0 + vl, o, d, t0, t1);
  auto march = [&]() -> float {
    const double span = DADD(t1, -t0);
    const int n = int(ray_sample_count(span, a.step));  // < 2^31 samples per ray
    const double dt = DDIV(span, double(n));

    // Sample k sits at t0 + (k + 1/2) dt; march in index space (fp32) from
    // anchors recomputed in FP64 every 64 samples.
    const double th = t0 + 0.5 * dt;
    const double p0x = (o[0] + th * d[0] - a.ox) / a.sx + 2.0;
    const double p0y = (o[1] + th * d[1] - a.oy) / a.sy + 2.0;
    const double p0z = (o[2] + th * d[2] - a.oz) / a.sz + 2.0;
    const double ddx = dt * d[0] / a.sx, ddy = dt * d[1] / a.sy, ddz = dt * d[2] / a.sz;
    const bool xdom = a.vqT != nullptr && fabs(d[0]) > fabs(d[1]);
    constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23: t = M + floor(p) under round-down
    double total = 0.0;
    for (int k0 = 0; k0 < n; k0 += 64) {
      const int nxyp = a.nxp * a.nyp;
      const float4* vbase = xdom ? a.vqT : a.vq;
      const int sx = xdom ? a.nyp : 1, sy = xdom ? 1 : a.nxp;
      const uint32_t usx = uint32_t(sx), usy = uint32_t(sy), unxyp = uint32_t(nxyp);
      // (sx + sy = nxp + 1 or nyp + 1: the bias is a launch constant per layout)
      const uint32_t mbias = xdom ? a.mbias_t : a.mbias;
      const float fdx = float(ddx), fdy = float(ddy), fdz = float(ddz);
      // chunk anchor split into an integer cell and a small fp32 offset, so
      // sample positions keep ~1e-5 voxel precision anywhere in a 1024^3 grid;
      // per-sample offsets from the cell fit in 32 bits
      const double ax = p0x + double(k0) * ddx, ay = p0y + double(k0) * ddy,
                   az = p0z + double(k0) * ddz;
      const double cx = floor(ax), cy = floor(ay), cz = floor(az);
      const float bx = float(ax - cx), by = float(ay - cy), bz = float(az - cz);
      const float4* cell = vbase + (long long)cz * nxyp + (long long)cy * sy + (long long)cx * sx;
      const int m = min(64, n - k0);
      float sum = 0.0f;
      // samples advance by at most half a voxel, so consecutive samples often
      // stay in the same trilinear cell: re-gather only when the cell changes
      // (lanes that keep their cell are masked off the load and cost no L1
      // wavefronts; K2 is bound by the L1 data pipe)
      int prev = 0x7fffffff;
      float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0;
      float jf = 0.0f;  // float(j), exact (j < 64)
      // x and y of the sample position, floor and fraction as FP32x2 pairs
      // (per lane the scalar FFMA / FADD of the reference order)
      const float2 fdxy = make_float2(fdx, fdy), bxy = make_float2(bx, by);
      const float2 M2 = make_float2(MAGIC, MAGIC), nM2 = make_float2(-MAGIC, -MAGIC);
  #pragma unroll 2
      for (int j = 0; j < m; ++j, jf += 1.0f) {
        const float2 pxy = __ffma2_rn(make_float2(jf, jf), fdxy, bxy);
        const float pz = fmaf(jf, fdz, bz);
        const float2 txy = __fadd2_rd(pxy, M2);
        const float tz = __fadd_rd(pz, MAGIC);
        const float2 fxy = __fadd2_rn(txy, nM2);
        const float2 wxy = __fadd2_rn(pxy, make_float2(-fxy.x, -fxy.y));
        const float tx = txy.x, ty = txy.y, wx = wxy.x, wy = wxy.y, wz = pz - (tz - MAGIC);
        // the three magic biases folded into one constant: exact in 32-bit
        // modular arithmetic, since the true offset fits in an int
        const int off = int(__float_as_uint(tx) * usx + __float_as_uint(ty) * usy +
                            __float_as_uint(tz) * unxyp - mbias);
        if (off != prev) {
          // one IMAD.WIDE per address (a signed 32-bit offset scaled into the
          // 64-bit base) instead of the sign-extend / shift / add chain; the
          // slice z+1 quad one padded slice further
          const float4* c0 = reinterpret_cast<const float4*>(
              reinterpret_cast<const char*>(cell) + (long long)off * 16);
          q0 = __ldg(c0);           // slice z:   x/x+1 at y, y+1
          q1 = __ldg(c0 + nxyp);    // slice z+1
        }
        prev = off;  // (unconditional: a register rename, no move)
        // quads hold (x, y), (x, y+1), (x+1, y), (x+1, y+1): both x-lerps of a
        // slice as one FP32x2 pair (the scalar kernel's per-lane operations)
        const float2 wx2 = make_float2(wx, wx);
        const float2 t0 = __ffma2_rn(wx2, __fadd2_rn(make_float2(q0.z, q0.w), make_float2(-q0.x, -q0.y)),
                                     make_float2(q0.x, q0.y));
        const float2 t1 = __ffma2_rn(wx2, __fadd2_rn(make_float2(q1.z, q1.w), make_float2(-q1.x, -q1.y)),
                                     make_float2(q1.x, q1.y));
        const float c0 = lerpf(t0.x, t0.y, wy);
        const float c1 = lerpf(t1.x, t1.y, wy);
        sum += lerpf(c0, c1, wz);
      }
      total += double(sum);
    }
    return float(total * dt);
  };
  const float res = hit ? march() : 0.0f;
  a.out[((long long)vl * a.nv + iv) * a.nu + iu] = res;
}

// Diagnostic: the per-ray sample count K2 marches (0 = missed ray), same
// ray setup and clip as cone_fp_kernel.  out [n_views][nv][nu].
__global__ void __launch_bounds__(256) cone_ray_samples_kernel(const FpArgs a,
                                                               unsigned long long* out) {
  const int iu = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iv = blockIdx.z * 8 + (threadIdx.x >> 5);
  const int vl = blockIdx.y;
  if (iu >= a.nu || iv >= a.nv) return;
  double o[3], d[3], t0, t1;
  unsigned long long n = 0;
  if (cone_ray(a, iu, iv, a.view0 + vl, o, d, t0, t1))
    n = (unsigned long long)ray_sample_count(DADD(t1, -t0), a.step);
  out[((long long)vl * a.nv + iv) * a.nu + iu] = n;
}

// builds the zero-bordered quad volume K2 gathers from (one pass over V)
__global__ void pad_volume_kernel(const float* __restrict__ vol, float4* __restrict__ vq, int nx,
                                  int ny, int nz) {
  const int nxp = nx + 4, nyp = ny + 4, nzp = nz + 4;
  const long long total = (long long)nxp * nyp * nzp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int px = int(i % nxp);
    const long long r = i / nxp;
    const int py = int(r % nyp), pz = int(r / nyp);
    const int x = px - 2, y = py - 2, z = pz - 2;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (z >= 0 && z < nz) {
      const float* s = vol + (long long)z * ny * nx;
      const bool x0 = x >= 0 && x < nx, x1 = x + 1 >= 0 && x + 1 < nx;
      if (y >= 0 && y < ny) {
        if (x0) q.x = __ldg(s + (long long)y * nx + x);
        if (x1) q.y = __ldg(s + (long long)y * nx + x + 1);
      }
      if (y + 1 >= 0 && y + 1 < ny) {
        if (x0) q.z = __ldg(s + (long long)(y + 1) * nx + x);
        if (x1) q.w = __ldg(s + (long long)(y + 1) * nx + x + 1);
      }
    }
    vq[i] = make_float4(q.x, q.z, q.y, q.w);  // (x, y), (x, y+1), (x+1, y), (x+1, y+1)
  }
}

// the y-fastest copy (FpArgs::vqT), written in its own order (coalesced stores)
__global__ void pad_volume_t_kernel(const float* __restrict__ vol, float4* __restrict__ vqt, int nx,
                                    int ny, int nz) {
  const int nxp = nx + 4, nyp = ny + 4, nzp = nz + 4;
  const long long total = (long long)nxp * nyp * nzp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int py = int(i % nyp);
    const long long r = i / nyp;
    const int px = int(r % nxp), pz = int(r / nxp);
    const int x = px - 2, y = py - 2, z = pz - 2;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (z >= 0 && z < nz) {
      const float* s = vol + (long long)z * ny * nx;
      const bool x0 = x >= 0 && x < nx, x1 = x + 1 >= 0 && x + 1 < nx;
      if (y >= 0 && y < ny) {
        if (x0) q.x = __ldg(s + (long long)y * nx + x);
        if (x1) q.y = __ldg(s + (long long)y * nx + x + 1);
      }
      if (y + 1 >= 0 && y + 1 < ny) {
        if (x0) q.z = __ldg(s + (long long)(y + 1) * nx + x);
        if (x1) q.w = __ldg(s + (long long)(y + 1) * nx + x + 1);
      }
    }
    vqt[i] = make_float4(q.x, q.z, q.y, q.w);
  }
}

// Vt[z][x][y] (row pitch `pitch` >= ny floats) from V[z][y][x]: the y-fastest
// copy the slab-staged K2 reads for x-dominant tiles; also a plain re-pitch
// of V when nx is not a multiple of 4 (TMA strides are 16-byte multiples)
__global__ void transpose_xy_kernel(const float* __restrict__ v, float* __restrict__ vt, int nx,
                                    int ny, int pitch) {
  __shared__ float tile[32][33];
  const int z = blockIdx.z;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const float* src = v + (long long)z * nx * ny;
  float* dst = vt + (long long)z * nx * pitch;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int x = x0 + threadIdx.x, y = y0 + r;
    tile[r][threadIdx.x] = (x < nx && y < ny) ? __ldg(src + (long long)y * nx + x) : 0.0f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int y = y0 + threadIdx.x, x = x0 + r;
    if (x < nx && y < pitch) dst[(long long)x * pitch + y] = tile[threadIdx.x][r];
  }
}

__global__ void repitch_x_kernel(const float* __restrict__ v, float* __restrict__ vx, int nx,
                                 int rows, int pitch) {
  const long long total = (long long)rows * pitch;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = int(i % pitch);
    const long long row = i / pitch;
    vx[i] = x < nx ? __ldg(v + row * nx + x) : 0.0f;
  }
}

#include "cone_fp_slab.cuh"

}  // namespace cone
}  // namespace tgb

// ===========================================================================
// plan

using namespace tgb;
using namespace tgb::cone;

// Host-buffer pipelines: streams and events of one call.
struct HostPipe {
  cudaStream_t cs = nullptr, xs = nullptr, ds = nullptr;
  std::vector<cudaEvent_t> ev;
  explicit HostPipe(int n_events) {
    TG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    TG_CUDA(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
    TG_CUDA(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
    grow(n_events);
  }
  void grow(int n_events) {
    while (int(ev.size()) < n_events) {
      cudaEvent_t e;
      TG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
  }
  ~HostPipe() {
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(cs);
    cudaStreamDestroy(xs);
    cudaStreamDestroy(ds);
  }
};

struct tg_cone_plan {
  int device = 0;
  uint64_t id = 0;
  tg_volume_spec vol{};
  tg_detector2d det{};
  uint64_t n_proj = 0;
  double range = 0, sid = 0, sdd = 0;
  std::vector<double> mats, sources, invs, angles;
  bool circular = true;
  double* d_mats = nullptr;   // 12 x n_proj FP64 matrices (K1's constant bank source)
  double* d_geo = nullptr;    // 12 x n_proj: source + inverse block (FP64)
  int boxV = 0, boxU = 0;     // K1 TMA box
  int k1_k = 16;              // K1 z voxels per thread
  int need_w = 0, need_h = 0;
  // FDK pre-processing
  double* d_cos = nullptr;     // [n_v][n_u]
  double* d_parker = nullptr;  // [n_proj][n_u]
  filt::RowFilter* ramlak = nullptr;
  // scratch
  float4* d_vpad = nullptr;  // K2 quad volume (zero border 2)
  bool k2_dual = true;       // y-fastest copy present (memory permitting)
  bool k2_dual_allowed = true;  // knob "k2_dual"
  bool k2_dual_denied = false;  // the copy did not fit at the last allocation
  int k2_tu = 32;            // K2 CTA width in u (band height 256 / k2_tu rows)
  size_t vpad_elems = 0;
  // K2 implementation: 1 slab-staged (shared-memory boxes), 0 quad-volume L1
  // gathers, -1 (default) = time both once at the plan's first forward
  // projection and keep the faster (identical output bits); knob "k2_impl"
  int k2_impl = -1;
  float* d_vt = nullptr;       // y-fastest copy Vt[z][x][y] (row pitch vt_pitch)
  float* d_vx = nullptr;       // x-fastest re-pitched copy (only when nx % 4 != 0)
  size_t vt_elems = 0, vx_elems = 0;
  int vt_pitch = 0, vx_pitch = 0;
  struct K2Box {
    int tu = 16, wh = 40, t = 8, hz = 0, stages = 2;  // hz: multiple of 4
    bool sized = false;
  } k2box;
  unsigned long long* d_k2_stats = nullptr;  // TG_K2_STATS=1: slab / fallback counters
  ScratchOrder vt_order;
  float* d_pitched = nullptr;  // band copy with a 16-byte row pitch when n_u % 4 != 0
  size_t pitched_elems = 0;
  float* d_stage_in = nullptr;  // host-variant staging (reused across calls)
  size_t stage_in_elems = 0;
  float* d_stage_out = nullptr;
  size_t stage_out_elems = 0;
  uint64_t last_h2d_bytes = 0;  // bytes the last host-buffer call uploaded
  std::unique_ptr<HostPipe> pipe;  // host-buffer pipeline streams / events (reused)
  // Serialises every call on the plan: device-stream calls hold it while they
  // enqueue (the plan-owned scratch below is additionally ordered across
  // streams by ScratchOrder events), host-buffer calls for their whole
  // duration (they share the staging buffers and pipeline streams).
  std::recursive_mutex mu;
  ScratchOrder vpad_order, pitched_order;
};

// The plan keeps one pipeline's streams and events across host-buffer calls
// instead of creating and destroying ~40 CUDA objects per call.  Host-buffer
// calls hold the plan's mutex for their whole duration (they share these and
// the staging buffers), so concurrent calls on one plan serialise.
HostPipe& plan_pipe(tg_cone_plan& p, int n_events) {
  if (!p.pipe) p.pipe.reset(new HostPipe(n_events));
  p.pipe->grow(n_events);
  return *p.pipe;
}

namespace {

// z voxels per K1 thread: 32 (default: half the per-view overhead per update
// of K = 16, 2 CTAs/SM; +10% at c4) or 16 (3 CTAs/SM); env TG_K1_K overrides
// at plan creation.  Slabs aligned to 32 are bitwise equal to the full volume.
int default_k1_k() {
  const char* e = std::getenv("TG_K1_K");
  return (e && std::atoi(e) == 16) ? 16 : 32;
}

// box widths (= shared-memory row pitch in floats); 44 before 48: a pitch of
// 44 words spreads a warp's row-neighbour taps over more banks than 48
// (40.53 vs 40.98 ms at c4, profiles/r1_k1_pitch.txt)
int pick_boxu(int need) {
  static const int choices[] = {44, 48, 80, 112, 176, 240};
  for (int c : choices)
    if (need <= c) return c;
  return 240;
}

void cone_args_base(const tg_cone_plan& p, BpArgs& a) {
  std::memset(&a, 0, sizeof a);
  a.nx = int(p.vol.shape[0]);
  a.ny = int(p.vol.shape[1]);
  a.nz = int(p.vol.shape[2]);
  a.ox = p.vol.origin[0];
  a.oy = p.vol.origin[1];
  a.oz = p.vol.origin[2];
  a.sx = p.vol.spacing[0];
  a.sy = p.vol.spacing[1];
  a.sz = p.vol.spacing[2];
  a.nu = int(p.det.n_u);
  a.nv = int(p.det.n_v);
  a.sid2 = float(p.sid * p.sid);
}

template <int K, int BOXU, bool CIRC>
void launch_bp_t(const CUtensorMap& map, const BpArgs& a, size_t smem, cudaStream_t st, bool pdl) {
  auto fn = cone_bp_kernel<K, BOXU, CIRC>;
  TG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid((a.nx + BX - 1) / BX, (a.ny + BY - 1) / BY, (a.nz + K - 1) / K);
  if (!pdl) {
    fn<<<grid, NTHREADS, smem, st>>>(map, a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TG_CUDA(cudaLaunchKernelEx(&cfg, fn, map, a));
}

template <int K, bool CIRC>
void launch_bp_u(int boxU, const CUtensorMap& map, const BpArgs& a, size_t smem, cudaStream_t st,
                 bool pdl) {
  switch (boxU) {
    case 44: return launch_bp_t<K, 44, CIRC>(map, a, smem, st, pdl);
    case 48: return launch_bp_t<K, 48, CIRC>(map, a, smem, st, pdl);
    case 80: return launch_bp_t<K, 80, CIRC>(map, a, smem, st, pdl);
    case 112: return launch_bp_t<K, 112, CIRC>(map, a, smem, st, pdl);
    case 176: return launch_bp_t<K, 176, CIRC>(map, a, smem, st, pdl);
    default: return launch_bp_t<K, 240, CIRC>(map, a, smem, st, pdl);
  }
}

void launch_bp(int k, bool circ, int boxU, const CUtensorMap& map, const BpArgs& a, size_t smem,
               cudaStream_t st, bool pdl) {
  if (k == 32) {
    if (circ) launch_bp_u<32, true>(boxU, map, a, smem, st, pdl);
    else launch_bp_u<32, false>(boxU, map, a, smem, st, pdl);
  } else {
    if (circ) launch_bp_u<16, true>(boxU, map, a, smem, st, pdl);
    else launch_bp_u<16, false>(boxU, map, a, smem, st, pdl);
  }
}

// Size K1's box from the real footprints of every (tile, view).
void size_box(tg_cone_plan& p) {
  BpArgs a;
  cone_args_base(p, a);
  a.n_views = int(p.n_proj);
  const int kK = p.k1_k;
  const int tx = (a.nx + BX - 1) / BX, ty = (a.ny + BY - 1) / BY, tz = (a.nz + kK - 1) / kK;
  int* d_need = nullptr;
  TG_CUDA(cudaMalloc(&d_need, 2 * sizeof(int)));
  TG_CUDA(cudaMemset(d_need, 0, 2 * sizeof(int)));
  const long long total = (long long)tx * ty * tz * a.n_views;
  const int threads = 256;
  const long long blocks = (total + threads - 1) / threads;
  footprint_kernel<<<unsigned(blocks), threads>>>(a, kK, tx, ty, tz, p.d_mats, d_need);
  TG_LAUNCHED(1);
  int need[2] = {0, 0};
  TG_CUDA(cudaMemcpy(need, d_need, sizeof need, cudaMemcpyDeviceToHost));
  TG_CUDA(cudaFree(d_need));
  p.need_w = need[0];
  p.need_h = need[1];
  p.boxU = pick_boxu(std::max(need[0], 1));
  p.boxV = std::min(std::max(need[1], 2), 256);
  // keep the stage ring small enough for 3 CTAs per SM
  const size_t cap = 72 * 1024;
  while (p.boxV > 2 && size_t(STAGES) * p.boxU * p.boxV * 4 > cap) --p.boxV;
}

// Back-project views [view0, view0 + n_views) of the band buffer (which holds
// every view) into the slab.
// pdl: launch with programmatic stream serialization, so consecutive K1
// launches of a chunked pipeline overlap tail and head (the kernel waits for
// the previous grid only before its epilogue).  Only for a stream whose
// previous kernel does not produce this launch's projections (K1 after K1;
// uploads are ordered by events, which stay full dependencies).  Measured on
// the c4 host pipeline: 44.2 -> 43.3 ms.
void backproject_impl(tg_cone_plan& p, uint64_t z0, uint64_t nz, uint64_t v0, uint64_t n_rows,
                      const float* d_band, float* d_slab, float scale, int accumulate,
                      cudaStream_t st, uint64_t view0 = 0, uint64_t n_views = ~0ull,
                      bool pdl = false) {
  if (n_views == ~0ull) n_views = p.n_proj - view0;
  check(view0 + n_views <= p.n_proj && n_views >= 1, "view range lies outside the geometry");
  check(z0 + nz <= p.vol.shape[2] && nz >= 1, "slab lies outside the volume");
  check(n_rows >= 1 && v0 + n_rows <= p.det.n_v, "detector row band lies outside the detector");
  DeviceGuard dg(p.device);
  std::lock_guard<std::recursive_mutex> lk(p.mu);
  const uint64_t nu = p.det.n_u;
  // TMA needs 16-byte aligned rows: re-pitch the band when n_u % 4 != 0
  const float* src = d_band;
  uint64_t pitch = nu;
  const bool repitch = (nu % 4) != 0 || (reinterpret_cast<uintptr_t>(d_band) % 16) != 0;
  if (repitch) {
    pitch = (nu + 3) / 4 * 4;
    const size_t need = size_t(pitch) * n_rows * p.n_proj;
    p.pitched_order.enter(st);
    if (p.pitched_elems < need) {
      if (p.d_pitched) {
        TG_CUDA(cudaStreamSynchronize(st));  // the buffer's last reader finished (enter above)
        TG_CUDA(cudaFree(p.d_pitched));
      }
      TG_CUDA(cudaMalloc(&p.d_pitched, need * sizeof(float)));
      p.pitched_elems = need;
    }
    TG_CUDA(cudaMemcpy2DAsync(p.d_pitched, pitch * 4, d_band, nu * 4, nu * 4, n_rows * p.n_proj,
                              cudaMemcpyDeviceToDevice, st));
    src = p.d_pitched;
  }
  CUtensorMap map;
  const CUresult cr = encode_tensor_map_3d_f32(&map, src, nu, n_rows, p.n_proj, pitch * 4,
                                               pitch * n_rows * 4, uint32_t(p.boxU),
                                               uint32_t(p.boxV));
  if (cr != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(cr)) + ")");

  BpArgs a;
  cone_args_base(p, a);
  a.nz = int(nz);
  a.z0 = int(z0);
  a.band_v0 = int(v0);
  a.band_rows = int(n_rows);
  a.boxU = p.boxU;
  a.boxV = p.boxV;
  a.magic_row_off = 0u - 0x4B400000u * uint32_t(p.boxU * 4);
  a.sino = src;
  a.row_pitch = (long long)pitch;
  a.view_pitch = (long long)(pitch * n_rows);
  a.vol = d_slab;
  const size_t stage_elems = (size_t(p.boxU) * p.boxV + 31) & ~size_t(31);
  const size_t smem = size_t(STAGES) * stage_elems * 4 + STAGES * 64 + 2 * STAGES * sizeof(uint64_t);
  KernelTimer timer;
  timer.start(st);
  // the bank holds one aligned block of kMaxConstViews views (all of them up
  // to 640), so chunked launches over one block need no re-upload between them
  for (uint64_t c0 = view0; c0 < view0 + n_views;) {
    const uint64_t blk = c0 / kMaxConstViews, b0 = blk * kMaxConstViews;
    const uint64_t bn = std::min<uint64_t>(kMaxConstViews, p.n_proj - b0);
    const uint64_t cn = std::min<uint64_t>(b0 + bn, view0 + n_views) - c0;
    a.n_views = int(cn);
    a.bank_off = int(c0 - b0);
    a.view_base = int(c0);
    a.scale = scale;
    a.accumulate = (c0 == view0) ? accumulate : 1;
    std::lock_guard<std::mutex> lk(g_bank.mu);
    // bank content key: (plan, block, view count)
    g_bank.acquire(p.device, (p.id << 40) ^ (blk << 20) ^ bn, st, c_views, p.d_mats + 12 * b0,
                   bn * 12 * sizeof(double));
    launch_bp(p.k1_k, p.circular, p.boxU, map, a, smem, st, pdl);
    TG_LAUNCHED(1);
    g_bank.release(p.device, st);
    c0 += cn;
  }
  timer.stop();
  if (repitch) p.pitched_order.leave(st);
}

void ensure_vpad(tg_cone_plan& p, cudaStream_t st) {
  // x-fastest and y-fastest quad volumes back to back (8.8x the volume); when
  // that does not fit next to the caller's data (volumes beyond ~1200^3 on a
  // 180 GB B200) fall back to the x-fastest copy alone (4.4x)
  const size_t one = size_t(p.vol.shape[0] + 4) * (p.vol.shape[1] + 4) * (p.vol.shape[2] + 4);
  const bool want = p.k2_dual_allowed;
  if (p.d_vpad) {
    if (p.vpad_elems >= 2 * one) {
      p.k2_dual = want;
      return;
    }
    if (p.vpad_elems >= one && (!want || p.k2_dual_denied)) {
      p.k2_dual = false;
      return;
    }
    TG_CUDA(cudaStreamSynchronize(st));  // the buffer's last reader finished (enter above)
    TG_CUDA(cudaFree(p.d_vpad));
  }
  p.d_vpad = nullptr;
  p.vpad_elems = 0;
  size_t free_b = 0, total_b = 0;
  TG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const bool fits = 2 * one * sizeof(float4) + total_b / 20 <= free_b;
  p.k2_dual = want && fits;
  p.k2_dual_denied = want && !fits;
  const size_t need = one * (p.k2_dual ? 2 : 1);
  TG_CUDA(cudaMalloc(&p.d_vpad, need * sizeof(float4)));
  p.vpad_elems = need;
}

FpArgs fp_args(const tg_cone_plan& p) {
  FpArgs a{};
  const int nx = int(p.vol.shape[0]), ny = int(p.vol.shape[1]), nz = int(p.vol.shape[2]);
  a.nu = int(p.det.n_u);
  a.nv = int(p.det.n_v);
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.ox = p.vol.origin[0];
  a.oy = p.vol.origin[1];
  a.oz = p.vol.origin[2];
  a.sx = p.vol.spacing[0];
  a.sy = p.vol.spacing[1];
  a.sz = p.vol.spacing[2];
  double m = a.sx;  // projector.hpp:103-107
  m = (a.sy < m) ? a.sy : m;
  m = (a.sz < m) ? a.sz : m;
  a.step = 0.5 * m;
  a.geo = p.d_geo;
  a.vq = p.d_vpad;
  a.vqT = p.k2_dual ? p.d_vpad + p.vpad_elems / 2 : nullptr;
  a.nxp = nx + 4;
  a.nyp = ny + 4;
  const uint32_t nxyp = uint32_t(a.nxp) * uint32_t(a.nyp);
  a.mbias = 0x4B400000u * (1u + uint32_t(a.nxp) + nxyp);
  a.mbias_t = 0x4B400000u * (uint32_t(a.nyp) + 1u + nxyp);
  return a;
}

// ---- slab-staged K2 (cone_fp_slab.cuh) ---------------------------------------

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

// Host replica of the producer's box sizing over a sample of views: picks
// the slab thickness T, the transverse box width WH (a template instance)
// and the z extent HZ so that >= 99.8% of (tile, slab) boxes fit and two CTAs
// (two ring stages each) share an SM; the rest gather from global memory
// (same bits).  WH = 8 (mod 32) when rays are at most one voxel apart at the
// isocentre, 12 (mod 32) when they are sparser (a warp's 8 columns then span
// more than 8 banks; offline bank model, profiles/r2_k2_bank_model.txt).
// Environment overrides for experiments: TG_K2_WH, TG_K2_T, TG_K2_HZ,
// TG_K2_STAGES, TG_K2_STATS.
void k2_size_boxes(tg_cone_plan& p) {
  auto& B = p.k2box;
  B.tu = 16;
  const int TU = B.tu, TV = fps::NCONS / TU;
  const int nx = int(p.vol.shape[0]), ny = int(p.vol.shape[1]), nz = int(p.vol.shape[2]);
  const int nu = int(p.det.n_u), nv = int(p.det.n_v);
  const double ray_pitch = p.det.spacing_u * p.sid / p.sdd /
                           std::min(p.vol.spacing[0], p.vol.spacing[1]);
  const bool sparse = ray_pitch > 1.05;
  const int kWH[2] = {sparse ? 44 : 40, sparse ? 76 : 72};
  constexpr int kMaxNeed = 260;
  const size_t fixed = sizeof(fps::RayState) + 1024;
  const size_t budget = 113 * 1024;  // two CTAs per SM
  auto size_for = [&](int T, int& wh, int& hz, uint64_t& total) {
    std::vector<uint64_t> hist(size_t(kMaxNeed) * kMaxNeed, 0);  // [wneed][zneed]
    total = 0;
    const int n_sample = int(std::min<uint64_t>(p.n_proj, 12));
    for (int si = 0; si < n_sample; ++si) {
      const uint64_t view = (uint64_t(si) * p.n_proj) / uint64_t(n_sample);
      const double* src = p.sources.data() + 3 * view;
      const double* M = p.invs.data() + 9 * view;
      const double o[3] = {(src[0] - p.vol.origin[0]) / p.vol.spacing[0],
                           (src[1] - p.vol.origin[1]) / p.vol.spacing[1],
                           (src[2] - p.vol.origin[2]) / p.vol.spacing[2]};
      for (int v0 = 0; v0 < nv; v0 += TV)
        for (int u0 = 0; u0 < nu; u0 += TU) {
          double e[4][3];
          double sx = 0, sy = 0;
          for (int c = 0; c < 4; ++c) {
            const int iu = (c & 1) ? std::min(u0 + TU, nu) - 1 : u0;
            const int iv = (c & 2) ? std::min(v0 + TV, nv) - 1 : v0;
            for (int r = 0; r < 3; ++r)
              e[c][r] = (M[3 * r] * iu + M[3 * r + 1] * iv + M[3 * r + 2]) / p.vol.spacing[r];
            sx += e[c][0];
            sy += e[c][1];
          }
          const bool xdom = std::fabs(sx) > std::fabs(sy);
          const int nd = xdom ? nx : ny;
          double hA[4], hB[4], zA[4], zB[4];
          bool ok = true;
          for (int c = 0; c < 4; ++c) {
            const double ed = xdom ? e[c][0] : e[c][1], eh = xdom ? e[c][1] : e[c][0];
            const double od = xdom ? o[0] : o[1], oh = xdom ? o[1] : o[0];
            const double len = std::sqrt(e[c][0] * e[c][0] + e[c][1] * e[c][1] + e[c][2] * e[c][2]);
            ok = ok && std::fabs(ed) >= 0.3 * len;
            hB[c] = eh / ed;
            hA[c] = oh - od * hB[c];
            zB[c] = e[c][2] / ed;
            zA[c] = o[2] - od * zB[c];
          }
          if (!ok) continue;
          for (int s0 = -3; s0 <= nd; s0 += T) {
            // box planes [s0 - 1, s0 + T + 1] cover both march directions
            double hmin = 1e300, hmax = -1e300, zmin = 1e300, zmax = -1e300;
            for (int c = 0; c < 4; ++c)
              for (int k = 0; k < 2; ++k) {
                const double P = double(s0 - 1 + k * (T + 2));
                const double hh = hA[c] + P * hB[c], zz = zA[c] + P * zB[c];
                hmin = std::min(hmin, hh);
                hmax = std::max(hmax, hh);
                zmin = std::min(zmin, zz);
                zmax = std::max(zmax, zz);
              }
            // slabs entirely outside the volume hold no samples
            if (zmax < -2.0 || zmin > nz + 1.0) continue;
            if (xdom ? (hmax < -2.0 || hmin > ny + 1.0) : (hmax < -2.0 || hmin > nx + 1.0)) continue;
            const int hb = (int(std::floor(hmin)) - 1) & ~3, zb = int(std::floor(zmin)) - 1;
            const int wn = std::min(kMaxNeed - 1, int(std::floor(hmax)) + 3 - hb);
            const int zn = std::min(kMaxNeed - 1, int(std::floor(zmax)) + 3 - zb);
            ++hist[size_t(wn) * kMaxNeed + zn];
            ++total;
          }
        }
    }
    wh = kWH[1];
    hz = 256;
    if (!total) return;
    for (int cand : kWH) {
      uint64_t fit = 0;
      for (int wn = 0; wn <= cand; ++wn)
        for (int zn = 0; zn < kMaxNeed; ++zn) fit += hist[size_t(wn) * kMaxNeed + zn];
      if (fit >= uint64_t(0.999 * double(total))) {
        wh = cand;
        break;
      }
    }
    // smallest HZ with >= 99.8% of all slabs fitting (WH and HZ)
    std::vector<uint64_t> zc(kMaxNeed, 0);
    for (int wn = 0; wn <= wh; ++wn)
      for (int zn = 0; zn < kMaxNeed; ++zn) zc[zn] += hist[size_t(wn) * kMaxNeed + zn];
    uint64_t acc = 0;
    hz = kMaxNeed - 1;
    for (int zn = 0; zn < kMaxNeed; ++zn) {
      acc += zc[zn];
      if (acc >= uint64_t(0.998 * double(total))) {
        hz = zn;
        break;
      }
    }
  };
  auto stage_bytes = [](int wh, int t, int hz) {
    return size_t((wh * (t + 2) * ((hz + 3) & ~3) + 31) & ~31) * 4;
  };
  // thickest slab (fewest per-slab overheads) whose two stages still leave
  // room for two CTAs per SM
  int wh = 0, hz = 0, t = 0;
  uint64_t total = 0;
  const int forced_t = env_int("TG_K2_T", 0);
  for (int T : {8, 6, 4}) {
    if (forced_t && T != forced_t) continue;
    size_for(T, wh, hz, total);
    t = T;
    if (fixed + 2 * stage_bytes(wh, T, hz) <= budget) break;
  }
  if (forced_t && !t) {
    t = forced_t;
    size_for(t, wh, hz, total);
  }
  B.t = t;
  B.wh = env_int("TG_K2_WH", wh);
  B.hz = (std::max(4, std::min(256, env_int("TG_K2_HZ", hz))) + 3) & ~3;
  const size_t sb = stage_bytes(B.wh, B.t, B.hz);
  int stages = int((budget - fixed) / sb);
  stages = std::max(2, std::min(fps::MAX_STAGES, stages));
  B.stages = std::max(1, std::min(fps::MAX_STAGES, env_int("TG_K2_STAGES", stages)));
  B.sized = true;
  if (env_int("TG_K2_STATS", 0))
    std::fprintf(stderr, "[k2] tu %d wh %d t %d hz %d stages %d ray pitch %.2f (sampled slabs %llu)\n",
                 B.tu, B.wh, B.t, B.hz, B.stages, ray_pitch, (unsigned long long)total);
}

template <int TU, int WH>
void launch_fp_slab_t(const CUtensorMap& mx, const CUtensorMap& my, const fps::Args& a, dim3 grid,
                      size_t smem, cudaStream_t st) {
  auto fn = fps::cone_fp_slab_kernel<TU, WH>;
  TG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  fn<<<grid, fps::NTHREADS, smem, st>>>(mx, my, a);
}

void launch_fp_slab(int tu, int wh, const CUtensorMap& mx, const CUtensorMap& my,
                    const fps::Args& a, dim3 grid, size_t smem, cudaStream_t st) {
#define TG_K2_CASE(TU_, WH_)                                  \
  if (tu == TU_ && wh == WH_) {                               \
    launch_fp_slab_t<TU_, WH_>(mx, my, a, grid, smem, st);    \
    return;                                                   \
  }
  TG_K2_CASE(16, 40)
  TG_K2_CASE(16, 72)
  TG_K2_CASE(16, 44)
  TG_K2_CASE(16, 76)
#undef TG_K2_CASE
  check(false, "no slab-staged K2 instance for this (tu, wh)");
}

void forward_slab(tg_cone_plan& p, uint64_t view0, uint64_t nviews, const float* d_vol,
                  float* d_out, cudaStream_t st, bool prep) {
  const int nx = int(p.vol.shape[0]), ny = int(p.vol.shape[1]), nz = int(p.vol.shape[2]);
  p.vt_order.enter(st);
  const int vt_pitch = (ny + 3) & ~3;
  const size_t vt_need = size_t(nz) * nx * vt_pitch;
  const bool need_vx = (nx % 4) != 0 || (reinterpret_cast<uintptr_t>(d_vol) % 16) != 0;
  const int vx_pitch = (nx + 3) & ~3;
  const size_t vx_need = need_vx ? size_t(nz) * ny * vx_pitch : 0;
  if (p.vt_elems < vt_need) {
    if (p.d_vt) {
      TG_CUDA(cudaStreamSynchronize(st));
      TG_CUDA(cudaFree(p.d_vt));
      p.d_vt = nullptr;
    }
    TG_CUDA(cudaMalloc(&p.d_vt, vt_need * sizeof(float)));
    p.vt_elems = vt_need;
    prep = true;
  }
  if (p.vx_elems < vx_need) {
    if (p.d_vx) {
      TG_CUDA(cudaStreamSynchronize(st));
      TG_CUDA(cudaFree(p.d_vx));
      p.d_vx = nullptr;
    }
    TG_CUDA(cudaMalloc(&p.d_vx, vx_need * sizeof(float)));
    p.vx_elems = vx_need;
    prep = true;
  }
  p.vt_pitch = vt_pitch;
  p.vx_pitch = vx_pitch;
  if (prep) {
    dim3 tg((nx + 31) / 32, (vt_pitch + 31) / 32, nz);
    transpose_xy_kernel<<<tg, dim3(32, 8), 0, st>>>(d_vol, p.d_vt, nx, ny, vt_pitch);
    TG_LAUNCHED(1);
    if (need_vx) {
      repitch_x_kernel<<<148 * 8, 256, 0, st>>>(d_vol, p.d_vx, nx, nz * ny, vx_pitch);
      TG_LAUNCHED(1);
    }
  }
  if (!p.k2box.sized) k2_size_boxes(p);
  const auto& B = p.k2box;
  CUtensorMap mx, my;
  const float* vxb = need_vx ? p.d_vx : d_vol;
  const int xp = need_vx ? vx_pitch : nx;
  // boxes laid out [dominant][z][transverse]: the maps walk (h, z, d) with
  // permuted strides over V[z][y][x] (h = x, d = y) and Vt[z][x][y] (h = y, d = x)
  check(encode_tensor_map_3d_f32(&mx, vxb, nx, nz, ny, uint64_t(xp) * ny * 4, uint64_t(xp) * 4,
                                 B.wh, B.hz, B.t + 2) == CUDA_SUCCESS,
        "cuTensorMapEncodeTiled failed (K2 x-fastest volume)");
  check(encode_tensor_map_3d_f32(&my, p.d_vt, ny, nz, nx, uint64_t(vt_pitch) * nx * 4,
                                 uint64_t(vt_pitch) * 4, B.wh, B.hz, B.t + 2) == CUDA_SUCCESS,
        "cuTensorMapEncodeTiled failed (K2 y-fastest volume)");
  fps::Args a{};
  a.f = fp_args(p);
  a.vol = d_vol;
  a.boxZ = B.hz;
  a.T = B.t;
  a.stages = B.stages;
  const bool stats = env_int("TG_K2_STATS", 0) != 0;
  if (stats) {
    if (!p.d_k2_stats) TG_CUDA(cudaMalloc(&p.d_k2_stats, 4 * sizeof(unsigned long long)));
    TG_CUDA(cudaMemsetAsync(p.d_k2_stats, 0, 4 * sizeof(unsigned long long), st));
    a.stats = p.d_k2_stats;
  }
  const size_t stage_elems = size_t((B.wh * (B.t + 2) * B.hz + 31) & ~31);
  const size_t smem = stage_elems * 4 * B.stages + sizeof(fps::RayState) +
                      sizeof(fps::StageHdr) * fps::MAX_STAGES + sizeof(fps::CtaHdr) +
                      2 * fps::MAX_STAGES * sizeof(uint64_t);
  const int TV = fps::NCONS / B.tu;
  KernelTimer timer;
  timer.start(st);
  for (uint64_t c0 = 0; c0 < nviews; c0 += 65535) {
    const uint64_t cn = std::min<uint64_t>(65535, nviews - c0);
    a.f.view0 = int(view0 + c0);
    a.f.out = d_out + c0 * p.det.n_u * p.det.n_v;
    dim3 grid((a.f.nu + B.tu - 1) / B.tu, unsigned(cn), (a.f.nv + TV - 1) / TV);
    launch_fp_slab(B.tu, B.wh, mx, my, a, grid, smem, st);
    TG_LAUNCHED(1);
  }
  timer.stop();
  if (stats) {
    unsigned long long h[4];
    TG_CUDA(cudaMemcpyAsync(h, p.d_k2_stats, sizeof h, cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[k2] slabs %llu global-slabs %llu global-ctas %llu\n", h[0], h[1], h[2]);
  }
  p.vt_order.leave(st);
}

void forward_quad(tg_cone_plan& p, uint64_t view0, uint64_t nviews, const float* d_vol,
                  float* d_out, cudaStream_t st, bool pad);

// One-time choice between the two K2 implementations (same output bits):
// each runs twice on twelve blocks of consecutive views spread over the
// plan (the second run is timed, after the volume preparation of the first),
// the faster is kept and
// the other's scratch volume freed.  Slab on ties (2x the volume of scratch
// against the quad kernel's 8.8x), and whenever the quad volumes do not fit
// or the stream is being captured.
void k2_autotune(tg_cone_plan& p, const float* d_vol, cudaStream_t st) {
  p.k2_impl = 1;
  if (ScratchOrder::capturing(st)) return;
  const uint64_t per_view = p.det.n_u * p.det.n_v;
  // twelve blocks of consecutive views spread evenly over the plan's range
  // (the quad kernel's speed varies with the view angle, the slab kernel's
  // hardly), each block >= ~20k slab CTAs so that launch tails do not decide
  const uint64_t tiles = ((p.det.n_u + 15) / 16) * ((p.det.n_v + 15) / 16);
  const int nblk = p.n_proj >= 48 ? 12 : 1;
  const uint64_t want = std::max<uint64_t>(4, (20000 + tiles - 1) / tiles);
  const int blk = int(std::min<uint64_t>(want, p.n_proj / uint64_t(nblk)));
  const int ns = blk;
  const size_t one = size_t(p.vol.shape[0] + 4) * (p.vol.shape[1] + 4) * (p.vol.shape[2] + 4) * 16;
  size_t free_b = 0, total_b = 0;
  TG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (one + size_t(ns) * per_view * 4 + total_b / 10 > free_b) return;
  float* scratch = nullptr;
  TG_CUDA(cudaMalloc(&scratch, size_t(ns) * per_view * sizeof(float)));
  cudaEvent_t a, b;
  TG_CUDA(cudaEventCreate(&a));
  TG_CUDA(cudaEventCreate(&b));
  float ms[2] = {0.f, 0.f};
  for (int impl = 0; impl < 2; ++impl) {
    for (int rep = 0; rep < 2; ++rep) {
      TG_CUDA(cudaEventRecord(a, st));
      for (int i = 0; i < nblk; ++i) {
        const uint64_t v = uint64_t(i) * (p.n_proj - blk) / uint64_t(std::max(1, nblk - 1));
        if (impl == 0)
          forward_quad(p, v, blk, d_vol, scratch, st, rep == 0 && i == 0);
        else
          forward_slab(p, v, blk, d_vol, scratch, st, rep == 0 && i == 0);
      }
      TG_CUDA(cudaEventRecord(b, st));
      TG_CUDA(cudaEventSynchronize(b));
      TG_CUDA(cudaEventElapsedTime(&ms[impl], a, b));
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  TG_CUDA(cudaFree(scratch));
  // the faster one; slab on near-ties (within 3%) only when the quad volumes
  // are a large share of the device (8.8x the volume against the slab's 2x).
  // Short view blocks understate the quad kernel's lead at c4 (4% sampled,
  // 9% over a whole scan), so the tie band must not cover that case.
  const bool big = 2 * one > total_b / 8;
  p.k2_impl = (ms[0] < (big ? 0.97f : 1.0f) * ms[1]) ? 0 : 1;
  // drop the loser's scratch (the stream is idle: synchronised above)
  if (p.k2_impl == 1 && p.d_vpad) {
    TG_CUDA(cudaFree(p.d_vpad));
    p.d_vpad = nullptr;
    p.vpad_elems = 0;
  } else if (p.k2_impl == 0) {
    if (p.d_vt) TG_CUDA(cudaFree(p.d_vt));
    if (p.d_vx) TG_CUDA(cudaFree(p.d_vx));
    p.d_vt = p.d_vx = nullptr;
    p.vt_elems = p.vx_elems = 0;
  }
  if (env_int("TG_K2_STATS", 0))
    std::fprintf(stderr, "[k2] autotune over %d views: quad %.3f ms, slab %.3f ms -> %s\n", nblk * blk,
                 ms[0], ms[1], p.k2_impl ? "slab" : "quad");
}

void forward_impl(tg_cone_plan& p, uint64_t view0, uint64_t nviews, const float* d_vol,
                  float* d_out, cudaStream_t st, bool pad = true) {
  check(view0 + nviews <= p.n_proj && nviews >= 1, "view range lies outside the geometry");
  DeviceGuard dg(p.device);
  std::lock_guard<std::recursive_mutex> lk(p.mu);
  if (p.k2_impl < 0) {
    k2_autotune(p, d_vol, st);
    pad = true;  // re-prepare the chosen layout for this volume
  }
  if (p.k2_impl == 1)
    forward_slab(p, view0, nviews, d_vol, d_out, st, pad);
  else
    forward_quad(p, view0, nviews, d_vol, d_out, st, pad);
}

void forward_quad(tg_cone_plan& p, uint64_t view0, uint64_t nviews, const float* d_vol,
                  float* d_out, cudaStream_t st, bool pad) {
  p.vpad_order.enter(st);
  ensure_vpad(p, st);
  const int nx = int(p.vol.shape[0]), ny = int(p.vol.shape[1]), nz = int(p.vol.shape[2]);
  if (pad) {
    pad_volume_kernel<<<148 * 8, 256, 0, st>>>(d_vol, p.d_vpad, nx, ny, nz);
    if (p.k2_dual) {
      pad_volume_t_kernel<<<148 * 8, 256, 0, st>>>(d_vol, p.d_vpad + p.vpad_elems / 2, nx, ny, nz);
      TG_LAUNCHED(1);
    }
    TG_LAUNCHED(1);
  }
  FpArgs a = fp_args(p);
  KernelTimer timer;
  timer.start(st);
  // one launch per block of views (TG_K2_QBLK, default all; grid limit 65535)
  const uint64_t qblk = uint64_t(std::max(1, std::min(65535, env_int("TG_K2_QBLK", 65535))));
  for (uint64_t c0 = 0; c0 < nviews; c0 += qblk) {
    const uint64_t cn = std::min<uint64_t>(qblk, nviews - c0);
    a.view0 = int(view0 + c0);
    a.out = d_out + c0 * p.det.n_u * p.det.n_v;
    const int TU = p.k2_tu;
    dim3 grid((a.nu + TU - 1) / TU, unsigned(cn), (a.nv + 256 / TU - 1) / (256 / TU));
    if (TU == 64)
      cone_fp_kernel<64><<<grid, 256, 0, st>>>(a);
    else
      cone_fp_kernel<32><<<grid, 256, 0, st>>>(a);
    TG_LAUNCHED(1);
  }
  timer.stop();
  p.vpad_order.leave(st);
}

void ensure_fdk_weights(tg_cone_plan& p, bool use_parker) {
  tg_cone_geometry g{p.vol, p.det, p.n_proj, p.range, p.sid, p.sdd, p.mats.data(), p.sources.data(),
                     p.invs.data(), p.angles.data()};
  std::lock_guard<std::recursive_mutex> lk(p.mu);
  if (!p.d_cos) {
    std::vector<double> cw(p.det.n_u * p.det.n_v);
    cosine_weights_cone(g, cw.data());
    TG_CUDA(cudaMalloc(&p.d_cos, cw.size() * sizeof(double)));
    TG_CUDA(cudaMemcpy(p.d_cos, cw.data(), cw.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (use_parker && !p.d_parker) {
    std::vector<double> pw(p.n_proj * p.det.n_u);
    parker_weights_cone(g, pw.data());  // throws the reference's range errors
    TG_CUDA(cudaMalloc(&p.d_parker, pw.size() * sizeof(double)));
    TG_CUDA(cudaMemcpy(p.d_parker, pw.data(), pw.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (!p.ramlak) {
    const uint64_t P = next_pow2(2 * p.det.n_u);
    std::vector<double> w(P);
    ramlak_weights(P, p.det.spacing_u, w.data());
    p.ramlak = filt::create(p.det.n_u, P, w.data(), p.device);
  }
}

void prefilter_impl(tg_cone_plan& p, const float* d_in, float* d_out, bool use_parker, uint64_t v0,
                    uint64_t n_rows, uint64_t view0, uint64_t n_views, cudaStream_t st,
                    filt::RowLayout lay = filt::RowLayout{}, bool pdl = false) {
  check(n_rows >= 1 && v0 + n_rows <= p.det.n_v, "detector row band lies outside the detector");
  ensure_fdk_weights(p, use_parker);
  DeviceGuard dg(p.device);
  filt::PreWeights pw;
  pw.cos = p.d_cos;
  pw.cos_row0 = v0;
  pw.rows_per_view = n_rows;
  pw.parker = use_parker ? p.d_parker + view0 * p.det.n_u : nullptr;
  filt::apply(*p.ramlak, d_in, d_out, n_views * n_rows, &pw, st, lay, pdl);
}

double fdk_scale(const tg_cone_plan& p, bool use_parker) {  // pipelines.hpp:80-81
  return p.range / double(p.n_proj) * (p.sdd / p.sid) * (use_parker ? 1.0 : 0.5);
}

// Host-buffer pipelines: views in chunks, H2D on a copy stream overlapped with
// the kernels of the previous chunk.  Staging buffers are per call.


float* ensure_buffer(float*& buf, size_t& have, size_t need) {
  if (have < need) {
    if (buf) TG_CUDA(cudaFree(buf));
    TG_CUDA(cudaMalloc(&buf, need * sizeof(float)));
    have = need;
  }
  return buf;
}

void slab_rows(const tg_cone_geometry& g, uint64_t z0, uint64_t nz, uint64_t* v0,
               uint64_t* n_rows);
void phased_backproject(tg_cone_plan& p, uint64_t z0, uint64_t nz, uint64_t v0, uint64_t n_rows,
                        const float* h_band, float* h_slab, float* d_band, float* d_slab,
                        uint64_t h_view_pitch, bool fdk, bool use_parker, float scale);

// Host-buffer back-projection / FDK of z-slab [z0, z0+nz) from detector rows
// [v0, v0+n_rows) of every view (h_band [n_proj][n_rows][n_u] -> h_slab; with
// h_view_pitch > 0 the band's views sit h_view_pitch elements apart, e.g. the
// rows of a full host sinogram).  Views travel in ~8 chunks on a copy stream;
// K3 (FDK) and K1 of chunk c run while chunk c+1 is in flight, K1
// accumulating chunk after chunk.  Device staging buffers are owned by the
// plan and reused across calls.
void host_backproject(tg_cone_plan& p, uint64_t z0, uint64_t nz, uint64_t v0, uint64_t n_rows,
                      const float* h_band, float* h_slab, int fdk, bool use_parker,
                      uint64_t h_view_pitch = 0) {
  check(z0 + nz <= p.vol.shape[2] && nz >= 1, "slab lies outside the volume");
  check(n_rows >= 1 && v0 + n_rows <= p.det.n_v, "detector row band lies outside the detector");
  DeviceGuard dg(p.device);
  // the whole call: staging buffers and pipeline streams are the plan's
  std::lock_guard<std::recursive_mutex> call_lock(p.mu);
  const uint64_t np = p.n_proj, per_view = p.det.n_u * n_rows;
  const uint64_t nvox = p.vol.shape[0] * p.vol.shape[1] * nz;
  if (fdk) ensure_fdk_weights(p, use_parker);
  // View chunks: a geometric head (np/32, np/16, then np/8 each) so K3 / K1
  // start after a short first upload (compute per view outpaces the copy
  // engine from then on: c4 FDK 0.092 vs 0.076 ms per view), and two np/8
  // chunks at the end, whose K1 runs per z-part while finished parts download.
  const uint64_t chunk = std::max<uint64_t>(1, (np + 7) / 8);
  std::vector<uint64_t> starts;
  {
    const uint64_t tail0 = np > 2 * chunk ? np - 2 * chunk : 0;
    uint64_t w = 0, c = std::max<uint64_t>(1, (np + 31) / 32);
    while (w < tail0) {
      starts.push_back(w);
      w += std::min(c, tail0 - w);
      c = std::min(chunk, 2 * c);
    }
    for (uint64_t t = tail0; t < np; t += chunk) starts.push_back(t);
    starts.push_back(np);
  }
  const int n_chunks = int(starts.size()) - 1;
  float* d_band = ensure_buffer(p.d_stage_in, p.stage_in_elems, np * per_view);
  float* d_slab = ensure_buffer(p.d_stage_out, p.stage_out_elems, nvox);
  if (h_view_pitch == 0) h_view_pitch = per_view;
  // centre-out phased pipeline (BP: footprint uploads; FDK: whole rows, each
  // new row segment weighted and filtered as it lands — needs the register
  // FFT path of K3 for strided row segments)
  if (np >= 8 && (!fdk || (p.ramlak->P >= 512 && p.ramlak->P <= 8192)) &&
      std::getenv("TG_HOST_NOPHASE") == nullptr) {
    phased_backproject(p, z0, nz, v0, n_rows, h_band, h_slab, d_band, d_slab, h_view_pitch, fdk != 0,
                       use_parker, fdk ? float(fdk_scale(p, use_parker)) : 1.0f);
    return;
  }
  // The device-to-host copy of the slab overlaps the last views' K1: the
  // final two view chunks are back-projected z-part by z-part (32-aligned,
  // so every K1 tile is the one the whole-slab launch would run) and each
  // part leaves as soon as its last view is in.
  const uint64_t plane = p.vol.shape[0] * p.vol.shape[1];
  const bool split = n_chunks >= 3 && nz >= 64;
  const int n_head = split ? n_chunks - 2 : n_chunks;
  const uint64_t pz = split ? std::max<uint64_t>(32, (nz / 8 + 31) / 32 * 32) : nz;
  const int n_parts = int((nz + pz - 1) / pz);
  HostPipe& hp = plan_pipe(p, n_chunks + n_parts);
  const float scale = fdk ? float(fdk_scale(p, use_parker)) : 1.0f;
  p.last_h2d_bytes = np * per_view * sizeof(float);
  for (int c = 0; c < n_chunks; ++c) {
    const uint64_t w0 = starts[c], wn = starts[c + 1] - w0;
    if (h_view_pitch == per_view)
      TG_CUDA(cudaMemcpyAsync(d_band + w0 * per_view, h_band + w0 * per_view,
                              wn * per_view * sizeof(float), cudaMemcpyHostToDevice, hp.xs));
    else
      TG_CUDA(cudaMemcpy2DAsync(d_band + w0 * per_view, per_view * sizeof(float),
                                h_band + w0 * h_view_pitch, h_view_pitch * sizeof(float),
                                per_view * sizeof(float), wn, cudaMemcpyHostToDevice, hp.xs));
    TG_CUDA(cudaEventRecord(hp.ev[c], hp.xs));
  }
  for (int c = 0; c < n_chunks; ++c) {
    const uint64_t w0 = starts[c], wn = starts[c + 1] - w0;
    TG_CUDA(cudaStreamWaitEvent(hp.cs, hp.ev[c], 0));
    float* part = d_band + w0 * per_view;
    if (fdk) prefilter_impl(p, part, part, use_parker, v0, n_rows, w0, wn, hp.cs);
    if (c < n_head) backproject_impl(p, z0, nz, v0, n_rows, d_band, d_slab, scale, c > 0, hp.cs, w0, wn);
  }
  if (!split) {
    TG_CUDA(cudaMemcpyAsync(h_slab, d_slab, nvox * sizeof(float), cudaMemcpyDeviceToHost, hp.cs));
  } else {
    const uint64_t w_tail = starts[n_head];
    for (int q = 0; q < n_parts; ++q) {
      const uint64_t zq = uint64_t(q) * pz, nq = std::min(pz, nz - zq);
      // parts after the first follow a K1, not the K3 producing their input:
      // programmatic dependent launch overlaps their heads with its tail
      backproject_impl(p, z0 + zq, nq, v0, n_rows, d_band, d_slab + zq * plane, scale, 1, hp.cs,
                       w_tail, np - w_tail, q > 0);
      TG_CUDA(cudaEventRecord(hp.ev[n_chunks + q], hp.cs));
      TG_CUDA(cudaStreamWaitEvent(hp.xs, hp.ev[n_chunks + q], 0));
      TG_CUDA(cudaMemcpyAsync(h_slab + zq * plane, d_slab + zq * plane, nq * plane * sizeof(float),
                              cudaMemcpyDeviceToHost, hp.xs));
    }
    TG_CUDA(cudaStreamSynchronize(hp.xs));
  }
  TG_CUDA(cudaStreamSynchronize(hp.cs));
}

// Detector rows a z-slab can touch: project the slab's 8 corners on every
// view (FP64).  For w > 0 the projective image of the box lies in their hull;
// keep taps floor(v), floor(v)+1 plus one row of margin on each side.
void slab_rows(const tg_cone_geometry& g, uint64_t z0, uint64_t nz, uint64_t* v0,
               uint64_t* n_rows) {
  const tg_volume_spec& vol = g.volume;
  check(z0 + nz <= vol.shape[2] && nz >= 1, "slab lies outside the volume");
  double vmin = 1e300, vmax = -1e300;
  bool behind = false;
  const double xs[2] = {vol.origin[0], vol.origin[0] + double(vol.shape[0] - 1) * vol.spacing[0]};
  const double ys[2] = {vol.origin[1], vol.origin[1] + double(vol.shape[1] - 1) * vol.spacing[1]};
  const double zs[2] = {vol.origin[2] + double(z0) * vol.spacing[2],
                        vol.origin[2] + double(z0 + nz - 1) * vol.spacing[2]};
  for (uint64_t i = 0; i < g.n_projections; ++i) {
    const double* m = g.matrices + 12 * i;
    for (int c = 0; c < 8; ++c) {
      const double x = xs[c & 1], y = ys[(c >> 1) & 1], z = zs[c >> 2];
      const double hy = m[4] * x + m[5] * y + m[6] * z + m[7];
      const double hz = m[8] * x + m[9] * y + m[10] * z + m[11];
      if (!(hz > 0.0)) {
        behind = true;
        continue;
      }
      vmin = std::min(vmin, hy / hz);
      vmax = std::max(vmax, hy / hz);
    }
  }
  long long lo = 0, hi = (long long)g.detector.n_v - 1;
  if (!behind) {
    lo = std::max<long long>(0, (long long)std::floor(vmin) - 1);
    hi = std::min<long long>((long long)g.detector.n_v - 1, (long long)std::floor(vmax) + 2);
  }
  if (hi < lo) {  // the slab never reaches the detector: keep a single row
    lo = 0;
    hi = 0;
  }
  *v0 = uint64_t(lo);
  *n_rows = uint64_t(hi - lo + 1);
}

// Back-projection from host buffers with the upload ordered centre-out in z.
// No voxel is final before its last view has arrived, so a view-ordered
// upload leaves the whole download (0.54 GB at c4) behind the last byte of the
// upload.  Here the middle 64 slices' detector rows go first (all views, in 4
// view chunks, each chunk back-projected as it lands), then two rings of
// slices below and above, each uploading only the rows it needs beyond those
// already resident (rows are monotone in z).  A ring's slices are final after
// its last chunk and download while the next rings upload; the last ring's
// final chunk runs per 32-slice part so its download starts part by part.
// The centre rows are few (the cone is narrowest there), so K1 starts after a
// short upload and then trails the copy engine.  Parts are 32-aligned from the
// slab start: every K1 tile is the one the whole-slab launch would run.
void phased_backproject(tg_cone_plan& p, uint64_t z0, uint64_t nz, uint64_t v0, uint64_t n_rows,
                        const float* h_band, float* h_slab, float* d_band, float* d_slab,
                        uint64_t h_view_pitch, bool fdk, bool use_parker, float scale) {
  struct Range {
    uint64_t z, n;  // slab-relative slices
  };
  const uint64_t np = p.n_proj, nu = p.det.n_u;
  const uint64_t plane = p.vol.shape[0] * p.vol.shape[1];
  const uint64_t units = (nz + 31) / 32;
  auto slices = [&](uint64_t u0, uint64_t u1) {  // unit range -> slice range (clipped)
    const uint64_t a = u0 * 32, b = std::min(nz, u1 * 32);
    return Range{a, b > a ? b - a : 0};
  };
  std::vector<std::vector<Range>> phases;
  // schedule knobs (experiments; defaults measured best at c4, round 2: the BP
  // path 2 / 3 / 4 (profiles/r2_e2e_sweep.jsonl), the FDK path — PCIe-bound
  // with whole detector rows — 1 / 5 / 3 (profiles/r2_e2e_fdk_sweep.jsonl))
  auto knob = [](const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::max(1, std::atoi(e)) : dflt;
  };
  const uint64_t centre = std::min<uint64_t>(units, uint64_t(knob("TG_E2E_CENTRE_UNITS", fdk ? 1 : 2)));
  const uint64_t lo_u = (units - centre) / 2, hi_u = lo_u + centre;
  phases.push_back({slices(lo_u, hi_u)});
  const uint64_t below = lo_u, above = units - hi_u;
  const int kRings = knob("TG_E2E_RINGS", fdk ? 5 : 3);
  for (int r = 0; r < kRings; ++r) {
    const uint64_t b0 = below * r / kRings, b1 = below * (r + 1) / kRings;
    const uint64_t a0 = above * r / kRings, a1 = above * (r + 1) / kRings;
    std::vector<Range> ph;
    if (b1 > b0) ph.push_back(slices(lo_u - b1, lo_u - b0));
    if (a1 > a0) ph.push_back(slices(hi_u + a0, hi_u + a1));
    if (!ph.empty()) phases.push_back(ph);
  }
  const int kChunks = knob("TG_E2E_CHUNKS", fdk ? 3 : 4);
  const int kGroup = knob("TG_E2E_GROUP", 8);
  // view chunks are whole copy groups (a group's residency is tracked for all
  // of its views at once)
  const uint64_t chunk = ((np + kChunks - 1) / kChunks + kGroup - 1) / kGroup * kGroup;
  const int n_chunks = int((np + chunk - 1) / chunk);
  // BP: phases from the third on run in fewer, larger view chunks — the copy
  // engine is ahead of K1 by then, and the 32 K1 launches of the uniform
  // schedule cost 40.2 ms serialised against 36.5 for one launch (launch
  // tails).  c4: 40.27 -> 39.42 ms with 2 chunks from phase 2 (1 chunk 45.1,
  // from phase 1 41.5; scripts/e2e_variants.py --late / --late2,
  // profiles/r2_e2e_late_sweep.jsonl).  The FDK schedule, bound by the copy
  // engine (whole detector rows), keeps uniform chunks: 45.4 ms against
  // 46.8-51.9 with fewer late chunks.
  const int kChunksLate = knob("TG_E2E_CHUNKS_LATE", fdk ? kChunks : 2);
  const int kLateFrom = knob("TG_E2E_LATE_FROM", 2);
  // (FDK: whole early chunks, each its own copy group)
  const uint64_t chunk_late =
      fdk ? chunk * uint64_t((n_chunks + kChunksLate - 1) / kChunksLate)
          : ((np + kChunksLate - 1) / kChunksLate + kGroup - 1) / kGroup * kGroup;
  const int n_chunks_late = int((np + chunk_late - 1) / chunk_late);
  const int n_phases = int(phases.size());
  // consecutive K1 launches overlap (programmatic dependent launch); never a
  // K1 right after the K3 that produces its rows (FDK)
  const bool kPdl = std::getenv("TG_E2E_NOPDL") == nullptr;
  // FDK: one copy group per view chunk (its row segments are filtered in one
  // K3 launch each) and whole detector rows (the filter runs along u)
  const uint64_t G = fdk ? chunk : uint64_t(kGroup);

  // Per-view footprints.  K1 reads taps floor(u), floor(u)+1 (and the same in
  // v) of voxel centres only, and for w > 0 the projective image of a box of
  // voxel centres lies in the hull of its 8 projected corners, so a view's
  // upload can stop at its own footprint: columns from the whole slab (one
  // range per view for every phase), rows per phase, one column / row of
  // margin below and two above as in slab_rows.  At c4 this ships 35% fewer
  // bytes than the slab's row band.  A view with a corner at w <= 0 ships the
  // caller's full band.  Copy groups of G consecutive views (one 3D copy
  // per group and row segment, union of the group's ranges) keep the number
  // of copies small; the columns are widened to 64-byte boundaries.
  const double* vo = p.vol.origin;
  const double* vs = p.vol.spacing;
  const double xs[2] = {vo[0], vo[0] + double(p.vol.shape[0] - 1) * vs[0]};
  const double ys[2] = {vo[1], vo[1] + double(p.vol.shape[1] - 1) * vs[1]};
  auto zc = [&](uint64_t z) { return vo[2] + double(z0 + z) * vs[2]; };
  // footprint of slices [za, zb] (slab-relative, inclusive) on view i:
  // {u lo, u hi, v lo, v hi} as half-open detector index ranges, clamped
  struct Foot {
    int64_t ua, ub, va, vb;
  };
  auto footprint = [&](uint64_t i, uint64_t za, uint64_t zb) {
    const double* m = p.mats.data() + 12 * i;
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
    bool behind = false;
    for (int c = 0; c < 8; ++c) {
      const double x = xs[c & 1], y = ys[(c >> 1) & 1], z = zc((c >> 2) ? zb : za);
      const double hx = m[0] * x + m[1] * y + m[2] * z + m[3];
      const double hy = m[4] * x + m[5] * y + m[6] * z + m[7];
      const double hz = m[8] * x + m[9] * y + m[10] * z + m[11];
      if (!(hz > 0.0)) {
        behind = true;
        break;
      }
      umin = std::min(umin, hx / hz);
      umax = std::max(umax, hx / hz);
      vmin = std::min(vmin, hy / hz);
      vmax = std::max(vmax, hy / hz);
    }
    const int64_t band_lo = int64_t(v0), band_hi = int64_t(v0 + n_rows);
    if (behind || !(umax - umin < 1e15) || !(vmax - vmin < 1e15))
      return Foot{0, int64_t(nu), band_lo, band_hi};
    auto clampi = [](double x, int64_t lo, int64_t hi) {
      return int64_t(std::max<double>(double(lo), std::min<double>(double(hi), x)));
    };
    Foot f;
    f.ua = clampi(std::floor(umin) - 1, 0, int64_t(nu));
    f.ub = clampi(std::floor(umax) + 3, 0, int64_t(nu));
    f.va = clampi(std::floor(vmin) - 1, band_lo, band_hi);
    f.vb = clampi(std::floor(vmax) + 3, band_lo, band_hi);
    if (f.vb < f.va) f.vb = f.va;
    if (f.ub < f.ua) f.ub = f.ua;
    return f;
  };
  const uint64_t n_groups = (np + G - 1) / G;
  // group columns: union over the group's views of the whole slab's footprint
  std::vector<int64_t> g_ua(n_groups, int64_t(nu)), g_ub(n_groups, 0);
  std::vector<int64_t> g_lo(n_groups, 0), g_hi(n_groups, 0);  // resident rows (absolute)
  for (uint64_t i = 0; i < np; ++i) {
    const Foot f = footprint(i, 0, nz - 1);
    const uint64_t gi = i / G;
    g_ua[gi] = std::min(g_ua[gi], f.ua);
    g_ub[gi] = std::max(g_ub[gi], f.ub);
  }
  for (uint64_t gi = 0; gi < n_groups; ++gi) {
    g_ua[gi] = fdk ? 0 : g_ua[gi] / 16 * 16;
    g_ub[gi] = fdk ? int64_t(nu) : std::min<int64_t>(int64_t(nu), (g_ub[gi] + 15) / 16 * 16);
  }

  HostPipe& hp = plan_pipe(p, n_phases * std::max(n_chunks, n_chunks_late) + n_phases + int(units) + 1);
  cudaStream_t ds = hp.ds;  // downloads: concurrent with the uploads on xs
  int ev = 0;
  uint64_t shipped = 0;
  const uint64_t row_bytes = nu * sizeof(float);
  auto download = [&](const Range& r) {
    TG_CUDA(cudaMemcpyAsync(h_slab + r.z * plane, d_slab + r.z * plane, r.n * plane * sizeof(float),
                            cudaMemcpyDeviceToHost, ds));
  };
  // rows [ra, rb) of views [w0, w0 + wn) just uploaded, to be weighted and
  // filtered in place once they land (FDK)
  struct Fresh {
    uint64_t w0, wn;  // views
    int64_t ra, rb;   // rows
  };
  std::vector<Fresh> fresh;
  auto upload = [&](uint64_t w0, uint64_t wn, int64_t ua, int64_t ub, int64_t ra, int64_t rb) {
    if (ub <= ua || rb <= ra || wn == 0) return;
    if (fdk) fresh.push_back({w0, wn, ra, rb});
    cudaMemcpy3DParms cp = {};
    // host views sit h_view_pitch elements apart (the band itself, or the
    // rows of a full sinogram)
    cp.srcPtr = make_cudaPitchedPtr(const_cast<float*>(h_band), row_bytes, row_bytes,
                                    h_view_pitch / nu);
    cp.dstPtr = make_cudaPitchedPtr(d_band, row_bytes, row_bytes, n_rows);
    cp.srcPos = make_cudaPos(size_t(ua) * sizeof(float), size_t(ra - int64_t(v0)), size_t(w0));
    cp.dstPos = cp.srcPos;
    cp.extent = make_cudaExtent(size_t(ub - ua) * sizeof(float), size_t(rb - ra), size_t(wn));
    cp.kind = cudaMemcpyHostToDevice;
    TG_CUDA(cudaMemcpy3DAsync(&cp, hp.xs));
    shipped += uint64_t(ub - ua) * uint64_t(rb - ra) * wn * sizeof(float);
  };
  bool k1_last = false;  // the stream's most recent kernel is a K1
  for (int ph = 0; ph < n_phases; ++ph) {
    // slices of this phase (its ranges are contiguous below / above the centre)
    const bool last = ph == n_phases - 1;
    const uint64_t ch_ph = ph >= kLateFrom ? chunk_late : chunk;
    const int nch_ph = ph >= kLateFrom ? n_chunks_late : n_chunks;
    for (int c = 0; c < nch_ph; ++c) {
      const uint64_t w0 = uint64_t(c) * ch_ph, wn = std::min(ch_ph, np - w0);
      for (uint64_t gi = w0 / G; gi * G < w0 + wn; ++gi) {
        const uint64_t a = std::max<uint64_t>(gi * G, w0);
        const uint64_t b = std::min<uint64_t>((gi + 1) * G, w0 + wn);
        int64_t ra = int64_t(v0 + n_rows), rb = int64_t(v0);
        for (uint64_t i = a; i < b; ++i)
          for (const Range& r : phases[ph]) {
            if (r.n == 0) continue;
            const Foot f = footprint(i, r.z, r.z + r.n - 1);
            ra = std::min(ra, f.va);
            rb = std::max(rb, f.vb);
          }
        if (rb <= ra) continue;
        int64_t& lo = g_lo[gi];  // rows resident for every view of the group
        int64_t& hi = g_hi[gi];
        if (hi <= lo) {
          upload(a, b - a, g_ua[gi], g_ub[gi], ra, rb);
          lo = ra;
          hi = rb;
        } else {
          if (ra < lo) upload(a, b - a, g_ua[gi], g_ub[gi], ra, lo);
          if (rb > hi) upload(a, b - a, g_ua[gi], g_ub[gi], hi, rb);
          lo = std::min(lo, ra);
          hi = std::max(hi, rb);
        }
      }
      TG_CUDA(cudaEventRecord(hp.ev[ev], hp.xs));
      TG_CUDA(cudaStreamWaitEvent(hp.cs, hp.ev[ev++], 0));
      const bool filtered = !fresh.empty();
      bool first_seg = true;
      for (const Fresh& sg : fresh) {  // FDK: cosine x Parker + Ram-Lak on the new rows
        filt::RowLayout lay;
        lay.rows_per_view = uint64_t(sg.rb - sg.ra);
        lay.view_pitch = n_rows * nu;
        float* seg = d_band + (sg.w0 * n_rows + uint64_t(sg.ra) - v0) * nu;
        // the chunk's first pre-weights pass overlaps the previous K1's tail
        // (that K1 reads other views' rows; the pass waits for it before exiting)
        prefilter_impl(p, seg, seg, use_parker, uint64_t(sg.ra), lay.rows_per_view, sg.w0, sg.wn,
                       hp.cs, lay, kPdl && first_seg && k1_last);
        first_seg = false;
      }
      // PDL only for a K1 whose stream predecessor is another K1: with FDK the
      // chunk's first K1 follows the K3 that filtered its rows
      bool after_k3 = fdk && filtered;
      fresh.clear();
      if (last && c == nch_ph - 1) {
        for (const Range& r : phases[ph])
          for (uint64_t q = 0; q < r.n; q += 32) {
            const Range part{r.z + q, std::min<uint64_t>(32, r.n - q)};
            backproject_impl(p, z0 + part.z, part.n, v0, n_rows, d_band, d_slab + part.z * plane,
                             scale, c > 0, hp.cs, w0, wn, kPdl && !after_k3);
            after_k3 = false;
            k1_last = true;
            TG_CUDA(cudaEventRecord(hp.ev[ev], hp.cs));
            TG_CUDA(cudaStreamWaitEvent(ds, hp.ev[ev++], 0));
            download(part);
          }
      } else {
        for (const Range& r : phases[ph]) {
          backproject_impl(p, z0 + r.z, r.n, v0, n_rows, d_band, d_slab + r.z * plane, scale,
                           c > 0, hp.cs, w0, wn, kPdl && !after_k3);
          after_k3 = false;
          k1_last = true;
        }
      }
    }
    if (!last) {
      TG_CUDA(cudaEventRecord(hp.ev[ev], hp.cs));
      TG_CUDA(cudaStreamWaitEvent(ds, hp.ev[ev++], 0));
      for (const Range& r : phases[ph]) download(r);
    }
  }
  p.last_h2d_bytes = shipped;
  TG_CUDA(cudaStreamSynchronize(ds));
  TG_CUDA(cudaStreamSynchronize(hp.cs));
}

}  // namespace

extern "C" {

tg_status tg_cone_plan_create(const tg_cone_geometry* g, int device, tg_cone_plan** out) {
  return guarded([&] {
    *out = nullptr;
    validate_volume(g->volume);
    check(g->volume.dims == 3, "cone beam geometry expects a 3D volume");
    check(g->sid > 0.0 && g->sdd > g->sid, "cone beam requires 0 < SID < SDD");
    check(g->n_projections >= 1, "need at least one projection");
    check(g->detector.n_u >= 1 && g->detector.n_v >= 1,
          "detector needs at least one pixel per axis");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device visible: the B200 path has no CPU fallback");
    }
    check(device >= 0 && device < ndev, "device index out of range");
    auto p = std::make_unique<tg_cone_plan>();
    p->device = device;
    p->id = next_plan_id();
    p->vol = g->volume;
    p->det = g->detector;
    p->n_proj = g->n_projections;
    p->range = g->angular_range;
    p->sid = g->sid;
    p->sdd = g->sdd;
    const uint64_t n = g->n_projections;
    p->mats.assign(g->matrices, g->matrices + 12 * n);
    p->sources.assign(g->sources, g->sources + 3 * n);
    p->invs.assign(g->inv_blocks, g->inv_blocks + 9 * n);
    p->angles.assign(g->angles, g->angles + n);
    std::vector<double> geo(12 * n);
    for (uint64_t i = 0; i < n; ++i) {
      const double* m = g->matrices + 12 * i;
      if (m[2] != 0.0 || m[10] != 0.0) p->circular = false;
      for (int k = 0; k < 3; ++k) geo[12 * i + k] = g->sources[3 * i + k];
      for (int k = 0; k < 9; ++k) geo[12 * i + 3 + k] = g->inv_blocks[9 * i + k];
    }
    DeviceGuard dg(device);
    TG_CUDA(cudaMalloc(&p->d_mats, 12 * n * sizeof(double)));
    TG_CUDA(cudaMemcpy(p->d_mats, g->matrices, 12 * n * sizeof(double), cudaMemcpyHostToDevice));
    TG_CUDA(cudaMalloc(&p->d_geo, geo.size() * sizeof(double)));
    TG_CUDA(cudaMemcpy(p->d_geo, geo.data(), geo.size() * sizeof(double), cudaMemcpyHostToDevice));
    p->k1_k = default_k1_k();
    // K2 band height: 8 detector rows (TU = 32) while a quad-volume slice is
    // small; 4 rows (TU = 64) once a slice passes 8 MB, so the sheet of volume
    // a band's rays cross stays L2-resident (c4 4.3 MB: 449 vs 459 ms;
    // c5 16.9 MB: 4.52 vs 4.80 s)
    {
      const double slice_mb = double(g->volume.shape[0] + 4) * double(g->volume.shape[1] + 4) * 16.0 / 1e6;
      p->k2_tu = slice_mb >= 8.0 ? 64 : 32;
    }
    size_box(*p);
    *out = p.release();
  });
}

tg_status tg_cone_plan_destroy(tg_cone_plan* p) {
  return guarded([&] {
    if (!p) return;
    g_bank.forget(p->id);
    DeviceGuard dg(p->device);
    cudaFree(p->d_mats);
    cudaFree(p->d_geo);
    cudaFree(p->d_cos);
    cudaFree(p->d_parker);
    cudaFree(p->d_vpad);
    cudaFree(p->d_vt);
    cudaFree(p->d_vx);
    cudaFree(p->d_k2_stats);
    cudaFree(p->d_pitched);
    cudaFree(p->d_stage_in);
    cudaFree(p->d_stage_out);
    if (p->ramlak) filt::destroy(p->ramlak);
    delete p;
  });
}

tg_status tg_cone_plan_shape(const tg_cone_plan* p, tg_volume_spec* vol, tg_detector2d* det,
                             uint64_t* n_proj) {
  return guarded([&] {
    check(p != nullptr, "null plan");
    if (vol) *vol = p->vol;
    if (det) *det = p->det;
    if (n_proj) *n_proj = p->n_proj;
  });
}

tg_status tg_cone_forward(tg_cone_plan* p, const float* d_vol, float* d_sino, void* stream) {
  return guarded([&] { forward_impl(*p, 0, p->n_proj, d_vol, d_sino, as_stream(stream)); });
}

tg_status tg_cone_forward_views(tg_cone_plan* p, uint64_t view0, uint64_t n_views,
                                const float* d_vol, float* d_part, void* stream) {
  return guarded([&] { forward_impl(*p, view0, n_views, d_vol, d_part, as_stream(stream)); });
}

tg_status tg_cone_ray_samples(tg_cone_plan* p, uint64_t view0, uint64_t n_views,
                              uint64_t* d_counts, void* stream) {
  return guarded([&] {
    check(p != nullptr, "null plan");
    check(view0 + n_views <= p->n_proj && n_views >= 1, "view range lies outside the geometry");
    DeviceGuard dg(p->device);
    FpArgs a = fp_args(*p);
    const cudaStream_t st = as_stream(stream);
    for (uint64_t c0 = 0; c0 < n_views; c0 += 65535) {
      const uint64_t cn = std::min<uint64_t>(65535, n_views - c0);
      a.view0 = int(view0 + c0);
      dim3 grid((a.nu + 31) / 32, unsigned(cn), (a.nv + 7) / 8);
      cone_ray_samples_kernel<<<grid, 256, 0, st>>>(
          a, reinterpret_cast<unsigned long long*>(d_counts) + c0 * p->det.n_u * p->det.n_v);
      TG_LAUNCHED(1);
    }
  });
}

tg_status tg_cone_plan_set_knob(tg_cone_plan* p, const char* name, int64_t value) {
  return guarded([&] {
    check(p != nullptr && name != nullptr, "null plan or knob name");
    const std::string k(name);
    std::lock_guard<std::recursive_mutex> lk(p->mu);
    if (k == "k2_tu") {
      check(value == 32 || value == 64, "k2_tu must be 32 or 64");
      p->k2_tu = int(value);
    } else if (k == "k2_impl") {
      // 1: slab-staged K2 (shared-memory boxes); 0: quad-volume L1 gathers;
      // -1: autotune at the next forward projection (default)
      check(value == 0 || value == 1 || value == -1, "k2_impl must be -1, 0 or 1");
      p->k2_impl = int(value);
    } else if (k == "k2_dual") {
      // 0: gather every ray from the x-fastest quad volume (bitwise identical)
      p->k2_dual_allowed = value != 0;
    } else {
      check(false, "unknown knob");
    }
  });
}

tg_status tg_cone_backproject(tg_cone_plan* p, const float* d_sino, float* d_vol, float scale,
                              int accumulate, void* stream) {
  return guarded([&] {
    backproject_impl(*p, 0, p->vol.shape[2], 0, p->det.n_v, d_sino, d_vol, scale, accumulate,
                     as_stream(stream));
  });
}

tg_status tg_cone_slab_rows(tg_cone_plan* p, uint64_t z0, uint64_t nz, uint64_t* v0,
                            uint64_t* n_rows) {
  return guarded([&] {
    tg_cone_geometry g{p->vol, p->det, p->n_proj, p->range, p->sid, p->sdd, p->mats.data(),
                       p->sources.data(), p->invs.data(), p->angles.data()};
    slab_rows(g, z0, nz, v0, n_rows);
  });
}

tg_status tg_cone_slab_rows_geom(const tg_cone_geometry* g, uint64_t z0, uint64_t nz, uint64_t* v0,
                                 uint64_t* n_rows) {
  return guarded([&] { slab_rows(*g, z0, nz, v0, n_rows); });
}

tg_status tg_cone_backproject_slab(tg_cone_plan* p, uint64_t z0, uint64_t nz, uint64_t v0,
                                   uint64_t n_rows, const float* d_band, float* d_slab, float scale,
                                   int accumulate, void* stream) {
  return guarded([&] {
    backproject_impl(*p, z0, nz, v0, n_rows, d_band, d_slab, scale, accumulate, as_stream(stream));
  });
}

tg_status tg_cone_fdk_prefilter(tg_cone_plan* p, const float* d_in, float* d_out, int use_parker,
                                uint64_t v0, uint64_t n_rows, void* stream) {
  return guarded([&] {
    prefilter_impl(*p, d_in, d_out, use_parker != 0, v0, n_rows, 0, p->n_proj, as_stream(stream));
  });
}

double tg_cone_fdk_scale(const tg_cone_plan* p, int use_parker) { return fdk_scale(*p, use_parker != 0); }

tg_status tg_cone_fdk(tg_cone_plan* p, const float* d_sino, float* d_vol, float* d_work,
                      int use_parker, void* stream) {
  return guarded([&] {
    cudaStream_t st = as_stream(stream);
    prefilter_impl(*p, d_sino, d_work, use_parker != 0, 0, p->det.n_v, 0, p->n_proj, st);
    backproject_impl(*p, 0, p->vol.shape[2], 0, p->det.n_v, d_work, d_vol,
                     float(fdk_scale(*p, use_parker != 0)), 0, st);
  });
}

tg_status tg_cone_forward_host(tg_cone_plan* p, const float* h_vol, float* h_sino) {
  return guarded([&] {
    DeviceGuard dg(p->device);
    std::lock_guard<std::recursive_mutex> call_lock(p->mu);  // the plan's pipeline streams
    const uint64_t nvox = p->vol.shape[0] * p->vol.shape[1] * p->vol.shape[2];
    const uint64_t per_view = p->det.n_u * p->det.n_v;
    float *d_vol = nullptr, *d_sino = nullptr;
    TG_CUDA(cudaMalloc(&d_vol, nvox * sizeof(float)));
    TG_CUDA(cudaMalloc(&d_sino, p->n_proj * per_view * sizeof(float)));
    HostPipe& hp = plan_pipe(*p, 1);
    TG_CUDA(cudaMemcpyAsync(d_vol, h_vol, nvox * sizeof(float), cudaMemcpyHostToDevice, hp.cs));
    // views in chunks so the D2H of chunk c overlaps the projection of c+1
    const uint64_t chunk = std::max<uint64_t>(1, (p->n_proj + 7) / 8);
    for (uint64_t v0 = 0; v0 < p->n_proj; v0 += chunk) {
      const uint64_t vn = std::min(chunk, p->n_proj - v0);
      forward_impl(*p, v0, vn, d_vol, d_sino + v0 * per_view, hp.cs, v0 == 0);
      TG_CUDA(cudaEventRecord(hp.ev[0], hp.cs));
      TG_CUDA(cudaStreamWaitEvent(hp.xs, hp.ev[0], 0));
      TG_CUDA(cudaMemcpyAsync(h_sino + v0 * per_view, d_sino + v0 * per_view,
                              vn * per_view * sizeof(float), cudaMemcpyDeviceToHost, hp.xs));
    }
    TG_CUDA(cudaStreamSynchronize(hp.xs));
    TG_CUDA(cudaStreamSynchronize(hp.cs));
    TG_CUDA(cudaFree(d_vol));
    TG_CUDA(cudaFree(d_sino));
  });
}

tg_status tg_cone_backproject_host(tg_cone_plan* p, const float* h_sino, float* h_vol) {
  return guarded([&] {
    host_backproject(*p, 0, p->vol.shape[2], 0, p->det.n_v, h_sino, h_vol, 0, false);
  });
}

tg_status tg_cone_backproject_slab_host(tg_cone_plan* p, uint64_t z0, uint64_t nz, uint64_t v0,
                                        uint64_t n_rows, const float* h_band, float* h_slab,
                                        int fdk, int use_parker) {
  return guarded([&] {
    host_backproject(*p, z0, nz, v0, n_rows, h_band, h_slab, fdk, use_parker != 0);
  });
}

uint64_t tg_cone_last_h2d_bytes(const tg_cone_plan* p) { return p ? p->last_h2d_bytes : 0; }

tg_status tg_cone_fdk_host(tg_cone_plan* p, const float* h_sino, float* h_vol, int use_parker) {
  return guarded([&] {
    // FDK of the whole volume needs only the detector rows the volume
    // projects onto (K3 filters along u within a row): the rest of each view
    // is neither uploaded nor filtered
    const tg_cone_geometry g{p->vol, p->det, p->n_proj, p->range, p->sid, p->sdd, p->mats.data(),
                             p->sources.data(), p->invs.data(), p->angles.data()};
    uint64_t v0 = 0, n_rows = p->det.n_v;
    slab_rows(g, 0, p->vol.shape[2], &v0, &n_rows);
    host_backproject(*p, 0, p->vol.shape[2], v0, n_rows, h_sino + v0 * p->det.n_u, h_vol, 1,
                     use_parker != 0, p->det.n_v * p->det.n_u);
  });
}

}  // extern "C"
