// planar.cu — parallel- and fan-beam 2D operators (K4-K7).
//   K7 parallel forward  projector.hpp:171-184   K6 parallel back  projector.hpp:186-208
//   K5 fan forward       projector.hpp:212-230   K4 fan back (1/U^2) projector.hpp:232-260
//
// Forward (K5/K7): one ray per (view, bin), 1-8 threads per ray.  Ray setup,
// clip and sample count run in IEEE FP64 without contraction (bit-exact hit
// test and n, shared with the tg_planar_ray_samples diagnostic); the march
// runs in fp32 from FP64 anchors every 64 samples and gathers one 16-byte
// "quad" (the four bilinear taps) per trilinear cell from a zero-bordered
// quad image, x-fastest or y-fastest so that the lanes of a warp (adjacent
// bins) read neighbouring quads.
//
// Back-projection (K4/K6): CTA = 32 x 16 pixel tile, 2 pixels per thread;
// per (tile, view) one thread builds the view's map in FP64 at the tile
// origin (bin = N / D with N, D affine in the pixel's tile-local index; D = 1
// for parallel beam), shifted by an integer bin base so that the fp32
// per-pixel evaluation works with small numbers.  The views are split over
// the CTAs of a thread-block cluster (1 x 1 x G); partial sums are reduced
// through distributed shared memory in a fixed order (deterministic, one
// writer per pixel, no atomics, no scratch image).
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include <cooperative_groups.h>

#include "device_common.cuh"

namespace cg = cooperative_groups;

namespace tgb {
namespace planar {

#define DADD __dadd_rn
#define DMUL __dmul_rn
#define DDIV __ddiv_rn

struct FpArgs {
  int nb, n_views;
  int nx, ny;
  double ox, oy, sx, sy, step;
  double det_origin, det_spacing;
  double sid, sdd;
  int fan;
  const double* __restrict__ rays;  // n x 2
  // zero-bordered quads (+2 each side): element (px, py) holds
  // (V[y][x], V[y][x+1], V[y+1][x], V[y+1][x+1]) at x = px - 2, y = py - 2
  const float4* __restrict__ q;   // x-fastest: px + py * nxp
  const float4* __restrict__ qT;  // y-fastest: py + px * nyp
  int nxp, nyp;
  int segs;  // threads per ray (1, 2, 4, 8)
  float* out;
};

__device__ __forceinline__ bool clip_ray2(const FpArgs& a, const double o[2], const double d[2],
                                          double& t0, double& t1) {
  // projector.hpp:83-101
  const double org[2] = {a.ox, a.oy}, sp[2] = {a.sx, a.sy};
  const int n[2] = {a.nx, a.ny};
  t0 = -1e300;
  t1 = 1e300;
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
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

// projector.hpp:171-184 (parallel: origin s * axis, direction r) and
// 212-230 (fan: source -SID r, direction normalise(pixel - source)) for bin j
// of view i, then the clip; FP64 without contraction.
__device__ __forceinline__ bool planar_ray(const FpArgs& a, int i, int j, double o[2], double d[2],
                                           double& t0, double& t1) {
  const double rx = a.rays[2 * i], ry = a.rays[2 * i + 1];
  const double axx = -ry, axy = rx;
  if (!a.fan) {
    const double s = DADD(a.det_origin, DMUL(double(j), a.det_spacing));
    o[0] = DMUL(s, axx);
    o[1] = DMUL(s, axy);
    d[0] = rx;
    d[1] = ry;
  } else {
    const double ns = -a.sid;
    const double sx = DMUL(ns, rx), sy = DMUL(ns, ry);
    const double u = DADD(a.det_origin, DMUL(double(j), a.det_spacing));
    const double px = DADD(DADD(sx, DMUL(a.sdd, rx)), DMUL(u, axx));
    const double py = DADD(DADD(sy, DMUL(a.sdd, ry)), DMUL(u, axy));
    const double dx = DADD(px, -sx), dy = DADD(py, -sy);
    const double s = DDIV(1.0, __dsqrt_rn(DADD(DMUL(dx, dx), DMUL(dy, dy))));
    o[0] = sx;
    o[1] = sy;
    d[0] = DMUL(s, dx);
    d[1] = DMUL(s, dy);
  }
  return clip_ray2(a, o, d, t0, t1);
}

// projector.hpp:117: n = ceil((t1 - t0) / step)
__device__ __forceinline__ long long ray_sample_count(double span, double step) {
  return (long long)ceil(DDIV(span, step));
}

__device__ __forceinline__ float lerpf(float a, float b, float w) { return fmaf(w, b - a, a); }

// MUFU reciprocal (<= 1 ulp)
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// K5 / K7.  Lane layout: a warp holds 32 adjacent rays (consecutive bins of
// a view, so its lanes gather neighbouring quads: L1 locality) at one segment;
// the 8 warps of a CTA hold 8 / S ray groups x S segments, segment s
// marching the 64-sample chunks s, s + S, ... of its ray.  The segments'
// partial sums are combined in shared memory by a fixed pairwise tree
// ((s0 + s1) + (s2 + s3) ...), so the result does not depend on scheduling.
// 7 CTAs (56 warps) per SM at 32 registers: the march is L2-latency bound
// (64 registers / 4 CTAs -> 40 / 6: c2 371 -> 320 us, c1 104 -> 99 us,
// profiles/r2_planar_fp_variants.txt; with only the anchor state live across
// chunks 6 -> 7 CTAs: c2 312.7 -> 291.1 us, c1 97.1 -> 95.6 us; 8 is the same
// 32-register build)
#ifndef TG_PLANAR_FP_MINB
#define TG_PLANAR_FP_MINB 7
#endif
template <bool REUSE>
__global__ void __launch_bounds__(256, TG_PLANAR_FP_MINB) planar_fp_kernel(const FpArgs a) {
  __shared__ double part[8][32];
  const int S = a.segs;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = w / S, seg = w % S;
  const long long ray = ((long long)blockIdx.x * (8 / S) + g) * 32 + lane;
  const long long total_rays = (long long)a.n_views * a.nb;
  double total = 0.0, dt = 0.0;
  bool hit = false;
  if (ray < total_rays) {
    const int i = int(ray / a.nb), j = int(ray % a.nb);
    double o[2], d[2], t0, t1;
    hit = planar_ray(a, i, j, o, d, t0, t1);
    if (hit) {
      const double span = DADD(t1, -t0);
      const int n = int(ray_sample_count(span, a.step));  // < 2^31 samples per ray
      dt = DDIV(span, double(n));
      // sample k at t0 + (k + 1/2) dt (projector.hpp:109-128), in padded
      // index coordinates
      const double th = t0 + 0.5 * dt;
      const double p0x = (o[0] + th * d[0] - a.ox) / a.sx + 2.0;
      const double p0y = (o[1] + th * d[1] - a.oy) / a.sy + 2.0;
      const double ddx = dt * d[0] / a.sx, ddy = dt * d[1] / a.sy;
      // rays running mostly along x: adjacent bins are displaced along y,
      // so gather from the y-fastest quads
      const bool xdom = fabs(d[0]) > fabs(d[1]);
      constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23: t = M + floor(p) under round-down
      constexpr int MAGIC_BITS = 0x4B400000;
      for (int k0 = 64 * seg; k0 < n; k0 += 64 * S) {
        // layout and fp32 steps re-derived per chunk: only the FP64 anchor
        // state and the layout bit live across chunks (fewer spills at the
        // register cap; as in K2, profiles/r2_k2_traffic.txt)
        const float4* base = xdom ? a.qT : a.q;
        const int stx = xdom ? a.nyp : 1, sty = xdom ? 1 : a.nxp;
        const float fdx = float(ddx), fdy = float(ddy);
        const double ax = p0x + double(k0) * ddx, ay = p0y + double(k0) * ddy;
        const double cx = floor(ax), cy = floor(ay);
        const float bx = float(ax - cx), by = float(ay - cy);
        const float4* cell = base + (long long)cy * sty + (long long)cx * stx;
        const int m = min(64, n - k0);
        float sum = 0.0f;
        int prev = 0x7fffffff;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int k = 0; k < m; ++k) {
          const float px = fmaf(float(k), fdx, bx), py = fmaf(float(k), fdy, by);
          const float tx = __fadd_rd(px, MAGIC), ty = __fadd_rd(py, MAGIC);
          const float wx = px - (tx - MAGIC), wy = py - (ty - MAGIC);
          const int off = (__float_as_int(tx) - MAGIC_BITS) * stx + (__float_as_int(ty) - MAGIC_BITS) * sty;
          if (!REUSE) {
            q = __ldg(cell + off);  // independent loads: the unrolled loop batches them
          } else if (off != prev) {
            q = __ldg(cell + off);
            prev = off;
          }
          sum += lerpf(lerpf(q.x, q.y, wx), lerpf(q.z, q.w, wx), wy);
        }
        total += double(sum);
      }
    }
  }
  if (S > 1) {
    part[w][lane] = total;
    __syncthreads();
    if (seg == 0) {
      // pairwise tree over the S segments of this ray group
      for (int step = 1; step < S; step <<= 1)
        for (int s0 = 0; s0 + step < S; s0 += 2 * step)
          part[g * S + s0][lane] += part[g * S + s0 + step][lane];
      total = part[g * S][lane];
    }
  }
  if (seg == 0 && ray < total_rays) a.out[ray] = hit ? float(total * dt) : 0.0f;
}

// Diagnostic: per-ray sample count of K5/K7 (0 = missed ray), same setup.
__global__ void __launch_bounds__(256) planar_ray_samples_kernel(const FpArgs a,
                                                                 unsigned long long* out) {
  const long long ray = (long long)blockIdx.x * 256 + threadIdx.x;
  if (ray >= (long long)a.n_views * a.nb) return;
  double o[2], d[2], t0, t1;
  unsigned long long n = 0;
  if (planar_ray(a, int(ray / a.nb), int(ray % a.nb), o, d, t0, t1))
    n = (unsigned long long)ray_sample_count(DADD(t1, -t0), a.step);
  out[ray] = n;
}

// builds both quad layouts of the zero-bordered image in one pass
__global__ void pad_quads_kernel(const float* __restrict__ img, float4* __restrict__ q,
                                 float4* __restrict__ qT, int nx, int ny) {
  const int nxp = nx + 4, nyp = ny + 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)nxp * nyp;
       i += (long long)gridDim.x * blockDim.x) {
    const int px = int(i % nxp), py = int(i / nxp);
    const int x = px - 2, y = py - 2;
    auto at = [&](int xx, int yy) {
      return (xx >= 0 && xx < nx && yy >= 0 && yy < ny) ? __ldg(img + (long long)yy * nx + xx) : 0.0f;
    };
    const float4 v = make_float4(at(x, y), at(x + 1, y), at(x, y + 1), at(x + 1, y + 1));
    q[i] = v;
    qT[(long long)px * nyp + py] = v;
  }
}

// ---------------------------------------------------------------------------
// K4 / K6
//
// CTA = 32 x 32 pixel tile, 256 threads, 4 pixels per thread (rows ty + 8q)
// processed as two FP32x2 pairs.  The views are split over the CTAs of a
// thread-block cluster (1 x 1 x G) and reduced through distributed shared
// memory in a fixed order (deterministic, one writer per pixel, no atomics).
// Per chunk of views: (1) one thread per view builds the view's FP64 map at
// the tile origin and the tile's footprint on the detector row (the bin
// coordinate is affine (parallel) or projective with positive depth (fan)
// over the tile, so its extremes sit on the 4 corners); (2) the CTA stages
// each view's footprint bins [b0, b0 + W) into shared memory, zero outside
// the detector (= the reference's zero-padded interp_row, projector.hpp:32-41);
// (3) every pixel interpolates from shared memory with no bounds checks.
// Views whose footprint is wider than the staging row, or that put part of
// the tile behind the source (fan), take a checked path from global memory.

constexpr int kTX = 32, kTY = 32;  // pixel tile
constexpr int kChunk = 64;         // views staged in shared memory at once
constexpr int kRow = 96;           // staged bins per view
constexpr int kMaxCluster = 8;

struct BpArgs {
  int nx, ny, nb, n_views;
  int vpg;  // views per cluster rank
  double ox, oy, sx, sy;
  double det_origin, det_spacing, inv_ds;
  double sid, sdd;
  const double* __restrict__ rays;  // n x 2
  float scale;
  int accumulate;
  const float* __restrict__ sino;
  float* img;
};

// tile-local map of one view: bin - b0 = (n0 + lx na + ly nb) / (d0 + lx da + ly db)
struct ViewMap {
  float n0, na, nb, d0, da, db;
  int b0;    // first staged bin
  int fast;  // footprint staged (and, fan: whole tile in front of the source)
};

// FP64 map of view i for the tile at pixel (x0, y0), mirroring
// projector.hpp:186-208 (parallel) / 232-260 (fan), shifted by the bin b0.
template <bool FAN>
__device__ ViewMap make_map(const BpArgs& a, int i, int x0, int y0) {
  const double rx = a.rays[2 * i], ry = a.rays[2 * i + 1];
  const double axx = -ry, axy = rx;  // detector axis: ray rotated +90 deg
  const double X0 = a.ox + double(x0) * a.sx, Y0 = a.oy + double(y0) * a.sy;
  const int ex = min(kTX, a.nx - x0) - 1, ey = min(kTY, a.ny - y0) - 1;
  ViewMap m;
  if (!FAN) {
    // bin(x, y) = ((x, y) . axis - origin) / spacing: affine
    const double t00 = (X0 * axx + Y0 * axy - a.det_origin) * a.inv_ds;
    const double tx = a.sx * axx * a.inv_ds, ty = a.sy * axy * a.inv_ds;
    const double lo = t00 + fmin(0.0, ex * tx) + fmin(0.0, ey * ty);
    const double hi = t00 + fmax(0.0, ex * tx) + fmax(0.0, ey * ty);
    const int b0 = int(floor(fmax(lo, -1e8))) - 1;
    m.b0 = b0;
    m.fast = (floor(fmin(hi, 1e8)) + 2.0 - double(b0) < double(kRow)) ? 1 : 0;
    m.n0 = float(t00 - double(b0));
    m.na = float(tx);
    m.nb = float(ty);
    m.d0 = 1.0f;
    m.da = 0.0f;
    m.db = 0.0f;
  } else {
    // depth D = q . r and bin numerator N = SDD q . axis, q = (x, y) + SID r:
    // bin = (N / D - origin) / spacing, projective in (x, y)
    const double qx = X0 + a.sid * rx, qy = Y0 + a.sid * ry;
    const double D0 = qx * rx + qy * ry;
    const double M0 = qx * axx + qy * axy;
    double lo = 1e300, hi = -1e300, dmin = 1e300;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double dx = (c & 1) ? ex * a.sx : 0.0, dy = (c & 2) ? ey * a.sy : 0.0;
      const double D = D0 + dx * rx + dy * ry;
      const double M = M0 + dx * axx + dy * axy;
      dmin = fmin(dmin, D);
      const double t = D > 0.0 ? (a.sdd * M / D - a.det_origin) * a.inv_ds : 0.0;
      lo = fmin(lo, t);
      hi = fmax(hi, t);
    }
    const int b0 = int(floor(fmin(fmax(lo, -1e8), 1e8))) - 1;
    m.b0 = b0;
    m.fast = (dmin > 0.0 && floor(fmin(hi, 1e8)) + 2.0 - double(b0) < double(kRow)) ? 1 : 0;
    const double c = a.det_origin + double(b0) * a.det_spacing;
    // bin - b0 = (SDD num - c depth) / (spacing depth)
    m.n0 = float((a.sdd * M0 - c * D0) * a.inv_ds);
    m.na = float((a.sdd * a.sx * axx - c * a.sx * rx) * a.inv_ds);
    m.nb = float((a.sdd * a.sy * axy - c * a.sy * ry) * a.inv_ds);
    m.d0 = float(D0);
    m.da = float(a.sx * rx);
    m.db = float(a.sy * ry);
  }
  return m;
}

// zero-padded linear interpolation along a sinogram row (projector.hpp:32-41)
__device__ __forceinline__ float interp_row(const float* __restrict__ row, int nb, int base, float t) {
  const float f = floorf(t);
  const float w = t - f;
  const int i0 = base + int(f);
  const float a0 = (unsigned)i0 < (unsigned)nb ? __ldg(row + i0) : 0.0f;
  const float a1 = (unsigned)(i0 + 1) < (unsigned)nb ? __ldg(row + i0 + 1) : 0.0f;
  return lerpf(a0, a1, w);
}

// 5 CTAs per SM (48 registers; the spills sit in the FP64 map builder and the
// checked path): c2 93.0 -> 90.3 us against the default 64 registers
template <bool FAN>
__global__ void __launch_bounds__(256, 5) planar_bp_kernel(const BpArgs a) {
  __shared__ ViewMap maps[kChunk];
  __shared__ float rows[kChunk][kRow];
  __shared__ float part[kTX * kTY];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = int(cluster.num_blocks());
  const int rank = int(cluster.block_rank());
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  // pixels past the image edge (partial tiles) evaluate a clamped in-tile
  // position — their result is discarded, but their taps stay in the footprint
  const int ex = min(kTX, a.nx - x0) - 1, ey = min(kTY, a.ny - y0) - 1;
  const float lx = float(min(tx, ex));
  // pixel pairs (ty, ty + 8) and (ty + 16, ty + 24)
  const float2 lyA = make_float2(float(min(ty, ey)), float(min(ty + 8, ey)));
  const float2 lyB = make_float2(float(min(ty + 16, ey)), float(min(ty + 24, ey)));
  const int v_begin = min(a.n_views, rank * a.vpg);
  const int v_end = min(a.n_views, v_begin + a.vpg);
  constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23: t = M + floor(p) under round-down
  const float2 M2 = make_float2(MAGIC, MAGIC), nM2 = make_float2(-MAGIC, -MAGIC);
  const float sid = float(a.sid);
  float2 accA = make_float2(0.f, 0.f), accB = accA;
  const uint32_t rows_base = smem_u32(&rows[0][0]);
  for (int c0 = v_begin; c0 < v_end; c0 += kChunk) {
    const int cn = min(kChunk, v_end - c0);
    __syncthreads();
    if (threadIdx.x < cn) maps[threadIdx.x] = make_map<FAN>(a, c0 + threadIdx.x, x0, y0);
    __syncthreads();
    // stage every view's footprint (coalesced per view; zero off the detector)
    for (int e = threadIdx.x; e < cn * kRow; e += 256) {
      const int v = e / kRow, i = e - v * kRow;
      const int b = maps[v].b0 + i;
      rows[v][i] = (maps[v].fast && (unsigned)b < (unsigned)a.nb)
                       ? __ldg(a.sino + (long long)(c0 + v) * a.nb + b)
                       : 0.0f;
    }
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < cn; ++k) {
      const ViewMap m = maps[k];
      const float n0 = fmaf(lx, m.na, m.n0);
      const float2 n02 = make_float2(n0, n0), nb2 = make_float2(m.nb, m.nb);
      if (m.fast) {
        const uint32_t rb = rows_base + uint32_t(k * kRow) * 4u - uint32_t(0x4B400000) * 4u;
        if (!FAN) {
          auto upd = [&](float2 ly, float2& acc) {
            const float2 t = __ffma2_rn(ly, nb2, n02);
            const float2 tt = __fadd2_rd(t, M2);
            const float2 fl = __fadd2_rn(tt, nM2);
            const float2 w = __fadd2_rn(t, make_float2(-fl.x, -fl.y));
            const uint32_t ia = rb + __float_as_uint(tt.x) * 4u, ib = rb + __float_as_uint(tt.y) * 4u;
            float a0, a1, b0, b1;
            asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];" : "=f"(a0), "=f"(a1) : "r"(ia));
            asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];" : "=f"(b0), "=f"(b1) : "r"(ib));
            const float2 lo = make_float2(a0, b0), hi = make_float2(a1, b1);
            const float2 v = __ffma2_rn(w, __fadd2_rn(hi, make_float2(-lo.x, -lo.y)), lo);
            acc = __fadd2_rn(acc, v);
          };
          upd(lyA, accA);
          upd(lyB, accB);
        } else {
          const float d0 = fmaf(lx, m.da, m.d0);
          const float2 d02 = make_float2(d0, d0), db2 = make_float2(m.db, m.db);
          auto upd = [&](float2 ly, float2& acc) {
            const float2 dd = __ffma2_rn(ly, db2, d02);
            float2 r;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(dd.x));
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(dd.y));
            const float2 t = __fmul2_rn(__ffma2_rn(ly, nb2, n02), r);
            const float2 tt = __fadd2_rd(t, M2);
            const float2 fl = __fadd2_rn(tt, nM2);
            const float2 w = __fadd2_rn(t, make_float2(-fl.x, -fl.y));
            const uint32_t ia = rb + __float_as_uint(tt.x) * 4u, ib = rb + __float_as_uint(tt.y) * 4u;
            float a0, a1, b0, b1;
            asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];" : "=f"(a0), "=f"(a1) : "r"(ia));
            asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];" : "=f"(b0), "=f"(b1) : "r"(ib));
            const float2 lo = make_float2(a0, b0), hi = make_float2(a1, b1);
            const float2 v = __ffma2_rn(w, __fadd2_rn(hi, make_float2(-lo.x, -lo.y)), lo);
            // 1/U^2 = (SID / depth)^2 (projector.hpp:250-256)
            const float2 s = __fmul2_rn(make_float2(sid, sid), r);
            acc = __ffma2_rn(__fmul2_rn(v, s), s, acc);
          };
          upd(lyA, accA);
          upd(lyB, accB);
        }
      } else {
        // checked path: global row, per-pixel behind-source test
        const float* row = a.sino + (long long)(c0 + k) * a.nb;
        const float ly[4] = {lyA.x, lyA.y, lyB.x, lyB.y};
        float add[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float nn = fmaf(ly[q], m.nb, n0);
          if (!FAN) {
            add[q] = interp_row(row, a.nb, m.b0, nn);
          } else {
            const float dd = fmaf(ly[q], m.db, fmaf(lx, m.da, m.d0));
            add[q] = 0.0f;
            if (dd > 0.0f) {  // depth <= 0: behind the source (projector.hpp:247)
              const float r = rcp_approx(dd);
              const float sv = sid * r;
              add[q] = interp_row(row, a.nb, m.b0, nn * r) * sv * sv;
            }
          }
        }
        accA.x += add[0];
        accA.y += add[1];
        accB.x += add[2];
        accB.y += add[3];
      }
    }
  }
  // cluster reduction: rank r owns pixels p = r, r + G, ... of the tile and
  // sums the G partials in rank order
  part[ty * kTX + tx] = accA.x;
  part[(ty + 8) * kTX + tx] = accA.y;
  part[(ty + 16) * kTX + tx] = accB.x;
  part[(ty + 24) * kTX + tx] = accB.y;
  cluster.sync();
  for (int p = threadIdx.x; p < kTX * kTY; p += 256) {
    if (p % G != rank) continue;
    float s = 0.0f;
    for (int g = 0; g < G; ++g) s += cluster.map_shared_rank(part, g)[p];
    const int ix = x0 + (p % kTX), iy = y0 + (p / kTX);
    if (ix < a.nx && iy < a.ny) {
      float* o = a.img + (long long)iy * a.nx + ix;
      const float v = s * a.scale;
      *o = a.accumulate ? *o + v : v;
    }
  }
  cluster.sync();  // keep this CTA's partials alive until every rank has read them
}

}  // namespace planar
}  // namespace tgb

using namespace tgb;
using namespace tgb::planar;

struct tg_planar_plan {
  int device = 0;
  uint64_t id = 0;
  tg_volume_spec vol{};
  tg_detector1d det{};
  uint64_t n_proj = 0;
  double range = 0, sid = 0, sdd = 0;
  bool fan = false;
  double* d_rays = nullptr;
  float4* d_quads = nullptr;  // K5/K7 scratch: both quad layouts
  ScratchOrder quads_order;
  int n_sm = 148;
  std::mutex mu;
};

namespace {

FpArgs fp_args(const tg_planar_plan& p) {
  FpArgs a{};
  a.nb = int(p.det.n_bins);
  a.n_views = int(p.n_proj);
  a.nx = int(p.vol.shape[0]);
  a.ny = int(p.vol.shape[1]);
  a.ox = p.vol.origin[0];
  a.oy = p.vol.origin[1];
  a.sx = p.vol.spacing[0];
  a.sy = p.vol.spacing[1];
  a.step = 0.5 * ((a.sy < a.sx) ? a.sy : a.sx);  // projector.hpp:103-107
  a.det_origin = p.det.origin;
  a.det_spacing = p.det.spacing;
  a.sid = p.sid;
  a.sdd = p.sdd;
  a.fan = p.fan;
  a.rays = p.d_rays;
  a.nxp = a.nx + 4;
  a.nyp = a.ny + 4;
  return a;
}

void planar_forward_impl(tg_planar_plan& p, const float* d_img, float* d_sino, cudaStream_t st) {
  DeviceGuard dg(p.device);
  std::lock_guard<std::mutex> lk(p.mu);
  FpArgs a = fp_args(p);
  const size_t nq = size_t(a.nxp) * a.nyp;
  if (!p.d_quads) TG_CUDA(cudaMalloc(&p.d_quads, 2 * nq * sizeof(float4)));
  p.quads_order.enter(st);
  pad_quads_kernel<<<p.n_sm * 4, 256, 0, st>>>(d_img, p.d_quads, p.d_quads + nq, a.nx, a.ny);
  TG_LAUNCHED(1);
  a.q = p.d_quads;
  a.qT = p.d_quads + nq;
  a.out = d_sino;
  // segments per ray: 4 measured best at both c1 (131k rays) and c2 (369k rays)
  // (c2: 1 / 2 / 4 / 8 segments 557 / 430 / 389 / 425 us), fewer for long scans
  const long long rays = (long long)a.n_views * a.nb;
  int S = rays <= 1500000 ? 4 : (rays <= 3000000 ? 2 : 1);
  if (const char* e = std::getenv("TG_PLANAR_SEGS")) S = std::max(1, std::min(8, std::atoi(e)));
  a.segs = S;
  const long long groups = (rays + 31) / 32;  // 32-ray groups, 8 / S per CTA
  KernelTimer timer;
  timer.start(st);
  const unsigned nb = unsigned((groups + 8 / S - 1) / (8 / S));
  // re-gather only when the cell changes (at 6 CTAs / SM: c2 320 vs 333 us for
  // unconditional gathers; at 4 CTAs / SM the unconditional ones won by 2%);
  // TG_PLANAR_REUSE=0 selects them
  static const int reuse = [] {
    const char* e = std::getenv("TG_PLANAR_REUSE");
    return e ? std::atoi(e) : 1;
  }();
  if (reuse)
    planar_fp_kernel<true><<<nb, 256, 0, st>>>(a);
  else
    planar_fp_kernel<false><<<nb, 256, 0, st>>>(a);
  TG_LAUNCHED(1);
  timer.stop();
  p.quads_order.leave(st);
}

template <bool FAN>
void launch_bp(const BpArgs& a, dim3 grid, int G, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = unsigned(G);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TG_CUDA(cudaLaunchKernelEx(&cfg, planar_bp_kernel<FAN>, a));
}

void planar_backproject_impl(tg_planar_plan& p, const float* d_sino, float* d_img, float scale,
                             int accumulate, cudaStream_t st) {
  DeviceGuard dg(p.device);
  BpArgs a{};
  a.nx = int(p.vol.shape[0]);
  a.ny = int(p.vol.shape[1]);
  a.nb = int(p.det.n_bins);
  a.n_views = int(p.n_proj);
  a.ox = p.vol.origin[0];
  a.oy = p.vol.origin[1];
  a.sx = p.vol.spacing[0];
  a.sy = p.vol.spacing[1];
  a.det_origin = p.det.origin;
  a.det_spacing = p.det.spacing;
  a.inv_ds = 1.0 / p.det.spacing;  // projector.hpp:193
  a.sid = p.sid;
  a.sdd = p.sdd;
  a.rays = p.d_rays;
  a.scale = scale;
  a.accumulate = accumulate;
  a.sino = d_sino;
  a.img = d_img;
  const dim3 tiles((a.nx + kTX - 1) / kTX, (a.ny + kTY - 1) / kTY, 1);
  // views split over a cluster of G CTAs per tile, at least 16 views per CTA:
  // 8 measured best at c1 (64 tiles) and c2 (256 tiles) — c2 4 / 5 / 8 / 12 /
  // 16: 89.9 / 90.3 / 88.3 / 108 / 125 us (12 and 16 need non-portable clusters)
  int G = std::max(1, std::min(kMaxCluster, a.n_views / 16));
  if (const char* e = std::getenv("TG_PLANAR_G")) G = std::max(1, std::min(kMaxCluster, std::atoi(e)));
  a.vpg = (a.n_views + G - 1) / G;
  KernelTimer timer;
  timer.start(st);
  const dim3 grid(tiles.x, tiles.y, unsigned(G));
  if (p.fan)
    launch_bp<true>(a, grid, G, st);
  else
    launch_bp<false>(a, grid, G, st);
  TG_LAUNCHED(1);
  timer.stop();
}

}  // namespace

extern "C" {

tg_status tg_planar_plan_create(const tg_planar_geometry* g, int device, tg_planar_plan** out) {
  return guarded([&] {
    *out = nullptr;
    validate_volume(g->volume);
    const bool fan = g->sdd != 0.0 || g->sid != 0.0;
    check(g->volume.dims == 2, fan ? "fan beam geometry expects a 2D volume"
                                   : "parallel beam geometry expects a 2D volume");
    if (fan) check(g->sid > 0.0 && g->sdd > g->sid, "fan beam requires 0 < SID < SDD");
    check(g->n_projections >= 1, "need at least one projection");
    check(g->detector.n_bins >= 1, "detector needs at least one bin");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device visible: the B200 path has no CPU fallback");
    }
    auto p = std::make_unique<tg_planar_plan>();
    p->device = device;
    p->id = next_plan_id();
    p->vol = g->volume;
    p->det = g->detector;
    p->n_proj = g->n_projections;
    p->range = g->angular_range;
    p->sid = g->sid;
    p->sdd = g->sdd;
    p->fan = fan;
    const uint64_t n = g->n_projections;
    DeviceGuard dg(device);
    TG_CUDA(cudaDeviceGetAttribute(&p->n_sm, cudaDevAttrMultiProcessorCount, device));
    TG_CUDA(cudaMalloc(&p->d_rays, 2 * n * sizeof(double)));
    TG_CUDA(cudaMemcpy(p->d_rays, g->rays, 2 * n * sizeof(double), cudaMemcpyHostToDevice));
    *out = p.release();
  });
}

tg_status tg_planar_plan_destroy(tg_planar_plan* p) {
  return guarded([&] {
    if (!p) return;
    DeviceGuard dg(p->device);
    cudaFree(p->d_rays);
    cudaFree(p->d_quads);
    delete p;
  });
}

tg_status tg_planar_plan_shape(const tg_planar_plan* p, tg_volume_spec* vol, tg_detector1d* det,
                               uint64_t* n_proj) {
  return guarded([&] {
    check(p != nullptr, "null plan");
    if (vol) *vol = p->vol;
    if (det) *det = p->det;
    if (n_proj) *n_proj = p->n_proj;
  });
}

tg_status tg_planar_forward(tg_planar_plan* p, const float* d_img, float* d_sino, void* stream) {
  return guarded([&] { planar_forward_impl(*p, d_img, d_sino, as_stream(stream)); });
}

tg_status tg_planar_backproject(tg_planar_plan* p, const float* d_sino, float* d_img, float scale,
                                int accumulate, void* stream) {
  return guarded(
      [&] { planar_backproject_impl(*p, d_sino, d_img, scale, accumulate, as_stream(stream)); });
}

tg_status tg_planar_ray_samples(tg_planar_plan* p, uint64_t* d_counts, void* stream) {
  return guarded([&] {
    check(p != nullptr, "null plan");
    DeviceGuard dg(p->device);
    const FpArgs a = fp_args(*p);
    const long long rays = (long long)a.n_views * a.nb;
    planar_ray_samples_kernel<<<unsigned((rays + 255) / 256), 256, 0, as_stream(stream)>>>(
        a, reinterpret_cast<unsigned long long*>(d_counts));
    TG_LAUNCHED(1);
  });
}

tg_status tg_planar_forward_host(tg_planar_plan* p, const float* h_img, float* h_sino) {
  return guarded([&] {
    DeviceGuard dg(p->device);
    const size_t ni = p->vol.shape[0] * p->vol.shape[1], ns = p->n_proj * p->det.n_bins;
    float *di = nullptr, *ds = nullptr;
    TG_CUDA(cudaMalloc(&di, ni * sizeof(float)));
    TG_CUDA(cudaMalloc(&ds, ns * sizeof(float)));
    TG_CUDA(cudaMemcpy(di, h_img, ni * sizeof(float), cudaMemcpyHostToDevice));
    planar_forward_impl(*p, di, ds, 0);
    TG_CUDA(cudaMemcpy(h_sino, ds, ns * sizeof(float), cudaMemcpyDeviceToHost));
    TG_CUDA(cudaFree(di));
    TG_CUDA(cudaFree(ds));
  });
}

tg_status tg_planar_backproject_host(tg_planar_plan* p, const float* h_sino, float* h_img) {
  return guarded([&] {
    DeviceGuard dg(p->device);
    const size_t ni = p->vol.shape[0] * p->vol.shape[1], ns = p->n_proj * p->det.n_bins;
    float *di = nullptr, *ds = nullptr;
    TG_CUDA(cudaMalloc(&di, ni * sizeof(float)));
    TG_CUDA(cudaMalloc(&ds, ns * sizeof(float)));
    TG_CUDA(cudaMemcpy(ds, h_sino, ns * sizeof(float), cudaMemcpyHostToDevice));
    planar_backproject_impl(*p, ds, di, 1.0f, 0, 0);
    TG_CUDA(cudaMemcpy(h_img, di, ni * sizeof(float), cudaMemcpyDeviceToHost));
    TG_CUDA(cudaFree(di));
    TG_CUDA(cudaFree(ds));
  });
}

}  // extern "C"
