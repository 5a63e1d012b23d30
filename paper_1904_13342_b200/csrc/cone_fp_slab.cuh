// cone_fp_slab.cuh — K2, ray-driven cone forward projection with the volume
// staged through shared memory (projector.hpp:264-281 over 130-152, 83-107,
// 66-78).  Included by cone.cu inside namespace tgb::cone after FpArgs,
// cone_ray() and ray_sample_count().
//
// A CTA owns a TU x TV tile of detector pixels of one view (256 rays, one
// per consumer thread) and sweeps the volume in slabs of T cells along the
// tile's dominant axis (x or y, whichever the rays advance along faster).
// Per slab a producer warp computes the box that holds every trilinear tap
// of every ray sample in the slab — the rays of a pixel rectangle from one
// source form a convex pyramid, so the extremes of its transverse
// coordinates over the slab sit on the 4 corner rays at the 2 bounding
// planes (FP64, one voxel of margin) — and issues one TMA box load of
// WH (transverse) x HZ (z) x (T + 2) (dominant) voxels into a ring of
// stages.  Consumers march their rays' samples through the slab reading
// the 8 taps from shared memory.  Rays whose tile runs along x read a
// y-fastest copy of the volume (Vt[z][x][y]) so that the transverse axis is
// the fastest in shared memory for both orientations.
//
// Box layout [dominant][z][transverse]: the tensor maps traverse the volume
// with permuted strides (dims (h, z, d)).  A warp holds 8 (u) x 4 (v) rays, so
// at one sample its lanes sit on ~8 transverse columns x 4 z rows and at most
// two neighbouring dominant planes.  With WH = 8 (mod 32) the 4 z rows start
// 8 banks apart and with HZ = 0 (mod 4) a dominant step moves 0 banks: the
// 32 lanes fall on distinct banks (or share a word) in the common case.
// ([z][dominant][h] with WH = 32 put all 4 z rows and both planes on one
// bank set: 4.7 shared wavefronts per LDS, profiles/r2_k2_slab_v1_ncu.json.)
//
// Sample positions, sample order and the accumulation are those of the
// L1-gather K2 (quad-volume) kernel: sample k at t0 + (k + 1/2) dt, fp32
// offsets from FP64 anchors every 64 samples, fp32 chunk sums folded into a
// double — the output is bitwise identical to it.  TMA fills out-of-volume
// voxels with zeros: the reference's zero-padded interp3 (projector.hpp:66-78).
// Slabs whose box does not fit (rare oblique tiles) gather from global
// memory with explicit bounds checks — same taps, same bits.
#pragma once

namespace fps {

constexpr int NCONS = 256;            // consumer threads = rays per CTA
constexpr int NTHREADS = NCONS + 32;  // + producer warp
constexpr int MAX_STAGES = 4;
constexpr int MODE_SMEM = 0, MODE_GLOBAL = 1;
constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23: t = M + floor(p) under round-down
constexpr int MAGIC_BITS = 0x4B400000;

struct Args {
  FpArgs f;                        // geometry, clip, output (vq / vqT unused)
  const float* __restrict__ vol;   // V[z][y][x] (global fallback)
  int boxZ;                        // box extent along z (multiple of 4)
  int T;                           // slab thickness (dominant cells); box holds T + 2 planes
  int stages;                      // ring depth (<= MAX_STAGES)
  unsigned long long* __restrict__ stats;  // optional: [slabs, global slabs, global CTAs]
};

struct StageHdr {
  int hb, zb, s0, mode;  // box origin (transverse, z), first dominant cell, mode
};

struct CtaHdr {
  int axis;  // 0: y-dominant (V, h = x), 1: x-dominant (Vt, h = y), 2: global
  int dir;   // +1 / -1 along the dominant axis
  int cmin, cmax;
};

// Per-ray FP64 state parked in shared memory (anchors are recomputed every
// 64 samples; keeping them out of registers leaves room for the taps), as a
// structure of arrays: field f of ray t at v[f * NCONS + t], so a warp's
// 8-byte reads are conflict-free (a 64-byte per-ray struct made them 16-way).
struct RayState {
  double v[8 * NCONS];
};
struct RayRef {
  double* v;
  __device__ __forceinline__ double& p0(int i) const { return v[i * NCONS]; }
  __device__ __forceinline__ double& dd(int i) const { return v[(3 + i) * NCONS]; }
  __device__ __forceinline__ double& dt() const { return v[6 * NCONS]; }
  __device__ __forceinline__ double& inv_dd() const { return v[7 * NCONS]; }
};

template <uint32_t OZ>
__device__ __forceinline__ void lds4(uint32_t ad, float& a0, float& a1, float& a2, float& a3) {
  asm volatile(
      "ld.shared.f32 %0, [%4];\n\t"
      "ld.shared.f32 %1, [%4+4];\n\t"
      "ld.shared.f32 %2, [%4+%5];\n\t"
      "ld.shared.f32 %3, [%4+%6];"
      : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
      : "r"(ad), "n"(OZ), "n"(OZ + 4));
}

__device__ __forceinline__ float vat(const Args& a, int x, int y, int z) {
  const FpArgs& f = a.f;
  return ((unsigned)x < (unsigned)f.nx && (unsigned)y < (unsigned)f.ny && (unsigned)z < (unsigned)f.nz)
             ? __ldg(a.vol + ((long long)z * f.ny + y) * f.nx + x)
             : 0.0f;
}

// One ray's march state between slabs.
struct Ray {
  int n, k, k0, m;     // samples, next sample, chunk start, chunk length
  int cx, cy, cz;      // chunk anchor cell (unpadded voxel index)
  float bx, by, bz;    // chunk anchor offset within the cell
  float fdx, fdy, fdz; // per-sample step (voxels)
  float sum;           // current chunk's fp32 sum
  double total;
};

__device__ __forceinline__ void anchor(Ray& r, const RayRef& rs) {
  // identical to the quad-volume kernel: padded index coordinates (+2)
  const double ax = rs.p0(0) + double(r.k0) * rs.dd(0), ay = rs.p0(1) + double(r.k0) * rs.dd(1),
               az = rs.p0(2) + double(r.k0) * rs.dd(2);
  const double cx = floor(ax), cy = floor(ay), cz = floor(az);
  r.bx = float(ax - cx);
  r.by = float(ay - cy);
  r.bz = float(az - cz);
  r.cx = int(cx) - 2;
  r.cy = int(cy) - 2;
  r.cz = int(cz) - 2;
  r.m = min(64, r.n - r.k0);
}

// Taps of one sample at box byte address ad (plane d) and ad + od (plane d+1),
// in the quad kernel's order: q0 = slice z (x,y) (x+1,y) (x,y+1) (x+1,y+1),
// q1 = slice z + 1.
template <int WH, bool XDOM>
__device__ __forceinline__ void taps_smem(uint32_t ad, uint32_t od, float4& q0, float4& q1) {
  constexpr uint32_t OZ = 4u * WH;
  float a0, a1, a2, a3, b0, b1, b2, b3;
  lds4<OZ>(ad, a0, a1, a2, a3);       // plane d: (h, z) (h+1, z) (h, z+1) (h+1, z+1)
  lds4<OZ>(ad + od, b0, b1, b2, b3);  // plane d + 1
  if (XDOM) {  // h = y, d = x
    q0 = make_float4(a0, b0, a1, b1);
    q1 = make_float4(a2, b2, a3, b3);
  } else {     // h = x, d = y
    q0 = make_float4(a0, a1, b0, b1);
    q1 = make_float4(a2, a3, b2, b3);
  }
}

__device__ __forceinline__ void taps_global(const Args& a, const Ray& r, int bxi, int byi, int bzi,
                                            float4& q0, float4& q1) {
  const int x = r.cx + (bxi - MAGIC_BITS), y = r.cy + (byi - MAGIC_BITS), z = r.cz + (bzi - MAGIC_BITS);
  q0 = make_float4(vat(a, x, y, z), vat(a, x + 1, y, z), vat(a, x, y + 1, z), vat(a, x + 1, y + 1, z));
  q1 = make_float4(vat(a, x, y, z + 1), vat(a, x + 1, y, z + 1), vat(a, x, y + 1, z + 1),
                   vat(a, x + 1, y + 1, z + 1));
}

__device__ __forceinline__ float trilerp(const float4& q0, const float4& q1, float wx, float wy,
                                         float wz) {
  const float c0 = lerpf(lerpf(q0.x, q0.y, wx), lerpf(q0.z, q0.w, wx), wy);
  const float c1 = lerpf(lerpf(q1.x, q1.y, wx), lerpf(q1.z, q1.w, wx), wy);
  return lerpf(c0, c1, wz);
}

// Byte address of the chunk anchor cell in the box (magic bias folded in).
template <int WH, bool XDOM>
__device__ __forceinline__ uint32_t chunk_base(const Ray& r, uint32_t sbase, uint32_t od, int hb,
                                               int d0, int zb) {
  constexpr uint32_t OZ = 4u * WH;
  const int ch = XDOM ? r.cy : r.cx, cd = XDOM ? r.cx : r.cy;
  return sbase + 4u * uint32_t(ch - hb) + OZ * uint32_t(r.cz - zb) + od * uint32_t(cd - d0) -
         uint32_t(MAGIC_BITS) * (4u + OZ + od);
}

// Samples [k, k + 2 pairs) of the ray, in pairs on the FP32x2 pipe with the
// scalar kernel's exact operations (FFMA2 / FADD2 round like FFMA / FADD),
// summed in order.  Every lane of the warp runs the same number of loop trips
// (the warp's largest pair count; lanes with fewer are masked off), so the
// 32 lanes stay converged across slab boundaries.  Pairs start at even
// sample indices within the 64-sample chunk, so a pair never straddles a
// chunk's FP64 anchor; the chunk is re-anchored inline.  The second sample of
// a ray's last pair is masked when the ray has an odd count.
//   box: gathers from the stage box (od = byte pitch of a dominant plane,
//   d0 = its first plane); else global memory (bounds-checked).
template <int WH, bool XDOM, bool SMEM>
__device__ __forceinline__ void march(const Args& a, Ray& r, const RayRef& rs, int pairs,
                                      uint32_t sbase, uint32_t od, int hb, int d0, int zb) {
  constexpr uint32_t OZ = 4u * WH;  // byte offset of z + 1
  const float2 M2 = make_float2(MAGIC, MAGIC), nM2 = make_float2(-MAGIC, -MAGIC);
  const int P = __reduce_max_sync(0xffffffffu, pairs);
  uint32_t cbase = chunk_base<WH, XDOM>(r, sbase, od, hb, d0, zb);
  float sum = r.sum;
#pragma unroll 2
  for (int p = 0; p < P; ++p) {
    if (p < pairs) {
      if (r.k - r.k0 == 64) {
        r.total += double(sum);
        sum = 0.0f;
        r.k0 += 64;
        anchor(r, rs);
        cbase = chunk_base<WH, XDOM>(r, sbase, od, hb, d0, zb);
      }
      const int j = r.k - r.k0;
      const float2 jj = make_float2(float(j), float(j + 1));
      const float2 px = __ffma2_rn(jj, make_float2(r.fdx, r.fdx), make_float2(r.bx, r.bx));
      const float2 py = __ffma2_rn(jj, make_float2(r.fdy, r.fdy), make_float2(r.by, r.by));
      const float2 pz = __ffma2_rn(jj, make_float2(r.fdz, r.fdz), make_float2(r.bz, r.bz));
      const float2 tx = __fadd2_rd(px, M2), ty = __fadd2_rd(py, M2), tz = __fadd2_rd(pz, M2);
      const float2 fx = __fadd2_rn(tx, nM2), fy = __fadd2_rn(ty, nM2), fz = __fadd2_rn(tz, nM2);
      const float2 wx = __fadd2_rn(px, make_float2(-fx.x, -fx.y));
      const float2 wy = __fadd2_rn(py, make_float2(-fy.x, -fy.y));
      const float2 wz = __fadd2_rn(pz, make_float2(-fz.x, -fz.y));
      float4 q0a, q1a, q0b, q1b;
      if (SMEM) {
        const uint32_t bha = __float_as_uint(XDOM ? ty.x : tx.x), bhb = __float_as_uint(XDOM ? ty.y : tx.y);
        const uint32_t bda = __float_as_uint(XDOM ? tx.x : ty.x), bdb = __float_as_uint(XDOM ? tx.y : ty.y);
        taps_smem<WH, XDOM>(cbase + 4u * bha + OZ * __float_as_uint(tz.x) + od * bda, od, q0a, q1a);
        taps_smem<WH, XDOM>(cbase + 4u * bhb + OZ * __float_as_uint(tz.y) + od * bdb, od, q0b, q1b);
      } else {
        taps_global(a, r, __float_as_int(tx.x), __float_as_int(ty.x), __float_as_int(tz.x), q0a, q1a);
        taps_global(a, r, __float_as_int(tx.y), __float_as_int(ty.y), __float_as_int(tz.y), q0b, q1b);
      }
      // the three lerp levels of both samples on the FP32x2 pipe
      const float2 p00 = make_float2(q0a.x, q0b.x), p01 = make_float2(q0a.y, q0b.y);
      const float2 p10 = make_float2(q0a.z, q0b.z), p11 = make_float2(q0a.w, q0b.w);
      const float2 r00 = make_float2(q1a.x, q1b.x), r01 = make_float2(q1a.y, q1b.y);
      const float2 r10 = make_float2(q1a.z, q1b.z), r11 = make_float2(q1a.w, q1b.w);
      auto lerp2 = [](float2 u, float2 v, float2 w) {
        return __ffma2_rn(w, __fadd2_rn(v, make_float2(-u.x, -u.y)), u);
      };
      const float2 c0 = lerp2(lerp2(p00, p01, wx), lerp2(p10, p11, wx), wy);
      const float2 c1 = lerp2(lerp2(r00, r01, wx), lerp2(r10, r11, wx), wy);
      const float2 v = lerp2(c0, c1, wz);
      sum += v.x;
      if (r.k + 1 < r.n) sum += v.y;
      r.k = min(r.k + 2, r.n);
    }
  }
  r.sum = sum;
}

template <int TU, int WH>
__global__ void __launch_bounds__(NTHREADS, 2)
    cone_fp_slab_kernel(const __grid_constant__ CUtensorMap tmapX,
                        const __grid_constant__ CUtensorMap tmapY, const Args a) {
  constexpr int TV = NCONS / TU;
  extern __shared__ __align__(128) unsigned char smem[];
  const FpArgs& f = a.f;
  const int T = a.T;
  const int box_elems = WH * a.boxZ * (T + 2);
  const int stage_elems = (box_elems + 31) & ~31;
  float* boxes = reinterpret_cast<float*>(smem);
  RayState* rstate = reinterpret_cast<RayState*>(boxes + a.stages * stage_elems);
  StageHdr* hdr = reinterpret_cast<StageHdr*>(rstate + 1);
  CtaHdr* cta = reinterpret_cast<CtaHdr*>(hdr + MAX_STAGES);
  uint64_t* full = reinterpret_cast<uint64_t*>(cta + 1);
  uint64_t* empty = full + MAX_STAGES;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int u_lo = blockIdx.x * TU, v_lo = blockIdx.z * TV;
  const int view = f.view0 + blockIdx.y;
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS / 32);
    }
    mbar_fence_init();
    cta->cmin = 0x7fffffff;
    cta->cmax = -0x7fffffff;
  }

  // ---- producer: corner rays of the tile in index space (FP64) -------------
  // lane c < 4 holds corner c's line as h(P) = hA + P hB, z(P) = zA + P zB
  // over the dominant index coordinate P
  double hA = 0, hB = 0, zA = 0, zB = 0;
  if (w == NCONS / 32) {
    const int iu = (lane & 1) ? min(u_lo + TU, f.nu) - 1 : u_lo;
    const int iv = (lane & 2) ? min(v_lo + TV, f.nv) - 1 : v_lo;
    const double* g = f.geo + 12 * view;
    const double* M = g + 3;
    double e[3], o[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) e[r] = M[3 * r] * double(iu) + M[3 * r + 1] * double(iv) + M[3 * r + 2];
    o[0] = (g[0] - f.ox) / f.sx;
    o[1] = (g[1] - f.oy) / f.sy;
    o[2] = (g[2] - f.oz) / f.sz;
    e[0] /= f.sx;
    e[1] /= f.sy;
    e[2] /= f.sz;
    // axis from the summed corner directions; every corner must advance
    // along it with the same sign and at least 0.3 of its length (then
    // consecutive samples move >= 0.15 voxel along it: the dominant cell
    // never steps back, and the box stays small)
    double sx = (lane < 4) ? e[0] : 0.0, sy = (lane < 4) ? e[1] : 0.0;
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, off);
      sy += __shfl_xor_sync(0xffffffffu, sy, off);
    }
    const bool xdom = fabs(sx) > fabs(sy);
    const double ed = xdom ? e[0] : e[1], eh = xdom ? e[1] : e[0];
    const double od = xdom ? o[0] : o[1], oh = xdom ? o[1] : o[0];
    const double len = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
    int ok = (lane >= 4) || (fabs(ed) >= 0.3 * len);
    int pos = (lane >= 4) || ed > 0.0, neg = (lane >= 4) || ed < 0.0;
    ok = __all_sync(0xffffffffu, ok);
    pos = __all_sync(0xffffffffu, pos);
    neg = __all_sync(0xffffffffu, neg);
    hB = eh / ed;
    hA = oh - od * hB;
    zB = e[2] / ed;
    zA = o[2] - od * zB;
    if (lane == 0) {
      cta->axis = (ok && (pos || neg) && a.vol != nullptr) ? (xdom ? 1 : 0) : 2;
      cta->dir = pos ? 1 : -1;
    }
  }
  __syncthreads();
  const int axis = cta->axis;

  // ---- consumers: ray setup (FP64, bit-exact n / hit) ------------------------
  Ray r;
  r.n = 0;
  r.k = 0;
  r.k0 = 0;
  r.sum = 0.0f;
  r.total = 0.0;
  float* out = nullptr;
  if (tid < NCONS) {
    const int iu = u_lo + (w % (TU / 8)) * 8 + (lane & 7);
    const int iv = v_lo + (w / (TU / 8)) * 4 + (lane >> 3);
    int cmin = 0x7fffffff, cmax = -0x7fffffff;
    if (iu < f.nu && iv < f.nv) {
      out = f.out + ((long long)blockIdx.y * f.nv + iv) * f.nu + iu;
      double o[3], d[3], t0, t1;
      if (!cone_ray(f, iu, iv, view, o, d, t0, t1)) {
        // zero stored at the end with the warp's other results (whole sectors)
      } else {
        const double span = DADD(t1, -t0);
        r.n = int(ray_sample_count(span, f.step));
        const RayRef rs{rstate->v + tid};
        rs.dt() = DDIV(span, double(r.n));
        const double th = t0 + 0.5 * rs.dt();
        rs.p0(0) = (o[0] + th * d[0] - f.ox) / f.sx + 2.0;
        rs.p0(1) = (o[1] + th * d[1] - f.oy) / f.sy + 2.0;
        rs.p0(2) = (o[2] + th * d[2] - f.oz) / f.sz + 2.0;
        rs.dd(0) = rs.dt() * d[0] / f.sx;
        rs.dd(1) = rs.dt() * d[1] / f.sy;
        rs.dd(2) = rs.dt() * d[2] / f.sz;
        r.fdx = float(rs.dd(0));
        r.fdy = float(rs.dd(1));
        r.fdz = float(rs.dd(2));
        anchor(r, rs);
        if (axis < 2) {
          const int dax = axis == 1 ? 0 : 1;
          rs.inv_dd() = 1.0 / rs.dd(dax);
          const double first = rs.p0(dax), last = rs.p0(dax) + double(r.n - 1) * rs.dd(dax);
          // fp32 sample cells may differ from the FP64 ones by one
          cmin = int(floor(fmin(first, last))) - 3;
          cmax = int(floor(fmax(first, last))) - 1;
        }
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, off));
      cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
    }
    if (lane == 0 && cmin <= cmax) {
      atomicMin(&cta->cmin, cmin);
      atomicMax(&cta->cmax, cmax);
    }
  }
  __syncthreads();
  const int dir = cta->dir;
  const int cmin = cta->cmin, cmax = cta->cmax;
  // global mode: one pass over every sample; else slabs of T cells
  const int n_slabs = axis == 2 ? 1 : (cmin > cmax ? 0 : (cmax - cmin + T) / T);

  if (tid >= NCONS) {
    // ---------------- producer ----------------
    // each TMA names its tensor map directly (a run-time select between the two
    // parameter addresses makes the map operand non-uniform: illegal instruction)
    if (lane == 0 && axis == 0) prefetch_tensor_map(&tmapX);
    if (lane == 0 && axis == 1) prefetch_tensor_map(&tmapY);
    for (int i = 0; i < n_slabs; ++i) {
      const int s = i % a.stages;
      StageHdr h;
      h.mode = MODE_GLOBAL;
      h.hb = h.zb = 0;
      h.s0 = dir > 0 ? cmin + i * T : cmax + 1 - (i + 1) * T;
      // box planes [d0, d0 + T + 1]: the slab's cells [s0, s0 + T) plus one cell
      // of overhang in the march direction (a lane's last pair may take one
      // sample past the slab; samples within 1e-4 voxel of the entry plane
      // may be counted to the previous slab) — see the consumers' pair counts
      const int d0 = dir > 0 ? h.s0 : h.s0 - 1;
      if (axis < 2) {
        // every sample with dominant position in [d0, d0 + T + 1] (index space
        // of the unpadded volume): the hull of the 4 corner rays at those planes
        double hmin = 1e300, hmax = -1e300, zmin = 1e300, zmax = -1e300;
        if (lane < 4) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double P = double(d0 + e * (T + 1));
            const double hh = hA + P * hB, zz = zA + P * zB;
            hmin = fmin(hmin, hh);
            hmax = fmax(hmax, hh);
            zmin = fmin(zmin, zz);
            zmax = fmax(zmax, zz);
          }
        }
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
          hmin = fmin(hmin, __shfl_xor_sync(0xffffffffu, hmin, off));
          hmax = fmax(hmax, __shfl_xor_sync(0xffffffffu, hmax, off));
          zmin = fmin(zmin, __shfl_xor_sync(0xffffffffu, zmin, off));
          zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, off));
        }
        const bool finite = fabs(hmin) < 1e7 && fabs(hmax) < 1e7 && fabs(zmin) < 1e7 && fabs(zmax) < 1e7;
        if (finite) {
          // the inner TMA coordinate must be a multiple of 4 floats (16 bytes;
          // anything else is an illegal instruction, scripts/tma_box_test.cu)
          h.hb = (int(floor(hmin)) - 1) & ~3;
          h.zb = int(floor(zmin)) - 1;
          const int wneed = int(floor(hmax)) + 3 - h.hb, zneed = int(floor(zmax)) + 3 - h.zb;
          if (wneed <= WH && zneed <= a.boxZ) h.mode = MODE_SMEM;
        }
      }
      // the box is computed before the stage frees up: only the header write and
      // the TMA issue wait for the consumers
      if (i >= a.stages) mbar_wait(&empty[s], ((i / a.stages) - 1) & 1);
      if (lane == 0) {
        hdr[s] = h;
        if (a.stats) {
          atomicAdd(&a.stats[0], 1ull);
          if (h.mode != MODE_SMEM) atomicAdd(&a.stats[1], 1ull);
          if (i == 0 && axis == 2) atomicAdd(&a.stats[2], 1ull);
        }
        if (h.mode == MODE_SMEM) {
          mbar_arrive_expect_tx(&full[s], uint32_t(box_elems * 4));
          if (axis == 1)
            tma_load_3d(boxes + s * stage_elems, &tmapY, &full[s], h.hb, h.zb, d0);
          else
            tma_load_3d(boxes + s * stage_elems, &tmapX, &full[s], h.hb, h.zb, d0);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- consumers ----------------
  const uint32_t box_base = smem_u32(boxes);
  for (int i = 0; i < n_slabs; ++i) {
    const int s = i % a.stages;
    mbar_wait(&full[s], (i / a.stages) & 1);
    const StageHdr h = hdr[s];
    const RayRef rs{rstate->v + tid};
    // this slab's samples: every sample whose exact (FP64) dominant position
    // lies in the slab's cells, up to 1e-4 voxel past its far plane (so no
    // sample whose fp32 cell is still inside is left behind), as whole pairs
    int pairs = 0;
    if (r.k < r.n) {
      if (axis == 2) {
        pairs = (r.n - r.k + 1) >> 1;
      } else {
        const double p0d = rs.p0(axis == 1 ? 0 : 1);  // padded coordinates (+2)
        double kf;
        if (dir > 0)
          kf = ceil((double(h.s0 + T) + 2.0 + 1e-4 - p0d) * rs.inv_dd());
        else
          kf = floor((double(h.s0) + 2.0 - 1e-4 - p0d) * rs.inv_dd()) + 1.0;
        kf = fmin(fmax(kf, double(r.k)), double(r.n));
        pairs = (int(kf) - r.k + 1) >> 1;
      }
    }
    {
      const int d0 = dir > 0 ? h.s0 : h.s0 - 1;
      const uint32_t sb = box_base + uint32_t(s * stage_elems) * 4u;
      const uint32_t od = 4u * uint32_t(WH * a.boxZ);
      if (h.mode == MODE_SMEM) {
        if (axis == 1)
          march<WH, true, true>(a, r, rs, pairs, sb, od, h.hb, d0, h.zb);
        else
          march<WH, false, true>(a, r, rs, pairs, sb, od, h.hb, d0, h.zb);
      } else if (axis == 1) {
        march<WH, true, false>(a, r, rs, pairs, sb, od, h.hb, d0, h.zb);
      } else {
        march<WH, false, false>(a, r, rs, pairs, sb, od, h.hb, d0, h.zb);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (out) {
    r.total += double(r.sum);
    *out = r.n > 0 ? float(r.total * RayRef{rstate->v + tid}.dt()) : 0.0f;
  }
}

}  // namespace fps
