// planar.cu — parallel- and fan-beam 2D operators (K4-K7).
//   K7 parallel forward  projector.hpp:171-184   K6 parallel back  projector.hpp:186-208
//   K5 fan forward       projector.hpp:212-230   K4 fan back (1/U^2) projector.hpp:232-260
// Ray setup, clipping and sample counts run in IEEE FP64 without contraction
// (bit-exact hit test and n); marching, interpolation and accumulation run
// in fp32 with FP64 chunk anchors.
#include <algorithm>
#include <memory>
#include <vector>

#include "device_common.cuh"

namespace tgb {
namespace planar {

constexpr int kMaxConstViews = 2048;
// per view (FP64): parallel -> detector axis (-r.y, r.x); fan -> ray r
__constant__ double2 c_pviews[kMaxConstViews];
static ConstBank g_bank;

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
  const float* __restrict__ ipad;   // zero-bordered image (+2 each side)
  int nxp;
  float* out;
};

__device__ __forceinline__ bool clip_ray2(const FpArgs& a, const double o[2], const double d[2],
                                          double& t0, double& t1) {
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

__device__ __forceinline__ float lerpf(float a, float b, float w) { return fmaf(w, b - a, a); }

__global__ void __launch_bounds__(256) planar_fp_kernel(const FpArgs a) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)a.n_views * a.nb) return;
  const int i = int(idx / a.nb), j = int(idx % a.nb);
  const double rx = a.rays[2 * i], ry = a.rays[2 * i + 1];
  const double axx = -ry, axy = rx;
  double o[2], d[2];
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
  double t0, t1;
  if (!clip_ray2(a, o, d, t0, t1)) {
    a.out[idx] = 0.0f;
    return;
  }
  const double span = DADD(t1, -t0);
  const long long n = (long long)ceil(DDIV(span, a.step));
  const double dt = DDIV(span, double(n));
  const double th = t0 + 0.5 * dt;
  const double p0x = (o[0] + th * d[0] - a.ox) / a.sx + 2.0;
  const double p0y = (o[1] + th * d[1] - a.oy) / a.sy + 2.0;
  const double ddx = dt * d[0] / a.sx, ddy = dt * d[1] / a.sy;
  const float fdx = float(ddx), fdy = float(ddy);
  double total = 0.0;
  for (long long k0 = 0; k0 < n; k0 += 64) {
    // integer cell + small fp32 offset keeps sample positions precise
    const double ax = p0x + double(k0) * ddx, ay = p0y + double(k0) * ddy;
    const double cx = floor(ax), cy = floor(ay);
    const float bx = float(ax - cx), by = float(ay - cy);
    const float* cell = a.ipad + (long long)cy * a.nxp + (long long)cx;
    const int m = int(min(64LL, n - k0));
    float sum = 0.0f;
    for (int k = 0; k < m; ++k) {
      const float px = fmaf(float(k), fdx, bx), py = fmaf(float(k), fdy, by);
      const float fx = floorf(px), fy = floorf(py);
      const float wx = px - fx, wy = py - fy;
      const float* b = cell + (long long)int(fy) * a.nxp + int(fx);
      sum += lerpf(lerpf(__ldg(b), __ldg(b + 1), wx), lerpf(__ldg(b + a.nxp), __ldg(b + a.nxp + 1), wx),
                   wy);
    }
    total += double(sum);
  }
  a.out[idx] = float(total * dt);
}

struct BpArgs {
  int nx, ny, nb, n_views, view_base;
  double ox, oy, sx, sy;
  double det_origin, inv_ds;
  double sid, sdd;
  int fan;
  float scale;
  int accumulate;
  const float* __restrict__ sino;
  float* img;
};

// zero-padded linear interpolation along one sinogram row (projector.hpp:32-41)
__device__ __forceinline__ double interp_row(const float* __restrict__ row, int n, double t) {
  const double f = floor(t);
  const int i0 = int(f);
  const double w1 = t - f;
  double acc = 0.0;
  if (i0 >= 0 && i0 < n) acc += (1.0 - w1) * double(__ldg(row + i0));
  if (i0 + 1 >= 0 && i0 + 1 < n) acc += w1 * double(__ldg(row + i0 + 1));
  return acc;
}

// K6 / K4: one thread per pixel, views from the constant bank.  These 2D
// operators are launch-bound at the BASELINE sizes (c1 2.4e7, c2 9.4e7
// updates), so the per-update geometry runs in FP64 like the reference.
__global__ void __launch_bounds__(256) planar_bp_kernel(const BpArgs a) {
  const int ix = blockIdx.x * 32 + threadIdx.x, iy = blockIdx.y * 8 + threadIdx.y;
  if (ix >= a.nx || iy >= a.ny) return;
  const double x = a.ox + double(ix) * a.sx;
  const double y = a.oy + double(iy) * a.sy;
  double acc = 0.0;
  for (int i = 0; i < a.n_views; ++i) {
    const double2 c = c_pviews[i];
    const float* row = a.sino + (long long)(a.view_base + i) * a.nb;
    if (!a.fan) {
      const double s = x * c.x + y * c.y;
      acc += interp_row(row, a.nb, (s - a.det_origin) * a.inv_ds);
    } else {
      const double qx = x + a.sid * c.x, qy = y + a.sid * c.y;
      const double depth = qx * c.x + qy * c.y;
      if (depth <= 0.0) continue;  // behind the source
      const double u = a.sdd * (qx * -c.y + qy * c.x) / depth;
      const double U = depth / a.sid;
      acc += interp_row(row, a.nb, (u - a.det_origin) * a.inv_ds) / (U * U);
    }
  }
  float* o = a.img + (long long)iy * a.nx + ix;
  const float v = float(acc) * a.scale;
  *o = a.accumulate ? *o + v : v;
}

__global__ void pad_image_kernel(const float* __restrict__ img, float* __restrict__ ipad, int nx,
                                 int ny) {
  const int nxp = nx + 4, nyp = ny + 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)nxp * nyp;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = int(i % nxp) - 2, y = int(i / nxp) - 2;
    ipad[i] = (x >= 0 && x < nx && y >= 0 && y < ny) ? __ldg(img + (long long)y * nx + x) : 0.0f;
  }
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
  double2* d_coef = nullptr;
  float* d_ipad = nullptr;
  std::mutex mu;
};

namespace {

void planar_forward_impl(tg_planar_plan& p, const float* d_img, float* d_sino, cudaStream_t st) {
  DeviceGuard dg(p.device);
  std::lock_guard<std::mutex> lk(p.mu);
  const int nx = int(p.vol.shape[0]), ny = int(p.vol.shape[1]);
  if (!p.d_ipad) TG_CUDA(cudaMalloc(&p.d_ipad, size_t(nx + 4) * (ny + 4) * sizeof(float)));
  pad_image_kernel<<<148 * 4, 256, 0, st>>>(d_img, p.d_ipad, nx, ny);
  TG_LAUNCHED(1);
  FpArgs a;
  a.nb = int(p.det.n_bins);
  a.n_views = int(p.n_proj);
  a.nx = nx;
  a.ny = ny;
  a.ox = p.vol.origin[0];
  a.oy = p.vol.origin[1];
  a.sx = p.vol.spacing[0];
  a.sy = p.vol.spacing[1];
  a.step = 0.5 * ((a.sy < a.sx) ? a.sy : a.sx);
  a.det_origin = p.det.origin;
  a.det_spacing = p.det.spacing;
  a.sid = p.sid;
  a.sdd = p.sdd;
  a.fan = p.fan;
  a.rays = p.d_rays;
  a.ipad = p.d_ipad;
  a.nxp = nx + 4;
  a.out = d_sino;
  const long long total = (long long)a.n_views * a.nb;
  KernelTimer timer;
  timer.start(st);
  planar_fp_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(a);
  TG_LAUNCHED(1);
  timer.stop();
}

void planar_backproject_impl(tg_planar_plan& p, const float* d_sino, float* d_img, float scale,
                             int accumulate, cudaStream_t st) {
  DeviceGuard dg(p.device);
  BpArgs a;
  a.nx = int(p.vol.shape[0]);
  a.ny = int(p.vol.shape[1]);
  a.nb = int(p.det.n_bins);
  a.ox = p.vol.origin[0];
  a.oy = p.vol.origin[1];
  a.sx = p.vol.spacing[0];
  a.sy = p.vol.spacing[1];
  a.det_origin = p.det.origin;
  a.inv_ds = 1.0 / p.det.spacing;
  a.sid = p.sid;
  a.sdd = p.sdd;
  a.fan = p.fan;
  a.sino = d_sino;
  a.img = d_img;
  dim3 grid((a.nx + 31) / 32, (a.ny + 7) / 8);
  KernelTimer timer;
  timer.start(st);
  for (uint64_t c0 = 0; c0 < p.n_proj; c0 += kMaxConstViews) {
    const uint64_t cn = std::min<uint64_t>(kMaxConstViews, p.n_proj - c0);
    a.n_views = int(cn);
    a.view_base = int(c0);
    a.scale = scale;
    a.accumulate = c0 == 0 ? accumulate : 1;
    std::lock_guard<std::mutex> lk(g_bank.mu);
    g_bank.acquire(p.device, (p.id << 24) ^ c0, st, c_pviews, p.d_coef + c0, cn * sizeof(double2));
    planar_bp_kernel<<<grid, dim3(32, 8), 0, st>>>(a);
    TG_LAUNCHED(1);
    g_bank.release(p.device, st);
  }
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
    std::vector<double2> coef(n);
    for (uint64_t i = 0; i < n; ++i) {
      const double rx = g->rays[2 * i], ry = g->rays[2 * i + 1];
      coef[i] = fan ? make_double2(rx, ry) : make_double2(-ry, rx);
    }
    DeviceGuard dg(device);
    TG_CUDA(cudaMalloc(&p->d_rays, 2 * n * sizeof(double)));
    TG_CUDA(cudaMemcpy(p->d_rays, g->rays, 2 * n * sizeof(double), cudaMemcpyHostToDevice));
    TG_CUDA(cudaMalloc(&p->d_coef, n * sizeof(double2)));
    TG_CUDA(cudaMemcpy(p->d_coef, coef.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
    *out = p.release();
  });
}

tg_status tg_planar_plan_destroy(tg_planar_plan* p) {
  return guarded([&] {
    if (!p) return;
    g_bank.forget(p->id);
    DeviceGuard dg(p->device);
    cudaFree(p->d_rays);
    cudaFree(p->d_coef);
    cudaFree(p->d_ipad);
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
