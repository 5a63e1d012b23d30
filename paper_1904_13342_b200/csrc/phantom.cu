// phantom.cu — GPU rasterisation of additive ellipse / ellipsoid phantoms
// (phantom.hpp:34-88), bit-exact with the reference: FP64 through explicit
// round-to-nearest intrinsics (never contracted), cos/sin of the rotation
// taken on the host with the same libm, and the voxel's float sum formed in
// primitive order.  Used to build synthetic inputs on the device (bench.py,
// SURVEY §8f row 3) without a host round trip.
#include <cmath>
#include <vector>

#include "device_common.cuh"

namespace tgb {
namespace {

#define DADD __dadd_rn
#define DMUL __dmul_rn
#define DDIV __ddiv_rn

struct Prim {
  double cx, cy, cz, a, b, c, cph, sph;
  float intensity;
};

__global__ void ellipsoid_kernel(const Prim* __restrict__ prims, int n_prims, int nx, int ny, int nz,
                                 double ox, double oy, double oz, double sx, double sy, double sz,
                                 float* __restrict__ out) {
  const long long total = (long long)nx * ny * nz;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ix = int(i % nx);
    const long long r = i / nx;
    const int iy = int(r % ny), iz = int(r / ny);
    float acc = 0.0f;
    for (int e = 0; e < n_prims; ++e) {
      const Prim p = prims[e];
      const double dz = DADD(DADD(oz, DMUL(double(iz), sz)), -p.cz);
      const double wz = DDIV(dz, p.c);
      const double rem = DADD(1.0, -DMUL(wz, wz));
      if (rem < 0.0) continue;
      const double dy = DADD(DADD(oy, DMUL(double(iy), sy)), -p.cy);
      const double dx = DADD(DADD(ox, DMUL(double(ix), sx)), -p.cx);
      const double u = DDIV(DADD(DMUL(p.cph, dx), DMUL(p.sph, dy)), p.a);
      const double v = DDIV(DADD(DMUL(-p.sph, dx), DMUL(p.cph, dy)), p.b);
      if (DADD(DMUL(u, u), DMUL(v, v)) <= rem) acc = __fadd_rn(acc, p.intensity);
    }
    out[i] = acc;
  }
}

__global__ void ellipse_kernel(const Prim* __restrict__ prims, int n_prims, int nx, int ny, double ox,
                               double oy, double sx, double sy, float* __restrict__ out) {
  const long long total = (long long)nx * ny;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ix = int(i % nx), iy = int(i / nx);
    float acc = 0.0f;
    for (int e = 0; e < n_prims; ++e) {
      const Prim p = prims[e];
      const double dy = DADD(DADD(oy, DMUL(double(iy), sy)), -p.cy);
      const double dx = DADD(DADD(ox, DMUL(double(ix), sx)), -p.cx);
      const double u = DDIV(DADD(DMUL(p.cph, dx), DMUL(p.sph, dy)), p.a);
      const double v = DDIV(DADD(DMUL(-p.sph, dx), DMUL(p.cph, dy)), p.b);
      if (DADD(DMUL(u, u), DMUL(v, v)) <= 1.0) acc = __fadd_rn(acc, p.intensity);
    }
    out[i] = acc;
  }
}

void upload(const std::vector<Prim>& h, Prim** d, cudaStream_t st) {
  TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(d), h.size() * sizeof(Prim), st));
  TG_CUDA(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(Prim), cudaMemcpyHostToDevice, st));
}

}  // namespace
}  // namespace tgb

using namespace tgb;

extern "C" {

tg_status tg_rasterize_ellipsoids(const tg_volume_spec* vol, const double* specs, uint64_t n,
                                  float* d_out, void* stream) {
  return guarded([&] {
    validate_volume(*vol);
    check(vol->dims == 3, "ellipsoid list needs a 3D volume");
    std::vector<Prim> h(n ? n : 1);
    for (uint64_t e = 0; e < n; ++e) {
      const double* s = specs + 8 * e;
      check(s[3] > 0.0 && s[4] > 0.0 && s[5] > 0.0, "ellipsoid semi-axes must be positive");
      const double phi = s[6] * kPi / 180.0;
      h[e] = Prim{s[0], s[1], s[2], s[3], s[4], s[5], std::cos(phi), std::sin(phi), float(s[7])};
    }
    cudaStream_t st = as_stream(stream);
    Prim* d = nullptr;
    upload(h, &d, st);
    const long long total = (long long)vol->shape[0] * vol->shape[1] * vol->shape[2];
    const int blocks = int(std::min<long long>((total + 255) / 256, 148 * 64));
    ellipsoid_kernel<<<blocks, 256, 0, st>>>(d, int(n), int(vol->shape[0]), int(vol->shape[1]),
                                             int(vol->shape[2]), vol->origin[0], vol->origin[1],
                                             vol->origin[2], vol->spacing[0], vol->spacing[1],
                                             vol->spacing[2], d_out);
    TG_LAUNCHED(1);
    TG_CUDA(cudaFreeAsync(d, st));
  });
}

tg_status tg_rasterize_ellipses(const tg_volume_spec* vol, const double* specs, uint64_t n,
                                float* d_out, void* stream) {
  return guarded([&] {
    validate_volume(*vol);
    check(vol->dims == 2, "ellipse list needs a 2D volume");
    std::vector<Prim> h(n ? n : 1);
    for (uint64_t e = 0; e < n; ++e) {
      const double* s = specs + 6 * e;
      check(s[2] > 0.0 && s[3] > 0.0, "ellipse semi-axes must be positive");
      const double phi = s[4] * kPi / 180.0;
      h[e] = Prim{s[0], s[1], 0.0, s[2], s[3], 1.0, std::cos(phi), std::sin(phi), float(s[5])};
    }
    cudaStream_t st = as_stream(stream);
    Prim* d = nullptr;
    upload(h, &d, st);
    const long long total = (long long)vol->shape[0] * vol->shape[1];
    const int blocks = int(std::min<long long>((total + 255) / 256, 148 * 64));
    ellipse_kernel<<<blocks, 256, 0, st>>>(d, int(n), int(vol->shape[0]), int(vol->shape[1]),
                                           vol->origin[0], vol->origin[1], vol->spacing[0],
                                           vol->spacing[1], d_out);
    TG_LAUNCHED(1);
    TG_CUDA(cudaFreeAsync(d, st));
  });
}

}  // extern "C"
