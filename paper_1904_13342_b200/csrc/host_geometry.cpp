// host_geometry.cpp — host-side geometry, weight and filter precompute.
//
// Written from scratch against the reference's documented behaviour and
// required to be BIT-EXACT with it: every expression keeps the
// reference's operation order, and the file is compiled with
// -ffp-contract=off and no -march (no FMA), exactly like the reference's
// Release build.  tests/test_host_geometry.py checks each entry point
// bitwise against the oracle and the compiled reference.
#include <cmath>
#include <complex>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "tg_internal.h"

namespace tgb {

namespace {
thread_local std::string t_last_error;
}

void set_last_error(const std::string& msg) { t_last_error = msg; }

bool is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }

uint64_t next_pow2(uint64_t n) {  // fft.hpp:17-21
  uint64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// image.hpp:213-223 VolumeSpec::validate
void validate_volume(const tg_volume_spec& v) {
  check(v.dims == 2 || v.dims == 3, "volume must be 2D or 3D");
  for (uint32_t a = 0; a < v.dims; ++a) check(v.shape[a] >= 1, "volume shape entries must be >= 1");
  for (uint32_t a = 0; a < v.dims; ++a) check(v.spacing[a] > 0.0, "volume spacing must be positive");
}

// geometry.hpp:30-39
void view_angles(uint64_t n, double range, double* out) {
  check(n >= 1, "need at least one projection");
  check(range > 0.0 && range <= 2.0 * kPi + 1e-12, "angular range must lie in (0, 2*pi]");
  for (uint64_t i = 0; i < n; ++i) out[i] = double(i) * range / double(n);
}

// geometry.hpp:181-194: rows (u axis, v axis, principal ray), t = (0, 0, SID)
void cone_projection_matrix(double theta, double sid, double sdd, const tg_detector2d& det,
                            double* m) {
  const double fu = sdd / det.spacing_u, fv = sdd / det.spacing_v;
  const double cu = -det.origin_u / det.spacing_u, cv = -det.origin_v / det.spacing_v;
  const double c = std::cos(theta), s = std::sin(theta);
  const double row[12] = {-fu * s + cu * c, fu * c + cu * s, 0.0, cu * sid,
                          cv * c,           cv * s,          fv,  cv * sid,
                          c,                s,               0.0, sid};
  std::memcpy(m, row, sizeof row);
}

namespace {

// core.hpp:60-71: cofactor inverse of a row-major 3x3 block
void inverse3(const double a[9], double r[9]) {
  const double c00 = a[4] * a[8] - a[5] * a[7];
  const double c01 = a[3] * a[8] - a[5] * a[6];
  const double c02 = a[3] * a[7] - a[4] * a[6];
  const double det = a[0] * c00 - a[1] * c01 + a[2] * c02;
  check(std::abs(det) > 1e-300, "matrix block is not invertible");
  const double k = 1.0 / det;
  r[0] = c00 * k;
  r[1] = (a[2] * a[7] - a[1] * a[8]) * k;
  r[2] = (a[1] * a[5] - a[2] * a[4]) * k;
  r[3] = (a[5] * a[6] - a[3] * a[8]) * k;
  r[4] = (a[0] * a[8] - a[2] * a[6]) * k;
  r[5] = (a[2] * a[3] - a[0] * a[5]) * k;
  r[6] = c02 * k;
  r[7] = (a[1] * a[6] - a[0] * a[7]) * k;
  r[8] = (a[0] * a[4] - a[1] * a[3]) * k;
}

}  // namespace

// geometry.hpp:144-177 ConeGeometry::set_matrices
void cone_set_matrices(uint64_t n, double sid, const double* in, double* mats, double* sources,
                       double* invs, double* angles) {
  if (mats != in) std::memmove(mats, in, sizeof(double) * 12 * n);
  for (uint64_t v = 0; v < n; ++v) {
    double* P = mats + 12 * v;
    // homogeneous depth of the iso-centre: P * (0,0,0,1), z row
    const double depth = P[8] * 0.0 + P[9] * 0.0 + P[10] * 0.0 + P[11];
    check(std::abs(depth) > 1e-12, "projection matrix puts the iso-center at zero depth");
    const double s = sid / depth;
    for (int e = 0; e < 12; ++e) P[e] *= s;
    const double block[9] = {P[0], P[1], P[2], P[4], P[5], P[6], P[8], P[9], P[10]};
    double* M = invs + 9 * v;
    inverse3(block, M);
    // source = -(M * p4)
    for (int r = 0; r < 3; ++r)
      sources[3 * v + r] = -1.0 * (M[3 * r] * P[3] + M[3 * r + 1] * P[7] + M[3 * r + 2] * P[11]);
  }
  // unwrapped source angles, measured from the first view
  const double two_pi = 2.0 * kPi;
  double last = 0.0, total = 0.0;
  for (uint64_t v = 0; v < n; ++v) {
    const double a = std::atan2(-sources[3 * v + 1], -sources[3 * v]);
    if (v > 0) {
      double step = a - last;
      while (step < 0.0) step += two_pi;
      while (step >= two_pi) step -= two_pi;
      total += step;
    }
    last = a;
    angles[v] = total;
  }
}

double cone_fan_half_angle(const tg_cone_geometry& g) {  // geometry.hpp:138-140
  return std::atan(0.5 * double(g.detector.n_u) * g.detector.spacing_u / g.sdd);
}

double planar_fan_half_angle(const tg_planar_geometry& g) {  // geometry.hpp:103-105
  return std::atan(0.5 * double(g.detector.n_bins) * g.detector.spacing / g.sdd);
}

// filtering.hpp:204-211
double parker_delta(double range, double fan_half_angle) {
  const double eps = 1e-6;
  check(range + eps >= kPi + 2.0 * fan_half_angle,
        "scan range is too short for redundancy weighting (need pi + fan angle)");
  check(range <= 2.0 * kPi + eps, "redundancy weighting expects at most a full turn");
  return 0.5 * (range - kPi);
}

// filtering.hpp:189-202: sin^2 ramps over the doubly measured wedges
double parker_weight(double beta, double gamma, double delta, double range) {
  const double tiny = 1e-12;
  const double lo = delta - gamma, hi = delta + gamma;
  if (lo > tiny && beta < 2.0 * lo) {
    const double s = std::sin(0.25 * kPi * beta / lo);
    return s * s;
  }
  if (hi > tiny && beta > range - 2.0 * hi) {
    const double s = std::sin(0.25 * kPi * (range - beta) / hi);
    return s * s;
  }
  return 1.0;
}

// filtering.hpp:168-181
void cosine_weights_cone(const tg_cone_geometry& g, double* out) {
  const tg_detector2d& d = g.detector;
  const double sid2 = g.sid * g.sid;
  for (uint64_t iv = 0; iv < d.n_v; ++iv) {
    const double v = d.origin_v + double(iv) * d.spacing_v;
    for (uint64_t iu = 0; iu < d.n_u; ++iu) {
      const double u = d.origin_u + double(iu) * d.spacing_u;
      out[iv * d.n_u + iu] = g.sid / std::sqrt(sid2 + u * u + v * v);
    }
  }
}

// filtering.hpp:234-251, compact: one u-profile per view
void parker_weights_cone(const tg_cone_geometry& g, double* out) {
  const double delta = parker_delta(g.angular_range, cone_fan_half_angle(g));
  const tg_detector2d& d = g.detector;
  std::vector<double> gamma(d.n_u);
  for (uint64_t iu = 0; iu < d.n_u; ++iu)
    gamma[iu] = std::atan((d.origin_u + double(iu) * d.spacing_u) / g.sdd);
  for (uint64_t i = 0; i < g.n_projections; ++i) {
    const double beta = g.angles[i] - g.angles[0];
    for (uint64_t iu = 0; iu < d.n_u; ++iu)
      out[i * d.n_u + iu] = parker_weight(beta, gamma[iu], delta, g.angular_range);
  }
}

namespace {

// fft.hpp:25-58 semantics (radix-2, forward unscaled); used only for the
// Ram-Lak weight vector, so it follows the reference's twiddle recurrence
// to stay bit-exact.
void fft_forward(std::vector<std::complex<double>>& a) {
  const uint64_t n = a.size();
  if (n == 1) return;
  for (uint64_t i = 1, j = 0; i < n; ++i) {
    uint64_t bit = n >> 1;
    while (j & bit) {
      j ^= bit;
      bit >>= 1;
    }
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (uint64_t len = 2; len <= n; len <<= 1) {
    const double ang = -1.0 * 2.0 * kPi / double(len);
    const std::complex<double> step(std::cos(ang), std::sin(ang));
    const uint64_t half = len / 2;
    for (uint64_t base = 0; base < n; base += len) {
      std::complex<double> w(1.0, 0.0);
      for (uint64_t k = 0; k < half; ++k) {
        const std::complex<double> x = a[base + k];
        const std::complex<double> y = a[base + k + half] * w;
        a[base + k] = x + y;
        a[base + k + half] = x - y;
        w *= step;
      }
    }
  }
}

double ramlak_tap(long m, double spacing) {  // filtering.hpp:60-65
  if (m == 0) return 1.0 / (4.0 * spacing * spacing);
  if (m % 2 == 0) return 0.0;
  const double q = double(m) * kPi * spacing;
  return -1.0 / (q * q);
}

}  // namespace

// filtering.hpp:68-82: spacing * Re(DFT(wrapped spatial kernel))
void ramlak_weights(uint64_t P, double spacing, double* out) {
  check(is_pow2(P), "filter window must be a power of two");
  check(spacing > 0.0, "detector spacing must be positive");
  std::vector<std::complex<double>> k(P, 0.0);
  k[0] = ramlak_tap(0, spacing);
  for (uint64_t m = 1; m <= P / 2; ++m) {
    const double t = ramlak_tap(long(m), spacing);
    k[m] = t;
    k[P - m] = t;
  }
  fft_forward(k);
  for (uint64_t i = 0; i < P; ++i) out[i] = k[i].real() * spacing;
}

// phantom.hpp:91-122 (unit-disk tables scaled by F)
void head_ellipsoids(double F, double* o) {
  const double t[10][8] = {
      {0.0, 0.0, 0.0, 0.6900 * F, 0.9200 * F, 0.810 * F, 0.0, 1.00},
      {0.0, -0.0184 * F, 0.0, 0.6624 * F, 0.8740 * F, 0.780 * F, 0.0, -0.98},
      {0.22 * F, 0.0, 0.0, 0.1100 * F, 0.3100 * F, 0.220 * F, -18.0, -0.02},
      {-0.22 * F, 0.0, 0.0, 0.1600 * F, 0.4100 * F, 0.280 * F, 18.0, -0.02},
      {0.0, 0.35 * F, -0.15 * F, 0.2100 * F, 0.2500 * F, 0.410 * F, 0.0, 0.01},
      {0.0, 0.10 * F, 0.25 * F, 0.0460 * F, 0.0460 * F, 0.050 * F, 0.0, 0.01},
      {0.0, -0.10 * F, 0.25 * F, 0.0460 * F, 0.0460 * F, 0.050 * F, 0.0, 0.01},
      {-0.08 * F, -0.605 * F, 0.0, 0.0460 * F, 0.0230 * F, 0.050 * F, 0.0, 0.01},
      {0.0, -0.606 * F, 0.0, 0.0230 * F, 0.0230 * F, 0.020 * F, 0.0, 0.01},
      {0.06 * F, -0.605 * F, 0.0, 0.0230 * F, 0.0460 * F, 0.020 * F, 0.0, 0.01}};
  std::memcpy(o, t, sizeof t);
}

void head_ellipses(double F, double* o) {
  const double t[10][6] = {{0.0, 0.0, 0.6900 * F, 0.9200 * F, 0.0, 1.00},
                           {0.0, -0.0184 * F, 0.6624 * F, 0.8740 * F, 0.0, -0.98},
                           {0.22 * F, 0.0, 0.1100 * F, 0.3100 * F, -18.0, -0.02},
                           {-0.22 * F, 0.0, 0.1600 * F, 0.4100 * F, 18.0, -0.02},
                           {0.0, 0.35 * F, 0.2100 * F, 0.2500 * F, 0.0, 0.01},
                           {0.0, 0.10 * F, 0.0460 * F, 0.0460 * F, 0.0, 0.01},
                           {0.0, -0.10 * F, 0.0460 * F, 0.0460 * F, 0.0, 0.01},
                           {-0.08 * F, -0.605 * F, 0.0460 * F, 0.0230 * F, 0.0, 0.01},
                           {0.0, -0.606 * F, 0.0230 * F, 0.0230 * F, 0.0, 0.01},
                           {0.06 * F, -0.605 * F, 0.0230 * F, 0.0460 * F, 0.0, 0.01}};
  std::memcpy(o, t, sizeof t);
}

double fov_half_extent(const tg_volume_spec& v) {  // phantom.hpp:124-128
  double h = double(v.shape[0]) * v.spacing[0];
  for (uint32_t a = 1; a < v.dims; ++a) {
    const double e = double(v.shape[a]) * v.spacing[a];
    if (e < h) h = e;
  }
  return 0.5 * h;
}

}  // namespace tgb

// ---------------------------------------------------------------------------
// C ABI: host geometry entry points

using namespace tgb;

namespace tgb {
namespace {
// pipelines.hpp:90-115 GaussianSource: Box-Muller on explicit mt19937_64 draws
class GaussianSource {
 public:
  explicit GaussianSource(uint64_t seed) : rng_(seed) {}
  double next() {
    if (have_) {
      have_ = false;
      return cached_;
    }
    const double u1 = (double(rng_() >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = double(rng_() >> 11) * 0x1.0p-53;          // [0, 1)
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * kPi * u2;
    cached_ = r * std::sin(a);
    have_ = true;
    return r * std::cos(a);
  }

 private:
  std::mt19937_64 rng_;
  bool have_ = false;
  double cached_ = 0.0;
};
}  // namespace
}  // namespace tgb

extern "C" {

tg_status tg_add_gaussian_noise(const float* in, float* out, uint64_t n, double relative_std,
                                uint64_t seed) {
  return tgb::guarded([&] {
    // pipelines.hpp:119-132
    tgb::check(relative_std >= 0.0, "noise level must be non-negative");
    if (relative_std == 0.0) {
      if (out != in) std::memmove(out, in, n * sizeof(float));
      return;
    }
    double peak = 0.0;
    for (uint64_t i = 0; i < n; ++i) peak = (peak < double(in[i])) ? double(in[i]) : peak;
    const double sigma = relative_std * peak;
    tgb::GaussianSource gauss(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = float(double(in[i]) + sigma * gauss.next());
  });
}

const char* tg_last_error(void) { return tgb::t_last_error.c_str(); }
int tg_abi_version(void) { return TG_ABI_VERSION; }

tg_status tg_view_angles(uint64_t n, double range, double* out) {
  return guarded([&] { view_angles(n, range, out); });
}

tg_status tg_make_planar(const tg_volume_spec* vol, const tg_detector1d* det, uint64_t n,
                         double range, double sid, double sdd, double* rays, double* angles) {
  return guarded([&] {
    validate_volume(*vol);
    const bool fan = sdd != 0.0 || sid != 0.0;
    check(vol->dims == 2, fan ? "fan beam geometry expects a 2D volume"
                              : "parallel beam geometry expects a 2D volume");
    if (fan) check(sid > 0.0 && sdd > sid, "fan beam requires 0 < SID < SDD");
    (void)det;
    view_angles(n, range, angles);
    for (uint64_t i = 0; i < n; ++i) {  // geometry.hpp:42-48
      rays[2 * i] = std::cos(angles[i]);
      rays[2 * i + 1] = std::sin(angles[i]);
    }
  });
}

tg_status tg_cone_projection_matrix(double theta, double sid, double sdd, const tg_detector2d* det,
                                    double* out12) {
  return guarded([&] { cone_projection_matrix(theta, sid, sdd, *det, out12); });
}

tg_status tg_make_cone(const tg_volume_spec* vol, const tg_detector2d* det, uint64_t n,
                       double range, double sid, double sdd, double* mats, double* sources,
                       double* invs, double* angles) {
  return guarded([&] {
    validate_volume(*vol);
    check(vol->dims == 3, "cone beam geometry expects a 3D volume");
    check(sid > 0.0 && sdd > sid, "cone beam requires 0 < SID < SDD");
    view_angles(n, range, angles);
    for (uint64_t i = 0; i < n; ++i) cone_projection_matrix(angles[i], sid, sdd, *det, mats + 12 * i);
    std::vector<double> scratch(n);
    cone_set_matrices(n, sid, mats, mats, sources, invs, scratch.data());
    view_angles(n, range, angles);  // geometry.hpp:221 keeps the nominal schedule
  });
}

tg_status tg_cone_set_matrices(uint64_t n, double sid, const double* in, double* mats,
                               double* sources, double* invs, double* angles) {
  return guarded([&] {
    check(n >= 1, "need at least one projection matrix");
    cone_set_matrices(n, sid, in, mats, sources, invs, angles);
  });
}

uint64_t tg_filter_window(uint64_t n_bins) { return next_pow2(2 * n_bins); }

tg_status tg_ramp_weights(uint64_t P, double spacing, double* w) {
  return guarded([&] {  // filtering.hpp:40-50
    check(is_pow2(P), "filter window must be a power of two");
    check(spacing > 0.0, "detector spacing must be positive");
    for (uint64_t k = 0; k < P; ++k) w[k] = 0.0;
    for (uint64_t k = 0; k <= P / 2; ++k) {
      const double f = double(k) / (double(P) * spacing);
      w[k] = f;
      if (k != 0) w[P - k] = f;
    }
  });
}

tg_status tg_ramlak_weights(uint64_t P, double spacing, double* out) {
  return guarded([&] { ramlak_weights(P, spacing, out); });
}

tg_status tg_cosine_weights_fan(const tg_planar_geometry* g, double* out) {
  return guarded([&] {  // filtering.hpp:157-166
    for (uint64_t j = 0; j < g->detector.n_bins; ++j) {
      const double u = g->detector.origin + double(j) * g->detector.spacing;
      out[j] = g->sid / std::sqrt(g->sid * g->sid + u * u);
    }
  });
}

tg_status tg_cosine_weights_cone(const tg_cone_geometry* g, double* out) {
  return guarded([&] { cosine_weights_cone(*g, out); });
}

tg_status tg_parker_weights_fan(const tg_planar_geometry* g, double* out) {
  return guarded([&] {  // filtering.hpp:215-230
    const double delta = parker_delta(g->angular_range, planar_fan_half_angle(*g));
    const uint64_t nb = g->detector.n_bins;
    for (uint64_t i = 0; i < g->n_projections; ++i) {
      const double beta = g->angles[i] - g->angles[0];
      for (uint64_t j = 0; j < nb; ++j) {
        const double gamma = std::atan((g->detector.origin + double(j) * g->detector.spacing) / g->sdd);
        out[i * nb + j] = parker_weight(beta, gamma, delta, g->angular_range);
      }
    }
  });
}

tg_status tg_parker_weights_cone(const tg_cone_geometry* g, double* out) {
  return guarded([&] { parker_weights_cone(*g, out); });
}

tg_status tg_head_phantom_ellipsoids(const tg_volume_spec* vol, double* out80) {
  return guarded([&] {
    check(vol->dims == 3, "3D head phantom needs a 3D volume");
    head_ellipsoids(fov_half_extent(*vol), out80);
  });
}

tg_status tg_head_phantom_ellipses(const tg_volume_spec* vol, double* out60) {
  return guarded([&] {
    check(vol->dims == 2, "2D head phantom needs a 2D volume");
    head_ellipses(fov_half_extent(*vol), out60);
  });
}

}  // extern "C"
