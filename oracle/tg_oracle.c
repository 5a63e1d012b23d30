/*
 * tg_oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see tg_oracle.h).
 *
 * Plain-C restatement of the reference's host geometry, projectors,
 * filters and FDK/FBP compositions.  Each function names the reference
 * file:line it restates (paths relative to proj/include/tomograd/).  The
 * expression order follows the reference term by term so that, compiled
 * with -ffp-contract=off and no FMA, results are bit-identical to it.
 */
#include "tg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846 /* std::numbers::pi */

static __thread char g_err[256];

const char* or_last_error(void) { return g_err; }

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

void or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n < 1 ? 1 : n);
#else
  (void)n;
#endif
}

static inline double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static inline double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* ---- geometry.hpp ------------------------------------------------------ */

/* geometry.hpp:30-39 */
int or_view_angles(uint64_t n, double range, double* out) {
  if (!(n >= 1)) return fail("need at least one projection");
  if (!(range > 0.0 && range <= 2.0 * OR_PI + 1e-12))
    return fail("angular range must lie in (0, 2*pi]");
  for (uint64_t i = 0; i < n; ++i) out[i] = (double)i * range / (double)n;
  return 0;
}

/* geometry.hpp:42-48 */
int or_circular_rays_2d(uint64_t n, double range, double* out2) {
  double* a = (double*)malloc(sizeof(double) * (n ? n : 1));
  if (or_view_angles(n, range, a)) {
    free(a);
    return 1;
  }
  for (uint64_t i = 0; i < n; ++i) {
    out2[2 * i] = cos(a[i]);
    out2[2 * i + 1] = sin(a[i]);
  }
  free(a);
  return 0;
}

/* geometry.hpp:181-194 */
void or_cone_projection_matrix(double theta, double sid, double sdd, const or_det2* det,
                               double* m) {
  const double fu = sdd / det->spacing_u;
  const double fv = sdd / det->spacing_v;
  const double cu = -det->origin_u / det->spacing_u;
  const double cv = -det->origin_v / det->spacing_v;
  const double ct = cos(theta), st = sin(theta);
  m[0] = -fu * st + cu * ct;
  m[1] = fu * ct + cu * st;
  m[2] = 0.0;
  m[3] = cu * sid;
  m[4] = cv * ct;
  m[5] = cv * st;
  m[6] = fv;
  m[7] = cv * sid;
  m[8] = ct;
  m[9] = st;
  m[10] = 0.0;
  m[11] = sid;
}

/* core.hpp:54-71 Mat33::det / inverse (cofactor form) */
static int mat33_inverse(const double* m, double* r) {
  const double d = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                   m[2] * (m[3] * m[7] - m[4] * m[6]);
  if (!(fabs(d) > 1e-300)) return fail("matrix block is not invertible");
  const double i = 1.0 / d;
  r[0] = (m[4] * m[8] - m[5] * m[7]) * i;
  r[1] = (m[2] * m[7] - m[1] * m[8]) * i;
  r[2] = (m[1] * m[5] - m[2] * m[4]) * i;
  r[3] = (m[5] * m[6] - m[3] * m[8]) * i;
  r[4] = (m[0] * m[8] - m[2] * m[6]) * i;
  r[5] = (m[2] * m[3] - m[0] * m[5]) * i;
  r[6] = (m[3] * m[7] - m[4] * m[6]) * i;
  r[7] = (m[1] * m[6] - m[0] * m[7]) * i;
  r[8] = (m[0] * m[4] - m[1] * m[3]) * i;
  return 0;
}

/* geometry.hpp:144-177 ConeGeometry::set_matrices */
int or_cone_set_matrices(uint64_t n, double sid, const double* mats_in, double* mats,
                         double* sources, double* invs, double* angles) {
  if (mats != mats_in) memcpy(mats, mats_in, sizeof(double) * 12 * n);
  for (uint64_t k = 0; k < n; ++k) {
    double* P = mats + 12 * k;
    /* core.hpp:95-99 mul_point({0,0,0}).z */
    const double iso_depth = P[8] * 0.0 + P[9] * 0.0 + P[10] * 0.0 + P[11];
    if (!(fabs(iso_depth) > 1e-12))
      return fail("projection matrix puts the iso-center at zero depth");
    const double s = sid / iso_depth;
    for (int e = 0; e < 12; ++e) P[e] *= s;
    const double lb[9] = {P[0], P[1], P[2], P[4], P[5], P[6], P[8], P[9], P[10]};
    double* inv = invs + 9 * k;
    if (mat33_inverse(lb, inv)) return 1;
    const double cx = P[3], cy = P[7], cz = P[11];
    /* core.hpp:73-77 Mat33::mul, then -1.0 * v */
    const double mx = inv[0] * cx + inv[1] * cy + inv[2] * cz;
    const double my = inv[3] * cx + inv[4] * cy + inv[5] * cz;
    const double mz = inv[6] * cx + inv[7] * cy + inv[8] * cz;
    sources[3 * k] = -1.0 * mx;
    sources[3 * k + 1] = -1.0 * my;
    sources[3 * k + 2] = -1.0 * mz;
  }
  double prev = 0.0, accum = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double a = atan2(-sources[3 * i + 1], -sources[3 * i]);
    if (i == 0) {
      prev = a;
    } else {
      double d = a - prev;
      while (d < 0.0) d += 2.0 * OR_PI;
      while (d >= 2.0 * OR_PI) d -= 2.0 * OR_PI;
      accum += d;
      prev = a;
    }
    angles[i] = accum;
  }
  return 0;
}

/* geometry.hpp:196-223 projection_matrices_circular + make_cone */
int or_make_cone(const or_det2* det, uint64_t n, double range, double sid, double sdd,
                 double* mats, double* sources, double* invs, double* angles) {
  if (!(sid > 0.0 && sdd > sid)) return fail("cone beam requires 0 < SID < SDD");
  if (or_view_angles(n, range, angles)) return 1;
  for (uint64_t i = 0; i < n; ++i) or_cone_projection_matrix(angles[i], sid, sdd, det, mats + 12 * i);
  double* scratch = (double*)malloc(sizeof(double) * n);
  const int rc = or_cone_set_matrices(n, sid, mats, mats, sources, invs, scratch);
  free(scratch);
  if (rc) return rc;
  return or_view_angles(n, range, angles); /* geometry.hpp:221 */
}

/* ---- projector.hpp helpers --------------------------------------------- */

/* projector.hpp:83-101 detail::clip_ray */
static int clip_ray(const or_volume* vol, const double* o, const double* d, double* t0p,
                    double* t1p) {
  double t0 = -1e300, t1 = 1e300;
  for (uint32_t a = 0; a < vol->dims; ++a) {
    const double lo = vol->origin[a] - vol->spacing[a];
    const double hi = vol->origin[a] + (double)vol->shape[a] * vol->spacing[a];
    if (fabs(d[a]) < 1e-12) {
      if (o[a] <= lo || o[a] >= hi) return 0;
      continue;
    }
    double ta = (lo - o[a]) / d[a];
    double tb = (hi - o[a]) / d[a];
    if (ta > tb) {
      const double t = ta;
      ta = tb;
      tb = t;
    }
    t0 = dmax(t0, ta);
    t1 = dmin(t1, tb);
  }
  *t0p = t0;
  *t1p = t1;
  return t1 > t0;
}

/* projector.hpp:103-107 detail::march_step */
static double march_step(const or_volume* vol) {
  double m = vol->spacing[0];
  for (uint32_t a = 1; a < vol->dims; ++a) m = dmin(m, vol->spacing[a]);
  return 0.5 * m;
}

static uint64_t ray_count(const or_volume* vol, const double* o, const double* d) {
  double t0, t1;
  if (!clip_ray(vol, o, d, &t0, &t1)) return 0;
  return (uint64_t)ceil((t1 - t0) / march_step(vol));
}

/* projector.hpp:264-281 ray setup only: samples per cone ray */
int or_cone_ray_samples(const or_cone* g, uint64_t* out) {
  const uint64_t nu = g->det.n_u, nv = g->det.n_v, pv = nu * nv;
#pragma omp parallel for schedule(static)
  for (uint64_t idx = 0; idx < g->n_proj * pv; ++idx) {
    const uint64_t i = idx / pv, iv = (idx % pv) / nu, iu = idx % nu;
    const double* M = g->invs + 9 * i;
    const double x = (double)iu, y = (double)iv, z = 1.0;
    double d[3] = {M[0] * x + M[1] * y + M[2] * z, M[3] * x + M[4] * y + M[5] * z,
                   M[6] * x + M[7] * y + M[8] * z};
    const double s = 1.0 / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] = s * d[0];
    d[1] = s * d[1];
    d[2] = s * d[2];
    out[idx] = ray_count(&g->vol, g->sources + 3 * i, d);
  }
  return 0;
}

/* projector.hpp:171-184 / 212-230 ray setup only */
int or_planar_ray_samples(const or_planar* g, uint64_t* out) {
  const uint64_t nb = g->det.n_bins;
  const int fan = g->sdd > 0.0;
#pragma omp parallel for schedule(static)
  for (uint64_t idx = 0; idx < g->n_proj * nb; ++idx) {
    const uint64_t i = idx / nb, j = idx % nb;
    const double rx = g->rays[2 * i], ry = g->rays[2 * i + 1];
    const double axx = -ry, axy = rx;
    double o[2], d[2];
    if (!fan) {
      const double s = g->det.origin + (double)j * g->det.spacing;
      o[0] = s * axx;
      o[1] = s * axy;
      d[0] = rx;
      d[1] = ry;
    } else {
      const double ns = -g->sid;
      const double sx = ns * rx, sy = ns * ry;
      const double u = g->det.origin + (double)j * g->det.spacing;
      const double px = sx + g->sdd * rx + u * axx, py = sy + g->sdd * ry + u * axy;
      double dx = px - sx, dy = py - sy;
      const double s = 1.0 / sqrt(dx * dx + dy * dy);
      o[0] = sx;
      o[1] = sy;
      d[0] = s * dx;
      d[1] = s * dy;
    }
    out[idx] = ray_count(&g->vol, o, d);
  }
  return 0;
}

/* ---- filtering.hpp / fft.hpp ------------------------------------------- */

static uint64_t next_pow2(uint64_t n) { /* fft.hpp:17-21 */
  uint64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
static int is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }

uint64_t or_filter_window(uint64_t n_bins) { return next_pow2(2 * n_bins); } /* filtering.hpp:34-37 */

/* fft.hpp:25-58 radix-2, forward unscaled, inverse x 1/n; interleaved re/im */
void or_fft(double* a, uint64_t n, int inverse) {
  if (n == 1) return;
  for (uint64_t i = 1, j = 0; i < n; ++i) {
    uint64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double t = a[2 * i];
      a[2 * i] = a[2 * j];
      a[2 * j] = t;
      t = a[2 * i + 1];
      a[2 * i + 1] = a[2 * j + 1];
      a[2 * j + 1] = t;
    }
  }
  const double sign = inverse ? 1.0 : -1.0;
  for (uint64_t len = 2; len <= n; len <<= 1) {
    const double ang = sign * 2.0 * OR_PI / (double)len;
    const double wr_len = cos(ang), wi_len = sin(ang);
    for (uint64_t i = 0; i < n; i += len) {
      double wr = 1.0, wi = 0.0;
      for (uint64_t k = 0; k < len / 2; ++k) {
        double* pu = a + 2 * (i + k);
        double* pv = a + 2 * (i + k + len / 2);
        const double ur = pu[0], ui = pu[1];
        /* complex<double> product (a*c - b*d, a*d + b*c) */
        const double vr = pv[0] * wr - pv[1] * wi;
        const double vi = pv[0] * wi + pv[1] * wr;
        pu[0] = ur + vr;
        pu[1] = ui + vi;
        pv[0] = ur - vr;
        pv[1] = ui - vi;
        const double nwr = wr * wr_len - wi * wi_len;
        const double nwi = wr * wi_len + wi * wr_len;
        wr = nwr;
        wi = nwi;
      }
    }
  }
  if (inverse) {
    const double inv = 1.0 / (double)n;
    for (uint64_t k = 0; k < 2 * n; ++k) a[k] *= inv;
  }
}

/* filtering.hpp:40-50 */
void or_ramp_weights(uint64_t P, double spacing, double* w) {
  for (uint64_t k = 0; k < P; ++k) w[k] = 0.0;
  for (uint64_t k = 0; k <= P / 2; ++k) {
    const double f = (double)k / ((double)P * spacing);
    w[k] = f;
    if (k != 0) w[P - k] = f;
  }
}

/* filtering.hpp:60-65 */
double or_ramlak_spatial(long m, double spacing) {
  if (m == 0) return 1.0 / (4.0 * spacing * spacing);
  if (m % 2 == 0) return 0.0;
  const double mpi = (double)m * OR_PI * spacing;
  return -1.0 / (mpi * mpi);
}

/* filtering.hpp:68-82 */
void or_ramlak_weights(uint64_t P, double spacing, double* w) {
  double* k = (double*)calloc(2 * P, sizeof(double));
  k[0] = or_ramlak_spatial(0, spacing);
  for (uint64_t m = 1; m <= P / 2; ++m) {
    const double v = or_ramlak_spatial((long)m, spacing);
    k[2 * m] = v;
    k[2 * m + 1] = 0.0;
    k[2 * (P - m)] = v;
    k[2 * (P - m) + 1] = 0.0;
  }
  or_fft(k, P, 0);
  for (uint64_t i = 0; i < P; ++i) w[i] = k[2 * i] * spacing;
  free(k);
}

/* filtering.hpp:157-166 */
void or_cosine_weights_fan(const or_planar* g, double* out) {
  for (uint64_t j = 0; j < g->det.n_bins; ++j) {
    const double u = g->det.origin + (double)j * g->det.spacing;
    out[j] = g->sid / sqrt(g->sid * g->sid + u * u);
  }
}

/* filtering.hpp:168-181 */
void or_cosine_weights_cone(const or_cone* g, double* out) {
  for (uint64_t iv = 0; iv < g->det.n_v; ++iv) {
    const double v = g->det.origin_v + (double)iv * g->det.spacing_v;
    for (uint64_t iu = 0; iu < g->det.n_u; ++iu) {
      const double u = g->det.origin_u + (double)iu * g->det.spacing_u;
      out[iv * g->det.n_u + iu] = g->sid / sqrt(g->sid * g->sid + u * u + v * v);
    }
  }
}

/* filtering.hpp:189-202 */
double or_parker_weight(double beta, double gamma, double delta, double range) {
  const double tiny = 1e-12;
  if (delta - gamma > tiny && beta < 2.0 * (delta - gamma)) {
    const double s = sin(0.25 * OR_PI * beta / (delta - gamma));
    return s * s;
  }
  if (delta + gamma > tiny && beta > range - 2.0 * (delta + gamma)) {
    const double s = sin(0.25 * OR_PI * (range - beta) / (delta + gamma));
    return s * s;
  }
  return 1.0;
}

/* filtering.hpp:204-211 */
static int parker_delta(double range, double fan_half_angle, double* delta) {
  const double eps = 1e-6;
  if (!(range + eps >= OR_PI + 2.0 * fan_half_angle))
    return fail("scan range is too short for redundancy weighting (need pi + fan angle)");
  if (!(range <= 2.0 * OR_PI + eps)) return fail("redundancy weighting expects at most a full turn");
  *delta = 0.5 * (range - OR_PI);
  return 0;
}

/* filtering.hpp:215-230 (fan_half_angle geometry.hpp:103-105) */
int or_parker_weights_fan(const or_planar* g, double* out) {
  double delta;
  const double fha = atan(0.5 * (double)g->det.n_bins * g->det.spacing / g->sdd);
  if (parker_delta(g->range, fha, &delta)) return 1;
  for (uint64_t i = 0; i < g->n_proj; ++i) {
    const double beta = g->angles[i] - g->angles[0];
    for (uint64_t j = 0; j < g->det.n_bins; ++j) {
      const double u = g->det.origin + (double)j * g->det.spacing;
      const double gamma = atan(u / g->sdd);
      out[i * g->det.n_bins + j] = or_parker_weight(beta, gamma, delta, g->range);
    }
  }
  return 0;
}

/* filtering.hpp:234-251 (fan_half_angle geometry.hpp:138-140); one row per view */
int or_parker_weights_cone(const or_cone* g, double* out) {
  double delta;
  const double fha = atan(0.5 * (double)g->det.n_u * g->det.spacing_u / g->sdd);
  if (parker_delta(g->range, fha, &delta)) return 1;
  for (uint64_t i = 0; i < g->n_proj; ++i) {
    const double beta = g->angles[i] - g->angles[0];
    for (uint64_t iu = 0; iu < g->det.n_u; ++iu) {
      const double u = g->det.origin_u + (double)iu * g->det.spacing_u;
      const double gamma = atan(u / g->sdd);
      out[i * g->det.n_u + iu] = or_parker_weight(beta, gamma, delta, g->range);
    }
  }
  return 0;
}

/* ---- phantom.hpp -------------------------------------------------------- */

/* phantom.hpp:108-122 */
void or_head_ellipsoids(double F, double* o) {
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
      {0.06 * F, -0.605 * F, 0.0, 0.0230 * F, 0.0460 * F, 0.020 * F, 0.0, 0.01},
  };
  memcpy(o, t, sizeof t);
}

/* phantom.hpp:91-105 */
void or_head_ellipses(double F, double* o) {
  const double t[10][6] = {
      {0.0, 0.0, 0.6900 * F, 0.9200 * F, 0.0, 1.00},
      {0.0, -0.0184 * F, 0.6624 * F, 0.8740 * F, 0.0, -0.98},
      {0.22 * F, 0.0, 0.1100 * F, 0.3100 * F, -18.0, -0.02},
      {-0.22 * F, 0.0, 0.1600 * F, 0.4100 * F, 18.0, -0.02},
      {0.0, 0.35 * F, 0.2100 * F, 0.2500 * F, 0.0, 0.01},
      {0.0, 0.10 * F, 0.0460 * F, 0.0460 * F, 0.0, 0.01},
      {0.0, -0.10 * F, 0.0460 * F, 0.0460 * F, 0.0, 0.01},
      {-0.08 * F, -0.605 * F, 0.0460 * F, 0.0230 * F, 0.0, 0.01},
      {0.0, -0.606 * F, 0.0230 * F, 0.0230 * F, 0.0, 0.01},
      {0.06 * F, -0.605 * F, 0.0230 * F, 0.0460 * F, 0.0, 0.01},
  };
  memcpy(o, t, sizeof t);
}

/* phantom.hpp:124-128 */
double or_fov_half_extent(const or_volume* vol) {
  double h = (double)vol->shape[0] * vol->spacing[0];
  for (uint32_t a = 1; a < vol->dims; ++a) h = dmin(h, (double)vol->shape[a] * vol->spacing[a]);
  return 0.5 * h;
}

/* ---- pipelines.hpp:90-115 GaussianSource: std::mt19937_64 + Box-Muller --- */

/* std::mt19937_64 (the C++ standard's parameters: w=64, n=312, m=156, r=31,
 * a=0xB5026F5AA96619E9, u=29, d=0x5555555555555555, s=17, b=0x71D67FFFEDA60000,
 * t=37, c=0xFFF7EEE000000000, l=43, f=6364136223846793005) */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64;

static void mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(or_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

typedef struct {
  or_mt64 rng;
  int have;
  double cached;
} or_gauss;

static double gauss_next(or_gauss* g) {
  if (g->have) {
    g->have = 0;
    return g->cached;
  }
  const double u1 = ((double)(mt64_next(&g->rng) >> 11) + 1.0) * 0x1.0p-53; /* (0, 1] */
  const double u2 = (double)(mt64_next(&g->rng) >> 11) * 0x1.0p-53;         /* [0, 1) */
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * OR_PI * u2;
  g->cached = r * sin(a);
  g->have = 1;
  return r * cos(a);
}

uint64_t or_mt19937_64_first(uint64_t seed, uint64_t k) {
  or_mt64 g;
  mt64_seed(&g, seed);
  uint64_t v = 0;
  for (uint64_t i = 0; i < k; ++i) v = mt64_next(&g);
  return v;
}

/* ---- storage-typed operators (instantiated for float and double) ------- */

#define T float
#define SUF f32
#include "tg_oracle_body.inc"
#undef T
#undef SUF

#define T double
#define SUF f64
#include "tg_oracle_body.inc"
#undef T
#undef SUF
