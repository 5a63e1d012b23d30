/*
 * tg_oracle.h — CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * A plain-C restatement of the reference toolkit's projector / FDK path
 * (tomograd, /root/reference/proj/include/tomograd/*.hpp), used ONLY by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker.  The product (paper_1904_13342_b200/, libtomograd_b200.so) never
 * links, loads or calls anything here.
 *
 * Parity pinning: every function is checked bit-for-bit against the
 * reference itself, compiled from its own headers into oracle/_ref/
 * (oracle/Makefile, oracle/ref_capi.cpp), and against the reference test
 * suites' known answers (tests/test_oracle_*.py) and committed golden
 * fixtures (tests/golden/).
 *
 * Arithmetic: double precision throughout, storage type T = float ("_f32")
 * or double ("_f64"), the same split the reference's templates make.  The
 * file is compiled with -ffp-contract=off and no -march, like the
 * reference's Release build (proj/CMakeLists.txt:3-8), so the restatement
 * is bit-identical to the reference on x86-64.
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* image.hpp:18-54 VolumeSpec (dims 2 or 3; x fastest) */
typedef struct {
  uint32_t dims;
  uint64_t shape[3];
  double spacing[3];
  double origin[3];
} or_volume;

/* image.hpp:57-67 Detector1D */
typedef struct {
  uint64_t n_bins;
  double spacing, origin;
} or_det1;

/* image.hpp:70-81 Detector2D */
typedef struct {
  uint64_t n_u, n_v;
  double spacing_u, spacing_v, origin_u, origin_v;
} or_det2;

/* geometry.hpp:50-124: parallel (sid = sdd = 0) or fan beam */
typedef struct {
  or_volume vol;
  or_det1 det;
  uint64_t n_proj;
  double range, sid, sdd;
  const double* rays; /* n_proj x 2 */
  const double* angles;
} or_planar;

/* geometry.hpp:126-178 ConeGeometry */
typedef struct {
  or_volume vol;
  or_det2 det;
  uint64_t n_proj;
  double range, sid, sdd;
  const double* mats;    /* n x 12, normalised */
  const double* sources; /* n x 3 */
  const double* invs;    /* n x 9 */
  const double* angles;  /* n */
} or_cone;

/* returns 0 on success, nonzero on a reference check() failure; the
 * message (the reference's exact text) is in or_last_error(). */
const char* or_last_error(void);
void or_set_threads(int n);

/* geometry.hpp */
int or_view_angles(uint64_t n, double range, double* out);
int or_circular_rays_2d(uint64_t n, double range, double* out2);
void or_cone_projection_matrix(double theta, double sid, double sdd, const or_det2* det,
                               double* out12);
int or_cone_set_matrices(uint64_t n, double sid, const double* mats_in, double* mats_out,
                         double* sources, double* invs, double* angles);
int or_make_cone(const or_det2* det, uint64_t n, double range, double sid, double sdd,
                 double* mats, double* sources, double* invs, double* angles);

/* projector.hpp — T = float / double storage */
#define OR_DECLARE(SUF, T)                                                                  \
  int or_parallel_forward_##SUF(const or_planar* g, const T* img, T* sino);                \
  int or_parallel_backproject_##SUF(const or_planar* g, const T* sino, T* img);            \
  int or_fan_forward_##SUF(const or_planar* g, const T* img, T* sino);                     \
  int or_fan_backproject_##SUF(const or_planar* g, const T* sino, T* img);                 \
  int or_cone_forward_##SUF(const or_cone* g, const T* vol, T* sino);                      \
  int or_cone_backproject_##SUF(const or_cone* g, const T* sino, T* vol);                  \
  int or_apply_filter_##SUF(T* data, uint64_t n_rows, uint64_t n, const double* weights,   \
                            uint64_t padded_n);                                             \
  void or_apply_weights_##SUF(T* data, uint64_t n_total, const double* map, uint64_t map_n);\
  int or_fdk_reconstruct_##SUF(const or_cone* g, const T* sino, T* vol, int use_parker);   \
  int or_fbp_reconstruct_##SUF(const or_planar* g, const T* sino, T* img,                  \
                               const double* weights, uint64_t padded_n);                   \
  int or_rasterize_ellipsoids_##SUF(const or_volume* vol, const double* specs, uint64_t n, \
                                    T* out);                                                \
  int or_rasterize_ellipses_##SUF(const or_volume* vol, const double* specs, uint64_t n,   \
                                  T* out);
#define OR_DECLARE_ITER(SUF, T)                                                             \
  double or_l2_value_##SUF(const T* a, const T* b, uint64_t n);                             \
  double or_tv_value_##SUF(const T* x, const uint64_t* shape, uint32_t dims);               \
  void or_tv_subgrad_acc_##SUF(const T* x, const uint64_t* shape, uint32_t dims, double gs,  \
                               double* gx);                                                  \
  int or_tv_reconstruct_cone_##SUF(const or_cone* g, const T* sino, T* x, uint64_t iters,    \
                                   double lr, double lambda, double* hist);                  \
  int or_tv_reconstruct_planar_##SUF(const or_planar* g, const T* sino, T* x,              \
                                     uint64_t iters, double lr, double lambda, double* hist); \
  int or_add_gaussian_noise_##SUF(const T* in, T* out, uint64_t n, double relative_std,     \
                                  uint64_t seed);                                              \
  int or_learn_filter_planar_##SUF(const or_planar* g, const T* sino, uint64_t P, double lr,  \
                                   uint64_t iterations, double* loss_h, double* dist_h,       \
                                   double* w_out, T* recon_out);
OR_DECLARE_ITER(f32, float)
OR_DECLARE_ITER(f64, double)
#undef OR_DECLARE_ITER
/* k-th output (1-based) of std::mt19937_64(seed) */
uint64_t or_mt19937_64_first(uint64_t seed, uint64_t k);

OR_DECLARE(f32, float)
OR_DECLARE(f64, double)
#undef OR_DECLARE

/* per-ray sample counts n = ceil((t1 - t0) / step) (0 for a miss) */
int or_cone_ray_samples(const or_cone* g, uint64_t* out);
int or_planar_ray_samples(const or_planar* g, uint64_t* out);

/* filtering.hpp / fft.hpp */
uint64_t or_filter_window(uint64_t n_bins);
void or_ramp_weights(uint64_t padded_n, double spacing, double* out);
double or_ramlak_spatial(long m, double spacing);
void or_ramlak_weights(uint64_t padded_n, double spacing, double* out);
void or_fft(double* re_im, uint64_t n, int inverse);
void or_cosine_weights_fan(const or_planar* g, double* out);
void or_cosine_weights_cone(const or_cone* g, double* out);
double or_parker_weight(double beta, double gamma, double delta, double range);
int or_parker_weights_fan(const or_planar* g, double* out);  /* n_proj x n_bins */
int or_parker_weights_cone(const or_cone* g, double* out);   /* n_proj x n_u (row-repeated) */

/* phantom.hpp: tables of 8 doubles {cx,cy,cz,a,b,c,phi_deg,intensity} / 6 for ellipses */
void or_head_ellipsoids(double fov_half, double* out80);
void or_head_ellipses(double fov_half, double* out60);
double or_fov_half_extent(const or_volume* vol);

#ifdef __cplusplus
}
#endif
#endif
