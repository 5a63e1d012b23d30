/*
 * tomograd_b200.h — C ABI of the B200-native projector / FDK path.
 *
 * This is the drop-in boundary for the reference toolkit's hot path
 * (tomograd, header-only C++20 CPU; paths below are relative to
 * proj/include/tomograd/ of the reference).  Every entry point names the
 * reference interface it replaces.  Plain C types only: POD structs,
 * pointers and sizes; no torch or C++ types cross it.
 *
 * Conventions
 *  - Layouts are the reference's (image.hpp:5-8, 150-163): volumes x-fastest
 *    data[(iz*ny+iy)*nx+ix]; cone sinograms [view][v][u]; planar sinograms
 *    [view][bin].  Device data is float32 (the reference's T = float).
 *  - "d_" pointers are caller-owned device memory on the plan's device,
 *    "h_" pointers host memory (pinned memory gets the fast DMA path).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Errors: every call returns tg_status; on failure tg_last_error() (thread
 *    local) returns the message.  Where the reference throws tomograd::Error
 *    the message is the reference's exact text, so a C++ shim can rethrow it
 *    unchanged (see include/tomograd_b200/projector.hpp).
 *  - Results are deterministic run to run: one writer per output element,
 *    no floating-point atomics.
 *  - Plans hold geometry (device constant / global memory) and scratch; calls
 *    do not allocate except the *_host convenience variants' staging buffers.
 *    Calls on distinct plans are thread-safe.
 */
#ifndef TOMOGRAD_B200_H
#define TOMOGRAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 1

typedef int32_t tg_status;
#define TG_OK 0
#define TG_ERROR 1          /* a reference check() failure; message in tg_last_error() */
#define TG_ERROR_CUDA 2     /* CUDA runtime / driver failure */
#define TG_ERROR_NO_DEVICE 3

/* ---- plain-data mirrors of the reference containers ------------------- */

/* image.hpp:18-54 VolumeSpec; dims = 2 (nx, ny) or 3 (nx, ny, nz) */
typedef struct tg_volume_spec {
  uint32_t dims;
  uint64_t shape[3];
  double spacing[3];
  double origin[3]; /* world position of the first element centre */
} tg_volume_spec;

/* image.hpp:57-67 Detector1D */
typedef struct tg_detector1d {
  uint64_t n_bins;
  double spacing;
  double origin;
} tg_detector1d;

/* image.hpp:70-81 Detector2D (u = columns, fastest) */
typedef struct tg_detector2d {
  uint64_t n_u, n_v;
  double spacing_u, spacing_v;
  double origin_u, origin_v;
} tg_detector2d;

/* geometry.hpp:50-71 ParallelGeometry (sid = sdd = 0) and
 * geometry.hpp:88-106 FanGeometry (0 < sid < sdd) */
typedef struct tg_planar_geometry {
  tg_volume_spec volume; /* 2D */
  tg_detector1d detector;
  uint64_t n_projections;
  double angular_range;
  double sid, sdd;
  const double* rays;   /* n_projections x 2: unit (cos t, sin t) per view */
  const double* angles; /* n_projections */
} tg_planar_geometry;

/* geometry.hpp:126-178 ConeGeometry, matrices already normalised by
 * set_matrices (iso-centre depth == SID) */
typedef struct tg_cone_geometry {
  tg_volume_spec volume; /* 3D */
  tg_detector2d detector;
  uint64_t n_projections;
  double angular_range;
  double sid, sdd;
  const double* matrices;   /* n x 12, row-major P = K[R|t] */
  const double* sources;    /* n x 3 */
  const double* inv_blocks; /* n x 9, inverse of P's left 3x3 block */
  const double* angles;     /* n, measured from the first view */
} tg_cone_geometry;

const char* tg_last_error(void);
int tg_abi_version(void);

/* ---- host geometry: bit-exact with the reference (double maths) -------- */

/* geometry.hpp:30-39 view_angles */
tg_status tg_view_angles(uint64_t n, double angular_range, double* out);
/* geometry.hpp:73-86 make_parallel / 108-124 make_fan: rays and angles
 * (sdd == 0 selects parallel beam) incl. the reference's argument checks */
tg_status tg_make_planar(const tg_volume_spec* vol, const tg_detector1d* det, uint64_t n,
                         double angular_range, double sid, double sdd, double* rays_out,
                         double* angles_out);
/* geometry.hpp:181-194 cone_projection_matrix */
tg_status tg_cone_projection_matrix(double theta, double sid, double sdd,
                                    const tg_detector2d* det, double* out12);
/* geometry.hpp:206-223 make_cone */
tg_status tg_make_cone(const tg_volume_spec* vol, const tg_detector2d* det, uint64_t n,
                       double angular_range, double sid, double sdd, double* matrices,
                       double* sources, double* inv_blocks, double* angles);
/* geometry.hpp:144-177 ConeGeometry::set_matrices (make_cone_from_matrices
 * geometry.hpp:226-242); matrices_in may alias matrices_out */
tg_status tg_cone_set_matrices(uint64_t n, double sid, const double* matrices_in,
                               double* matrices_out, double* sources, double* inv_blocks,
                               double* angles);
/* filtering.hpp:34-37 filter_window */
uint64_t tg_filter_window(uint64_t n_bins);
/* filtering.hpp:40-50 ramp_weights, 68-82 ramlak_weights (length padded_n) */
tg_status tg_ramp_weights(uint64_t padded_n, double spacing, double* out);
tg_status tg_ramlak_weights(uint64_t padded_n, double spacing, double* out);
/* filtering.hpp:157-181 cosine_weights: fan -> [n_bins], cone -> [n_v][n_u] */
tg_status tg_cosine_weights_fan(const tg_planar_geometry* g, double* out);
tg_status tg_cosine_weights_cone(const tg_cone_geometry* g, double* out);
/* filtering.hpp:215-251 parker_weights: fan -> [n_proj][n_bins]; cone ->
 * [n_proj][n_u] (the reference repeats each row over v) */
tg_status tg_parker_weights_fan(const tg_planar_geometry* g, double* out);
tg_status tg_parker_weights_cone(const tg_cone_geometry* g, double* out);

/* ---- cone beam (K1 back-projection, K2 forward projection, K3 FDK) ----- */

typedef struct tg_cone_plan tg_cone_plan;

tg_status tg_cone_plan_create(const tg_cone_geometry* g, int device, tg_cone_plan** out);
tg_status tg_cone_plan_destroy(tg_cone_plan* plan);
/* the plan's volume, detector and view count */
tg_status tg_cone_plan_shape(const tg_cone_plan* plan, tg_volume_spec* vol, tg_detector2d* det,
                             uint64_t* n_proj);

/* projector.hpp:264-281 forward_project(Image, ConeGeometry):
 * d_vol [nz][ny][nx] -> d_sino [n_proj][n_v][n_u] */
tg_status tg_cone_forward(tg_cone_plan* plan, const float* d_vol, float* d_sino, void* stream);
/* angle-sharded variant: views [view0, view0 + n_views) into
 * d_sino_part [n_views][n_v][n_u] */
tg_status tg_cone_forward_views(tg_cone_plan* plan, uint64_t view0, uint64_t n_views,
                                const float* d_vol, float* d_sino_part, void* stream);

/* projector.hpp:283-313 back_project(Sinogram, ConeGeometry):
 * d_vol = scale * BP(d_sino)  (+ d_vol if accumulate) */
tg_status tg_cone_backproject(tg_cone_plan* plan, const float* d_sino, float* d_vol, float scale,
                              int accumulate, void* stream);
/* z-slab back-projection for multi-GPU sharding: voxels z in [z0, z0+nz)
 * from detector rows [v0, v0+n_rows) of every view (d_band
 * [n_proj][n_rows][n_u]) into d_slab [nz][ny][nx].  Coordinates come from
 * global indices; when z0 and z0+nz are multiples of 32 (K1's z tile) or nz
 * reaches the volume's end, the slab is bitwise equal to the same z range of
 * the full-volume result.  The band must cover tg_cone_slab_rows(). */
tg_status tg_cone_slab_rows(tg_cone_plan* plan, uint64_t z0, uint64_t nz, uint64_t* v0,
                            uint64_t* n_rows);
/* the same from the geometry alone (host only, no device) */
tg_status tg_cone_slab_rows_geom(const tg_cone_geometry* g, uint64_t z0, uint64_t nz, uint64_t* v0,
                                 uint64_t* n_rows);
tg_status tg_cone_backproject_slab(tg_cone_plan* plan, uint64_t z0, uint64_t nz, uint64_t v0,
                                   uint64_t n_rows, const float* d_band, float* d_slab,
                                   float scale, int accumulate, void* stream);

/* filtering.hpp:136-154,115-125 as composed by pipelines.hpp:76-78:
 * out = RamLak( T(T(p*cos)*parker) ) row by row, for detector rows
 * [v0, v0+n_rows) of every view (d_in/d_out [n_proj][n_rows][n_u]; may alias) */
tg_status tg_cone_fdk_prefilter(tg_cone_plan* plan, const float* d_in, float* d_out, int use_parker,
                                uint64_t v0, uint64_t n_rows, void* stream);
/* pipelines.hpp:80-82 the FDK constant (range/n)(SDD/SID)(parker ? 1 : 1/2) */
double tg_cone_fdk_scale(const tg_cone_plan* plan, int use_parker);
/* pipelines.hpp:73-84 fdk_reconstruct; d_work is a sinogram-sized scratch
 * buffer (may equal d_sino to filter in place) */
tg_status tg_cone_fdk(tg_cone_plan* plan, const float* d_sino, float* d_vol, float* d_work,
                      int use_parker, void* stream);

/* host-buffer variants with the reference's by-value semantics; H2D copies
 * are pipelined against the kernels view-chunk by view-chunk */
tg_status tg_cone_forward_host(tg_cone_plan* plan, const float* h_vol, float* h_sino);
tg_status tg_cone_backproject_host(tg_cone_plan* plan, const float* h_sino, float* h_vol);
tg_status tg_cone_fdk_host(tg_cone_plan* plan, const float* h_sino, float* h_vol, int use_parker);
/* host-buffer z-slab back-projection (fdk = 0) or FDK (fdk = 1) of slab
 * [z0, z0+nz) from its detector row band h_band [n_proj][n_rows][n_u]
 * (raw projections when fdk = 1) into h_slab [nz][ny][nx].  Back-projection
 * copies only each view's detector footprint (pixels no voxel of the slab
 * interpolates are never read); FDK copies whole rows of the footprint's row
 * range (the filter runs along u).  Uploads run centre-out in z so finished
 * slices download while later rows upload. */
tg_status tg_cone_backproject_slab_host(tg_cone_plan* plan, uint64_t z0, uint64_t nz, uint64_t v0,
                                        uint64_t n_rows, const float* h_band, float* h_slab,
                                        int fdk, int use_parker);
/* bytes the plan's last host-buffer back-projection / FDK call copied host ->
 * device (the slab-BP path ships each view's own detector footprint only) */
uint64_t tg_cone_last_h2d_bytes(const tg_cone_plan* plan);

/* ---- parallel / fan beam 2D (K4-K7) ------------------------------------ */

typedef struct tg_planar_plan tg_planar_plan;

tg_status tg_planar_plan_create(const tg_planar_geometry* g, int device, tg_planar_plan** out);
tg_status tg_planar_plan_destroy(tg_planar_plan* plan);
tg_status tg_planar_plan_shape(const tg_planar_plan* plan, tg_volume_spec* vol,
                               tg_detector1d* det, uint64_t* n_proj);
/* projector.hpp:171-184 (parallel) / 212-230 (fan) forward_project */
tg_status tg_planar_forward(tg_planar_plan* plan, const float* d_img, float* d_sino, void* stream);
/* projector.hpp:186-208 (parallel) / 232-260 (fan, 1/U^2) back_project */
tg_status tg_planar_backproject(tg_planar_plan* plan, const float* d_sino, float* d_img,
                                float scale, int accumulate, void* stream);
tg_status tg_planar_forward_host(tg_planar_plan* plan, const float* h_img, float* h_sino);
tg_status tg_planar_backproject_host(tg_planar_plan* plan, const float* h_sino, float* h_img);

/* ---- row filters (K3 generic) ------------------------------------------ */

typedef struct tg_filter_plan tg_filter_plan;

/* filtering.hpp:27-32 Filter1D {filt_n_bins, padded_n, filt_spacing,
 * weights[n_weights]} bound to rows of row_len bins at row_spacing, with the
 * checks of apply_filter / filter_rows in the reference's order
 * (filtering.hpp:117-121, 97-99). */
tg_status tg_filter_plan_create(uint64_t row_len, double row_spacing, uint64_t filt_n_bins,
                                uint64_t padded_n, double filt_spacing, const double* weights,
                                uint64_t n_weights, int device, tg_filter_plan** out);
tg_status tg_filter_plan_destroy(tg_filter_plan* plan);
/* filtering.hpp:115-125 apply_filter on n_rows contiguous rows of n_bins
 * (d_in may alias d_out) */
tg_status tg_filter_apply(tg_filter_plan* plan, const float* d_in, float* d_out, uint64_t n_rows,
                          void* stream);
tg_status tg_filter_apply_host(tg_filter_plan* plan, const float* h_in, float* h_out,
                               uint64_t n_rows);

/* filtering.hpp:136-154 apply_weights: out[k] = T(double(in[k]) * map[k % map_n]) */
tg_status tg_apply_weights(const float* d_in, float* d_out, uint64_t n_total, const double* d_map,
                           uint64_t map_n, void* stream);
/* the same with a per-view row profile broadcast over detector rows (the cone
 * Parker map, filtering.hpp:246-247): data [n_views][n_rows][n], map [n_views][n] */
tg_status tg_apply_row_weights(const float* d_in, float* d_out, uint64_t n_views, uint64_t n_rows,
                               uint64_t n, const double* d_map, void* stream);

/* ---- iterative reconstruction ------------------------
 * The reference's graph pieces on the device path (graph.hpp, pipelines.hpp:273-299).
 * Reductions are FP64 with a fixed grid and ordered passes: deterministic. */

/* graph.hpp:345-353 l2_loss value + graph.hpp:498-509 gradient (upstream 1):
 * d_grad = 2 (a - b) (may alias d_a; NULL = value only); *d_sum = sum (a - b)^2 */
tg_status tg_l2_residual(const float* d_a, const float* d_b, float* d_grad, uint64_t n,
                         double* d_sum, void* stream);
/* graph.hpp:365-377 tv_value, graph.hpp:511-528 subgradient, graph.hpp:533-546
 * descent, fused: over a [nz][ny][nx] block (x fastest; nz = 1 for images),
 * x_out = x - lr * (lambda * subgrad_TV(x) + grad), *d_tv = TV of the forward
 * pairs the block owns.  has_lo / has_hi: the slice before / after the block
 * exists in memory (a z-slab of a full replica; multi-GPU).  d_grad = d_x_out =
 * NULL: value only.  d_x_out must not alias d_x. */
tg_status tg_tv_step(const float* d_x, const float* d_grad, float* d_x_out, uint64_t nx,
                     uint64_t ny, uint64_t nz, int has_lo, int has_hi, double tv_lambda,
                     double learning_rate, double* d_tv, void* stream);
/* Multi-GPU forms of the same kernels with the exchange fused in (SURVEY §8e,
 * config c5): destinations may be peer buffers mapped through CUDA IPC, so the
 * stores travel over NVLink / NVSwitch as the values are computed.
 * tg_l2_residual_scatter: K8 over this rank's views [view0, view0 + n_views) of
 * [n_v][n_u] projections, each residual row stored into every band that holds
 * it (band d: [n_proj][n_rows_d][n_u], rows [v0_d, v0_d + n_rows_d)).
 * tg_tv_step_multi: K9 with the updated block stored to 1..16 destinations. */
typedef struct tg_band_dest {
  float* band;
  uint64_t v0, n_rows;
} tg_band_dest;
tg_status tg_l2_residual_scatter(const float* d_fp, const float* d_p, uint64_t n_views,
                                 uint64_t n_v, uint64_t n_u, uint64_t view0,
                                 const tg_band_dest* dests, int n_dests, double* d_sum,
                                 void* stream);
tg_status tg_tv_step_multi(const float* d_x, const float* d_grad, float* const* d_x_outs, int n_out,
                           uint64_t nx, uint64_t ny, uint64_t nz, int has_lo, int has_hi,
                           double tv_lambda, double learning_rate, double* d_tv, void* stream);
/* device buffers shareable with the other ranks of a node (cudaMalloc bases,
 * zero-filled), their 64-byte CUDA IPC handles, and peer mappings */
tg_status tg_device_alloc(uint64_t bytes, int device, void** d_ptr);
tg_status tg_device_free(void* d_ptr);
tg_status tg_ipc_get_handle(const void* d_base, unsigned char* out64);
tg_status tg_ipc_open_handle(const unsigned char* in64, int device, void** d_ptr);
tg_status tg_ipc_close_handle(void* d_ptr);
/* pipelines.hpp:273-299 tv_reconstruct (graph: x -> forward_project -> l2_loss(., p)
 * + tv_lambda * tv_loss(x), plain gradient descent), on any geometry, device
 * resident: d_x holds the initial image (the reference starts from zero) and
 * receives the result; h_loss_history[iterations + 1] the loss before every
 * step and after the last (NULL allowed).  Non-finite loss -> TG_ERROR with the
 * reference's check_converging message (pipelines.hpp:166-170). */
tg_status tg_cone_tv_reconstruct(tg_cone_plan* plan, const float* d_sino, float* d_x,
                                 uint64_t iterations, double learning_rate, double tv_lambda,
                                 double* h_loss_history, void* stream);
tg_status tg_planar_tv_reconstruct(tg_planar_plan* plan, const float* d_sino, float* d_x,
                                   uint64_t iterations, double learning_rate, double tv_lambda,
                                   double* h_loss_history, void* stream);
/* the same with host buffers (h_x: initial image in, result out) */
tg_status tg_cone_tv_reconstruct_host(tg_cone_plan* plan, const float* h_sino, float* h_x,
                                      uint64_t iterations, double learning_rate, double tv_lambda,
                                      double* h_loss_history);
tg_status tg_planar_tv_reconstruct_host(tg_planar_plan* plan, const float* h_sino, float* h_x,
                                        uint64_t iterations, double learning_rate,
                                        double tv_lambda, double* h_loss_history);
/* ---- the remaining graph nodes on the device ---------
 * The reference's reverse-mode graph (graph.hpp) over device fp32 values:
 * forward_project / backproject nodes call the projector entry points above
 * (their registered gradients are each other, graph.hpp:408-434, with
 * accumulate = 1 for the back-projection); the rest are these.  Arithmetic is
 * FP64 rounded once to fp32; reductions use fixed grids (deterministic). */
/* add / scale nodes and gradient accumulation (graph.hpp:318-328, 498-508):
 * out = alpha a + beta b; d_b NULL: out = alpha a.  out may alias a or b. */
tg_status tg_axpby(const float* d_a, const float* d_b, float* d_out, uint64_t n, double alpha,
                   double beta, void* stream);
/* multiply_weights node (graph.hpp:137-149, 303-310): out[i] = x[i] w[i % block] */
tg_status tg_multiply_weights(const float* d_x, const float* d_w, float* d_out, uint64_t n,
                              uint64_t block, void* stream);
/* its gradient (graph.hpp:449-460): gx[i] += g[i] w[i % block];
 * gw[j] += sum over rows g x (either output may be NULL) */
tg_status tg_multiply_weights_grad(const float* d_g, const float* d_x, const float* d_w, float* d_gx,
                                   float* d_gw, uint64_t n, uint64_t block, void* stream);
/* fourier_filter node (graph.hpp:152-164, 312-316, 386-401): each of n_rows
 * rows of n samples zero-padded to P, Re(IFFT(k FFT(row))), first n kept; k is
 * a device vector of P weights (any real values: a trainable parameter) */
tg_status tg_fourier_filter(const float* d_x, const float* d_k, float* d_out, uint64_t n_rows,
                            uint64_t n, uint64_t P, void* stream);
/* its weight gradient (graph.hpp:478-496): gk[f] += sum_rows Re(X_f conj G_f) / P.
 * (The input gradient is tg_fourier_filter of the upstream gradient.) */
tg_status tg_fourier_filter_weight_grad(const float* d_x, const float* d_g, float* d_gk,
                                        uint64_t n_rows, uint64_t n, uint64_t P, void* stream);
/* l2_loss gradient (graph.hpp:498-509, upstream gs): d = 2 gs (a - b);
 * ga += d; gb -= d (either may be NULL).  The value is tg_l2_residual. */
tg_status tg_l2_grad(const float* d_a, const float* d_b, float* d_ga, float* d_gb, uint64_t n,
                     double gs, void* stream);
/* tv_loss gradient (graph.hpp:511-528, upstream gs) over an [nz][ny][nx]
 * block: gx += gs * subgrad_TV(x); *d_tv = TV(x).  d_gx must not alias d_x. */
tg_status tg_tv_grad(const float* d_x, float* d_gx, uint64_t nx, uint64_t ny, uint64_t nz,
                     double gs, double* d_tv, void* stream);

/* graph.hpp:389-393 check_grad_finite: *d_count += number of NaN entries of
 * d_x[0..n) (exact integer count; +-inf are not NaN, as std::isnan) */
tg_status tg_nan_count(const float* d_x, uint64_t n, uint64_t* d_count, void* stream);

/* pipelines.hpp:202-259 (experiment_learn_filter's loop), device resident on
 * a parallel / fan plan: frequency weights K (d_k: P floats; in: the initial
 * weights, out: the learned ones) descend on |pi/n BP(fourier_filter(p, K)) -
 * target|^2 at learning_rate.  h_init / h_ramlak (P doubles, host): the initial
 * and Ram-Lak weights for the recorded distance |K - ramlak| / |init - ramlak|.
 * h_loss / h_dist: iterations + 1 entries (NULL allowed); d_recon (NULL
 * allowed): the final reconstruction.  Non-finite loss -> TG_ERROR with the
 * reference's message. */
tg_status tg_planar_learn_filter(tg_planar_plan* plan, const float* d_sino, const float* d_target,
                                 float* d_k, uint64_t P, const double* h_init,
                                 const double* h_ramlak, double learning_rate, uint64_t iterations,
                                 double* h_loss, double* h_dist, float* d_recon, void* stream);
/* the same with host buffers (h_k: initial weights in, learned weights out;
 * h_recon may be NULL) */
tg_status tg_planar_learn_filter_host(tg_planar_plan* plan, const float* h_sino,
                                      const float* h_target, float* h_k, uint64_t P,
                                      const double* h_init, const double* h_ramlak,
                                      double learning_rate, uint64_t iterations, double* h_loss,
                                      double* h_dist, float* h_recon);
/* pipelines.hpp:119-132 add_gaussian_noise (host, bit-exact: std::mt19937_64
 * Box-Muller of pipelines.hpp:90-115; sigma = relative_std * max(in)) */
tg_status tg_add_gaussian_noise(const float* h_in, float* h_out, uint64_t n, double relative_std,
                                uint64_t seed);

/* ---- synthetic inputs (phantom.hpp:34-88, bit-exact, FP64) ------------- */

/* specs: n x 8 doubles {cx, cy, cz, a, b, c, phi_deg, intensity} */
tg_status tg_rasterize_ellipsoids(const tg_volume_spec* vol, const double* specs, uint64_t n,
                                  float* d_out, void* stream);
/* specs: n x 6 doubles {cx, cy, a, b, phi_deg, intensity} */
tg_status tg_rasterize_ellipses(const tg_volume_spec* vol, const double* specs, uint64_t n,
                                float* d_out, void* stream);
/* phantom.hpp:107-128 tables scaled by fov_half_extent(vol) */
tg_status tg_head_phantom_ellipsoids(const tg_volume_spec* vol, double* out80);
tg_status tg_head_phantom_ellipses(const tg_volume_spec* vol, double* out60);

/* ---- diagnostics ---------------------------------------------------------- */

/* projector.hpp:83-107,117,138: the per-ray sample count n = ceil((t1-t0)/step)
 * the forward projector marches (0 = the ray misses the volume), from the
 * device's own FP64 ray setup + clip (the code K2 / K5 / K7 run).
 * Cone: d_counts [n_views][n_v][n_u]; planar: [n_proj][n_bins]. */
tg_status tg_cone_ray_samples(tg_cone_plan* plan, uint64_t view0, uint64_t n_views,
                              uint64_t* d_counts, void* stream);
tg_status tg_planar_ray_samples(tg_planar_plan* plan, uint64_t* d_counts, void* stream);
/* plan knobs for experiments and tests (outputs are bitwise unchanged):
 * "k2_tu" = 32 | 64 (K2 CTA width / detector band height 8 | 4 rows),
 * "k2_dual" = 0 | 1 (keep the y-fastest quad volume for x-dominant rays),
 * "k2_impl" = 1 (slab-staged K2: shared-memory volume boxes) | 0 (quad-volume
 * K2: L1 gathers) | -1 (default: time both at the plan's first forward
 * projection and keep the faster) */
tg_status tg_cone_plan_set_knob(tg_cone_plan* plan, const char* name, int64_t value);

/* ---- instrumentation ---------------------------------------------------- */

/* number of kernels this library launched in the calling process so far */
uint64_t tg_kernel_launch_count(void);
/* average device time (ms) of the last call's dominant kernel, measured with
 * CUDA events on the launch stream when tg_set_timing(1) */
void tg_set_timing(int enable);
double tg_last_kernel_ms(void);

#ifdef __cplusplus
}
#endif
#endif /* TOMOGRAD_B200_H */
