// filter.cuh — K3: row-wise frequency-domain filtering (Ram-Lak / ramp /
// learned weights) with the FDK cosine and Parker weights fused into the
// load.  Reference: filtering.hpp:95-125 (filter_rows / apply_filter),
// 136-154 (apply_weights), fft.hpp:25-58 (the transform it replaces).
#pragma once

#include "device_common.cuh"

namespace tgb {
namespace filt {

struct RowFilter {
  int device = 0;
  uint64_t n = 0;          // row length (detector bins)
  uint64_t P = 0;          // power-of-two window
  bool symmetric = true;   // weights symmetrised at creation: two real rows share one complex FFT
  float* d_w = nullptr;    // P real weights (fp32)
  float2* d_tw = nullptr;  // P twiddles exp(-2 pi i k / P) (from FP64)
  float2* d_tw16 = nullptr;  // per-pass [r][k] twiddle tables of the radix-16 path
};

// Optional per-element weights applied (in FP64, rounded to fp32 after each
// map, like the reference's two apply_weights passes) before filtering.
// Row r of the launch is detector row cos_row0 + r % rows_per_view of view
// r / rows_per_view.
struct PreWeights {
  const double* cos = nullptr;     // [n_v][n] (full detector)
  uint64_t cos_row0 = 0;
  uint64_t rows_per_view = 1;
  const double* parker = nullptr;  // [views][n]
};

RowFilter* create(uint64_t n, uint64_t P, const double* weights, int device);

// graph fourier_filter node (device weights k[P], any real values; d_ks: P
// floats of scratch for the symmetrised copy) and its weight gradient
// gk (+)= sum_rows Re(X conj G) / P (d_partial: weight_grad_parts(n_rows) * P doubles)
void fourier_filter(const float* d_x, const float* d_k, float* d_ks, float* d_out,
                    uint64_t n_rows, uint64_t n, uint64_t P, cudaStream_t st);
int weight_grad_parts(uint64_t n_rows);
void weight_grad(const float* d_x, const float* d_g, float* d_gk, double* d_partial,
                 uint64_t n_rows, uint64_t n, uint64_t P, bool accumulate, cudaStream_t st);
void destroy(RowFilter* f);
// Row r of a launch starts at (r / rows_per_view) * view_pitch +
// (r % rows_per_view) * n elements (rows_per_view = 0: rows are contiguous) —
// a row segment of every view of a band buffer.  Strided layouts need a
// window P in [512, 8192] (the register FFT path).
struct RowLayout {
  uint64_t rows_per_view = 0;
  uint64_t view_pitch = 0;
};
__host__ __device__ inline uint64_t row_offset(uint64_t r, int n, const RowLayout& L) {
  return L.rows_per_view ? (r / L.rows_per_view) * L.view_pitch + (r % L.rows_per_view) * uint64_t(n)
                         : r * uint64_t(n);
}
// pdl: launch the pre-weights pass with programmatic stream serialization (it
// may start while the stream's previous kernel drains; it waits for that
// kernel before it exits, so its completion still implies the previous one's).
// Only when the previous kernel neither writes these rows nor reads them.
void apply(const RowFilter& f, const float* d_in, float* d_out, uint64_t n_rows,
           const PreWeights* pw, cudaStream_t st, RowLayout lay = RowLayout{}, bool pdl = false);

}  // namespace filt
}  // namespace tgb
