// graph.cu — the elementwise nodes of the reference's reverse-mode graph on
// the device (graph.hpp:137-190 builders, 296-343
// evaluation, 470-531 gradients).  The projector, filter, l2 and TV nodes run
// on K1-K9 (cone.cu, planar.cu, filter.cu, iterative.cu); these are the glue:
//
//   tg_axpby                 out = alpha a + beta b        add / scale nodes and
//                                                          every gradient accumulation
//   tg_multiply_weights      out = x * w[i % block]        graph.hpp:303-310
//   tg_multiply_weights_grad gx += g * w[i % block],       graph.hpp:449-460
//                            gw[j] += sum_r g x  (broadcast axes summed)
//
// All HBM-bound (12 B per element); arithmetic in FP64 rounded once to fp32
// (the reference keeps Tensor<double>; the device graph stores fp32).  The
// weight-gradient reduction runs over a fixed chunk grid in a fixed order:
// bit-for-bit deterministic run to run.
#include <algorithm>

#include "device_common.cuh"

namespace tgb {
namespace graph {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + kThreads - 1) / kThreads, 148 * 16)));
}

__global__ void axpby_kernel(const float* a, const float* b, float* out, uint64_t n, double alpha,
                             double beta) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = alpha * double(a[i]);
    if (b) v += beta * double(b[i]);
    out[i] = float(v);
  }
}

__global__ void multiply_weights_kernel(const float* x, const float* __restrict__ w, float* out,
                                        uint64_t n, uint64_t block) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = float(double(x[i]) * double(__ldg(w + i % block)));
}

// gx += g * w (elementwise; gx may be null)
__global__ void multiply_weights_gx_kernel(const float* __restrict__ g, const float* __restrict__ w,
                                           float* gx, uint64_t n, uint64_t block) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    gx[i] = float(double(gx[i]) + double(g[i]) * double(__ldg(w + i % block)));
}

// *count += number of NaN entries (graph.hpp:389-393 check_grad_finite tests
// std::isnan only: +-inf passes); integer atomics, so the count is exact
__global__ void nan_count_kernel(const float* __restrict__ g, uint64_t n,
                                 unsigned long long* count) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned c = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    c += isnan(g[i]) ? 1u : 0u;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

// partial[c][j] = sum over the rows of chunk c of g x at column j
// (grid: x over columns, y over row chunks; coalesced along j)
__global__ void multiply_weights_gw_partial(const float* __restrict__ g, const float* __restrict__ x,
                                            uint64_t rows, uint64_t block, uint64_t rows_per_chunk,
                                            double* __restrict__ partial) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= block) return;
  const uint64_t r0 = uint64_t(blockIdx.y) * rows_per_chunk;
  const uint64_t r1 = std::min(rows, r0 + rows_per_chunk);
  double acc = 0.0;
  for (uint64_t r = r0; r < r1; ++r) acc += double(g[r * block + j]) * double(x[r * block + j]);
  partial[uint64_t(blockIdx.y) * block + j] = acc;
}

__global__ void multiply_weights_gw_reduce(const double* __restrict__ partial, int chunks,
                                           uint64_t block, float* gw) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= block) return;
  double acc = 0.0;
  for (int c = 0; c < chunks; ++c) acc += partial[uint64_t(c) * block + j];
  gw[j] = float(double(gw[j]) + acc);
}

}  // namespace graph
}  // namespace tgb

using namespace tgb;

extern "C" {

tg_status tg_axpby(const float* d_a, const float* d_b, float* d_out, uint64_t n, double alpha,
                   double beta, void* stream) {
  return guarded([&] {
    if (n == 0) return;
    graph::axpby_kernel<<<graph::grid_for(n), graph::kThreads, 0, as_stream(stream)>>>(
        d_a, d_b, d_out, n, alpha, beta);
    TG_LAUNCHED(1);
  });
}

tg_status tg_multiply_weights(const float* d_x, const float* d_w, float* d_out, uint64_t n,
                              uint64_t block, void* stream) {
  return guarded([&] {
    check(block >= 1 && n % block == 0,
          "weight shape must equal the input shape or a prefix of it");
    if (n == 0) return;
    graph::multiply_weights_kernel<<<graph::grid_for(n), graph::kThreads, 0, as_stream(stream)>>>(
        d_x, d_w, d_out, n, block);
    TG_LAUNCHED(1);
  });
}

tg_status tg_multiply_weights_grad(const float* d_g, const float* d_x, const float* d_w, float* d_gx,
                                   float* d_gw, uint64_t n, uint64_t block, void* stream) {
  return guarded([&] {
    check(block >= 1 && n % block == 0,
          "weight shape must equal the input shape or a prefix of it");
    if (n == 0) return;
    const cudaStream_t st = as_stream(stream);
    if (d_gx) {
      graph::multiply_weights_gx_kernel<<<graph::grid_for(n), graph::kThreads, 0, st>>>(
          d_g, d_w, d_gx, n, block);
      TG_LAUNCHED(1);
    }
    if (d_gw) {
      const uint64_t rows = n / block;
      const int chunks = int(std::min<uint64_t>(rows, 256));
      const uint64_t per = (rows + chunks - 1) / chunks;
      const int used = int((rows + per - 1) / per);
      double* partial = nullptr;
      TG_CUDA(cudaMallocAsync(&partial, sizeof(double) * block * used, st));
      const dim3 grid(unsigned((block + graph::kThreads - 1) / graph::kThreads), unsigned(used));
      graph::multiply_weights_gw_partial<<<grid, graph::kThreads, 0, st>>>(d_g, d_x, rows, block,
                                                                          per, partial);
      graph::multiply_weights_gw_reduce<<<grid.x, graph::kThreads, 0, st>>>(partial, used, block,
                                                                           d_gw);
      TG_LAUNCHED(2);
      TG_CUDA(cudaFreeAsync(partial, st));
    }
  });
}

tg_status tg_nan_count(const float* d_x, uint64_t n, uint64_t* d_count, void* stream) {
  return guarded([&] {
    if (n == 0) return;
    graph::nan_count_kernel<<<graph::grid_for(n), graph::kThreads, 0, as_stream(stream)>>>(
        d_x, n, reinterpret_cast<unsigned long long*>(d_count));
    TG_LAUNCHED(1);
  });
}

}  // extern "C"
