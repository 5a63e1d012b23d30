// iterative.cu — the TV-regularised iterative reconstruction loop (SURVEY §8f
// row 1): the reference's graph pieces on the device path.
//
//   loss(x) = |A x - p|^2 + lambda * TV(x),  x <- x - lr * grad      (pipelines.hpp:273-299)
//
// Reference pieces restated here:
//   l2_loss value / gradient            graph.hpp:345-353, 498-509
//   tv_loss value (anisotropic, forward differences over every axis)
//                                        graph.hpp:365-377
//   tv_loss subgradient (sign, flat -> 0) graph.hpp:511-528
//   gradient_descent_step               graph.hpp:533-546
//   check_converging                    pipelines.hpp:166-170
//
// K8 l2_residual_kernel: one pass over the sinogram: g = 2 (a - b) in place
//    and sum (a - b)^2 in FP64 (fixed grid + ordered second pass: bit-for-bit
//    deterministic run to run).  HBM-bound: 12 B per detector pixel.
// K9 tv_step_kernel: one pass over the volume (or a z-slab of it with
//    one-slice halos): TV value of the forward differences it owns, the
//    subgradient, the data gradient (the back-projection) and the descent
//    update fused; x is double-buffered.  HBM-bound: 12 B per voxel
//    (x, grad in; x' out), neighbour re-reads hit L1/L2.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "filter.cuh"

namespace tgb {
namespace iter {

constexpr int kRedBlocks = 148 * 8;  // fixed reduction grid (deterministic partials)
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-level sum in a fixed order; result valid in thread 0
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[kRedThreads / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) ws[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kRedThreads / 32; ++i) r += ws[i];
  __syncthreads();
  return r;
}

// K8: g = 2 * gs * (a - b) (graph.hpp:503: d = 2.0 * gs * (a[i] - b[i])),
// partial[block] = sum (a - b)^2 (graph.hpp:347-351)
__global__ void __launch_bounds__(kRedThreads) l2_residual_kernel(const float* a,
                                                                   const float* __restrict__ b,
                                                                   float* g, uint64_t n, double gs2,
                                                                   double* __restrict__ partial) {
  double acc = 0.0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double d = double(a[i]) - double(b[i]);
    acc += d * d;
    if (g) g[i] = float(gs2 * d);
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// ordered sum of kRedBlocks partials -> out[0]
__global__ void sum_partials_kernel(const double* __restrict__ partial, int n, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) out[0] = acc;
}

__device__ __forceinline__ int sgn(double d) { return (d > 0.0) - (d < 0.0); }

// K9: over the voxels of a slab [nz][ny][nx] (x fastest) whose z neighbours
// outside the slab exist when has_lo / has_hi (the caller's pointer is into a
// full replica).  For each voxel i:
//   s_i = sum_a [ sgn(x_i - x_{i-s_a}) ] - [ sgn(x_{i+s_a} - x_i) ]
//   x'_i = x_i - lr * (lambda * s_i + grad_i)
// and the TV of the forward pairs (i, i + s_a) it owns.  Differences of fp32
// values are exact in FP64, so signs and |d| are exactly the reference's for
// the same x.  x_out == nullptr: value only.
// Destinations of one computed value: the local buffer and / or peer buffers
// mapped through CUDA IPC (NVLink / NVSwitch stores on a multi-GPU node).
constexpr int kMaxDest = 16;
struct OutList {
  float* p[kMaxDest];
  int n;
};

// subgradient count s_i of voxel i and the TV of the forward pairs it owns
// (graph.hpp:365-377, 511-528; axes x, y, z in the reference's order)
__device__ __forceinline__ int tv_stencil(const float* __restrict__ x, long long i, int nx, int ny,
                                          int nz, long long plane, int has_lo, int has_hi,
                                          double& tv) {
  const int ix = int(i % nx);
  const long long r = i / nx;
  const int iy = int(r % ny), iz = int(r / ny);
  const double xi = x[i];
  int s = 0;
  if (ix >= 1) s += sgn(xi - double(x[i - 1]));
  if (ix + 1 < nx) {
    const double d = double(x[i + 1]) - xi;
    s -= sgn(d);
    tv += fabs(d);
  }
  if (iy >= 1) s += sgn(xi - double(x[i - nx]));
  if (iy + 1 < ny) {
    const double d = double(x[i + nx]) - xi;
    s -= sgn(d);
    tv += fabs(d);
  }
  if (iz >= 1 || has_lo) s += sgn(xi - double(x[i - plane]));
  if (iz + 1 < nz || has_hi) {
    const double d = double(x[i + plane]) - xi;
    s -= sgn(d);
    tv += fabs(d);
  }
  return s;
}

__global__ void __launch_bounds__(kRedThreads) tv_step_kernel(
    const float* __restrict__ x, const float* __restrict__ grad, const OutList outs, int nx,
    int ny, int nz, int has_lo, int has_hi, double lambda, double lr, double* __restrict__ partial) {
  const long long plane = (long long)nx * ny;
  const long long n = plane * nz;
  double tv = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int s = tv_stencil(x, i, nx, ny, nz, plane, has_lo, has_hi, tv);
    if (outs.n) {
      const double xi = x[i];
      const double g = lambda * double(s) + double(grad[i]);
      const float v = float(xi - lr * g);
#pragma unroll 1
      for (int d = 0; d < outs.n; ++d) outs.p[d][i] = v;  // local and / or peer replicas
    }
  }
  tv = block_sum(tv);
  if (threadIdx.x == 0) partial[blockIdx.x] = tv;
}

// the backward of a graph tv_loss node alone (graph.hpp:511-528, upstream
// gradient gs): gx_i += gs * s_i, plus the TV value.  gx must not alias x.
__global__ void __launch_bounds__(kRedThreads) tv_grad_kernel(const float* __restrict__ x,
                                                              float* __restrict__ gx, int nx,
                                                              int ny, int nz, double gs,
                                                              double* __restrict__ partial) {
  const long long plane = (long long)nx * ny;
  const long long n = plane * nz;
  double tv = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int s = tv_stencil(x, i, nx, ny, nz, plane, 0, 0, tv);
    if (s) gx[i] = float(double(gx[i]) + gs * double(s));
  }
  tv = block_sum(tv);
  if (threadIdx.x == 0) partial[blockIdx.x] = tv;
}

// the backward of a graph l2_loss node (graph.hpp:498-509, upstream gs):
// d = 2 gs (a - b); ga += d; gb -= d (either may be null)
__global__ void l2_grad_kernel(const float* __restrict__ a, const float* __restrict__ b,
                               float* ga, float* gb, uint64_t n, double gs2) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double d = gs2 * (double(a[i]) - double(b[i]));
    if (ga) ga[i] = float(double(ga[i]) + d);
    if (gb) gb[i] = float(double(gb[i]) - d);
  }
}

// stream-ordered device buffer (pool-backed: no device-wide sync)
template <typename T>
struct AsyncBuf {
  T* p = nullptr;
  cudaStream_t st;
  AsyncBuf(size_t n, cudaStream_t s) : st(s) { TG_CUDA(cudaMallocAsync(&p, n * sizeof(T), st)); }
  ~AsyncBuf() { cudaFreeAsync(p, st); }
  AsyncBuf(const AsyncBuf&) = delete;
  AsyncBuf& operator=(const AsyncBuf&) = delete;
};

// keep freed stream-ordered allocations cached in the device pool (the
// default release threshold returns them to the driver at every sync, so each
// loop call would re-map its multi-GB work buffers)
inline void keep_pool(cudaStream_t st) {
  static std::once_flag once[64];
  int dev = 0;
  TG_CUDA(cudaGetDevice(&dev));
  std::call_once(once[dev & 63], [&] {
    cudaMemPool_t pool;
    TG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~0ull;
    TG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  });
  (void)st;
}

struct Scratch {
  AsyncBuf<double> buf;
  double* partial;
  explicit Scratch(cudaStream_t s) : buf(kRedBlocks, s), partial(buf.p) {}
};

OutList one_out(float* p) {
  OutList o;
  o.n = p ? 1 : 0;
  o.p[0] = p;
  return o;
}

// K8 with the exchange fused in: g = 2 (fp - p) of this rank's views, each
// row stored straight into the row band of every slab owner that needs it
// (peer buffers through IPC: the all_to_all of the sharded loop without a
// separate collective or staging copy).  fp is [n_views][nv][nu]; band d
// is [n_proj][n_rows_d][nu] holding rows [v0_d, v0_d + n_rows_d).
struct BandList {
  float* p[kMaxDest];
  int v0[kMaxDest], n_rows[kMaxDest];
  int n;
};

__global__ void __launch_bounds__(kRedThreads) l2_scatter_kernel(
    const float* __restrict__ fp, const float* __restrict__ pm, uint64_t n, int nv, int nu,
    int view0, const BandList bands, double* __restrict__ partial) {
  double acc = 0.0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double d = double(fp[i]) - double(pm[i]);
    acc += d * d;
    const float g = float(2.0 * d);
    const int u = int(i % nu);
    const uint64_t rv = i / nu;
    const int r = int(rv % nv);
    const long long view = (long long)(rv / nv) + view0;
#pragma unroll 1
    for (int b = 0; b < bands.n; ++b) {
      const int rr = r - bands.v0[b];
      if (rr >= 0 && rr < bands.n_rows[b])
        bands.p[b][(view * bands.n_rows[b] + rr) * nu + u] = g;
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

void l2_residual(const float* a, const float* b, float* g, uint64_t n, double* d_sum,
                 cudaStream_t st, const Scratch& sc) {
  l2_residual_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, g, n, 2.0 * 1.0, sc.partial);
  sum_partials_kernel<<<1, kRedThreads, 0, st>>>(sc.partial, kRedBlocks, d_sum);
  TG_LAUNCHED(2);
}

void tv_step(const float* x, const float* grad, const OutList& outs, uint64_t nx, uint64_t ny,
             uint64_t nz, int has_lo, int has_hi, double lambda, double lr, double* d_tv,
             cudaStream_t st, const Scratch& sc) {
  tv_step_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(x, grad, outs, int(nx), int(ny), int(nz),
                                                      has_lo, has_hi, lambda, lr, sc.partial);
  sum_partials_kernel<<<1, kRedThreads, 0, st>>>(sc.partial, kRedBlocks, d_tv);
  TG_LAUNCHED(2);
}

// One device-resident descent loop over any projector pair (fwd, bwd) —
// pipelines.hpp:276-298 with the graph's evaluation order: forward (loss of
// the current x), backward, step; a final forward records the last loss.
// appends the (data, tv) pair of the step just finished to sums[] at a
// device-side counter, so a captured iteration needs no per-step parameters
__global__ void record_kernel(const double* __restrict__ slot, double* __restrict__ sums,
                              int* __restrict__ counter) {
  const int c = counter[0];
  sums[2 * c] = slot[0];
  sums[2 * c + 1] = slot[1];
  counter[0] = c + 1;
}

// One device-resident descent loop over any projector pair (fwd, bwd) —
// pipelines.hpp:276-298 with the graph's evaluation order: forward (loss of
// the current x), backward, step; a final forward records the last loss.
// graph_ok: the pair may be captured into a CUDA graph (no constant-bank
// switches inside an iteration); small problems are launch-bound, so two
// iterations (x -> x2 -> x) are captured once and replayed.
template <typename Fwd, typename Bwd>
void tv_loop(Fwd fwd, Bwd bwd, uint64_t n_sino, uint64_t nx, uint64_t ny, uint64_t nz,
             const float* d_sino, float* d_x, uint64_t iterations, double lr, double lambda,
             double* h_hist, cudaStream_t st, bool graph_ok = false) {
  const uint64_t n_vox = nx * ny * nz;
  keep_pool(st);
  AsyncBuf<float> fp_b(n_sino, st), bp_b(n_vox, st), x2_b(n_vox, st);
  AsyncBuf<double> sums_b(2 * (iterations + 1), st);  // [iterations + 1][2] = (data, tv)
  AsyncBuf<double> slot_b(2, st);
  AsyncBuf<int> ctr_b(1, st);
  TG_CUDA(cudaMemsetAsync(ctr_b.p, 0, sizeof(int), st));
  float *fp = fp_b.p, *bp = bp_b.p, *x2 = x2_b.p;
  double *sums = sums_b.p, *slot = slot_b.p;
  int* ctr = ctr_b.p;
  Scratch sc(st);
  auto step = [&](float* cur, float* nxt, cudaStream_t s) {
    fwd(cur, fp, s);
    l2_residual(fp, d_sino, fp, n_sino, slot, s, sc);
    bwd(fp, bp, s);
    tv_step(cur, bp, one_out(nxt), nx, ny, nz, 0, 0, lambda, lr, slot + 1, s, sc);
    record_kernel<<<1, 1, 0, s>>>(slot, sums, ctr);
    TG_LAUNCHED(1);
  };
  float* cur = d_x;
  float* nxt = x2;
  uint64_t it = 0;
  if (graph_ok && iterations >= 5) {
    step(cur, nxt, st);  // plan state (pads, constant bank owner) settles un-captured
    std::swap(cur, nxt);
    ++it;
    // capture on a private stream (the caller's may be the legacy default)
    cudaStream_t gs;
    cudaEvent_t ev;
    TG_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
    TG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TG_CUDA(cudaEventRecord(ev, st));
    TG_CUDA(cudaStreamWaitEvent(gs, ev, 0));
    const uint64_t launches0 = tg_kernel_launch_count();
    TG_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
    step(cur, nxt, gs);
    step(nxt, cur, gs);
    cudaGraph_t g;
    TG_CUDA(cudaStreamEndCapture(gs, &g));
    const uint64_t per_replay = tg_kernel_launch_count() - launches0;
    cudaGraphExec_t ge;
    TG_CUDA(cudaGraphInstantiate(&ge, g, 0));
    const uint64_t replays = (iterations - it) / 2;
    for (uint64_t r = 0; r < replays; ++r) TG_CUDA(cudaGraphLaunch(ge, gs));
    count_launch(per_replay * (replays ? replays - 1 : 0));  // capture counted one replay's worth
    it += 2 * replays;
    TG_CUDA(cudaEventRecord(ev, gs));
    TG_CUDA(cudaStreamWaitEvent(st, ev, 0));
    TG_CUDA(cudaStreamSynchronize(gs));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaEventDestroy(ev);
    cudaStreamDestroy(gs);
  }
  for (; it < iterations; ++it) {
    step(cur, nxt, st);
    std::swap(cur, nxt);
  }
  fwd(cur, fp, st);
  l2_residual(fp, d_sino, nullptr, n_sino, slot, st, sc);
  tv_step(cur, nullptr, one_out(nullptr), nx, ny, nz, 0, 0, lambda, lr, slot + 1, st, sc);
  record_kernel<<<1, 1, 0, st>>>(slot, sums, ctr);
  TG_LAUNCHED(1);
  if (cur != d_x)
    TG_CUDA(cudaMemcpyAsync(d_x, cur, n_vox * sizeof(float), cudaMemcpyDeviceToDevice, st));
  std::vector<double> s(2 * (iterations + 1));
  TG_CUDA(cudaMemcpyAsync(s.data(), sums, s.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaStreamSynchronize(st));
  for (uint64_t i = 0; i <= iterations; ++i) {
    // graph add node: data + (tv * lambda)   (graph.hpp:331-343)
    const double loss = s[2 * i] + s[2 * i + 1] * lambda;
    if (h_hist) h_hist[i] = loss;
    if (!std::isfinite(loss))
      throw RefError("optimization diverged at iteration " + std::to_string(i) +
                     " (loss is not finite); lower the learning rate");
  }
}

// ---- filter learning (pipelines.hpp:202-259), device resident ------------
// One step on the trainable weights K (in place):
//   filtered = fourier_filter(p, K)             K3 (graph.hpp:312-316)
//   recon    = (pi / n) BP(filtered)            K6, scale node fused in the epilogue
//   loss     = |recon - target|^2, g = 2 (pi/n) (recon - target)   K8 (l2 + scale gradients)
//   gfil     = FP(g)                            K7 (backproject's registered gradient)
//   gK       = sum_rows Re(P conj G) / P        filter weight gradient (graph.hpp:478-496)
//   K       -= lr gK                            graph.hpp:533-546
// The recorded distance |K - ramlak|^2 is reduced on the device too, so a
// captured step needs no host round trip; one step is captured into a CUDA
// graph and replayed.
__global__ void lf_record_kernel(const double* __restrict__ loss_slot, const float* __restrict__ K,
                                 const double* __restrict__ ramlak, int P,
                                 double* __restrict__ hist, int* __restrict__ counter) {
  double d2 = 0.0;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const double d = double(K[k]) - ramlak[k];
    d2 += d * d;
  }
  d2 = block_sum(d2);
  if (threadIdx.x == 0) {
    const int c = counter[0];
    hist[2 * c] = loss_slot[0];
    hist[2 * c + 1] = d2;
    counter[0] = c + 1;
  }
}

__global__ void lf_descent_kernel(float* __restrict__ K, const float* __restrict__ gK, int P,
                                  double lr) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P; k += gridDim.x * blockDim.x)
    K[k] = float(double(K[k]) - lr * double(gK[k]));
}

template <typename Fwd, typename Bwd>
void learn_filter_loop(Fwd fwd, Bwd bwd, uint64_t n_rows, uint64_t n, uint64_t n_vox,
                       const float* d_sino, const float* d_target, float* d_k, uint64_t P,
                       const double* h_init, const double* h_ramlak, double lr,
                       uint64_t iterations, double factor, double* h_loss, double* h_dist,
                       float* d_recon, cudaStream_t st) {
  keep_pool(st);
  const uint64_t n_sino = n_rows * n;
  AsyncBuf<float> fil_b(n_sino, st), rec_b(n_vox, st), grec_b(n_vox, st), gfil_b(n_sino, st);
  AsyncBuf<float> ks_b(P, st), gk_b(P, st);
  AsyncBuf<double> part_b(size_t(filt::weight_grad_parts(n_rows)) * P, st);
  AsyncBuf<double> ramlak_b(P, st), hist_b(2 * (iterations + 1), st), slot_b(1, st);
  AsyncBuf<int> ctr_b(1, st);
  TG_CUDA(cudaMemcpyAsync(ramlak_b.p, h_ramlak, P * sizeof(double), cudaMemcpyHostToDevice, st));
  TG_CUDA(cudaMemsetAsync(ctr_b.p, 0, sizeof(int), st));
  Scratch sc(st);
  auto forward = [&](cudaStream_t s, bool with_grad) {
    filt::fourier_filter(d_sino, d_k, ks_b.p, fil_b.p, n_rows, n, P, s);
    bwd(fil_b.p, rec_b.p, float(factor), s);
    l2_residual_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(
        rec_b.p, d_target, with_grad ? grec_b.p : nullptr, n_vox, 2.0 * factor, sc.partial);
    sum_partials_kernel<<<1, kRedThreads, 0, s>>>(sc.partial, kRedBlocks, slot_b.p);
    lf_record_kernel<<<1, kRedThreads, 0, s>>>(slot_b.p, d_k, ramlak_b.p, int(P), hist_b.p,
                                               ctr_b.p);
    TG_LAUNCHED(3);
  };
  auto step = [&](cudaStream_t s) {
    forward(s, true);
    fwd(grec_b.p, gfil_b.p, s);
    filt::weight_grad(d_sino, gfil_b.p, gk_b.p, part_b.p, n_rows, n, P, false, s);
    lf_descent_kernel<<<unsigned((P + 255) / 256), 256, 0, s>>>(d_k, gk_b.p, int(P), lr);
    TG_LAUNCHED(1);
  };
  uint64_t it = 0;
  if (iterations >= 4) {
    step(st);  // un-captured: plan state and kernel attributes settle
    ++it;
    cudaStream_t gs;
    cudaEvent_t ev;
    TG_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
    TG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TG_CUDA(cudaEventRecord(ev, st));
    TG_CUDA(cudaStreamWaitEvent(gs, ev, 0));
    const uint64_t launches0 = tg_kernel_launch_count();
    TG_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
    step(gs);
    cudaGraph_t g;
    TG_CUDA(cudaStreamEndCapture(gs, &g));
    const uint64_t per_replay = tg_kernel_launch_count() - launches0;
    cudaGraphExec_t ge;
    TG_CUDA(cudaGraphInstantiate(&ge, g, 0));
    const uint64_t replays = iterations - it;
    for (uint64_t r = 0; r < replays; ++r) TG_CUDA(cudaGraphLaunch(ge, gs));
    count_launch(per_replay * (replays ? replays - 1 : 0));
    it += replays;
    TG_CUDA(cudaEventRecord(ev, gs));
    TG_CUDA(cudaStreamWaitEvent(st, ev, 0));
    TG_CUDA(cudaStreamSynchronize(gs));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaEventDestroy(ev);
    cudaStreamDestroy(gs);
  }
  for (; it < iterations; ++it) step(st);
  forward(st, false);
  if (d_recon)
    TG_CUDA(cudaMemcpyAsync(d_recon, rec_b.p, n_vox * sizeof(float), cudaMemcpyDeviceToDevice, st));
  std::vector<double> h(2 * (iterations + 1));
  TG_CUDA(cudaMemcpyAsync(h.data(), hist_b.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                          st));
  TG_CUDA(cudaStreamSynchronize(st));
  double gap = 0.0;
  for (uint64_t k = 0; k < P; ++k) {
    const double d = h_init[k] - h_ramlak[k];
    gap += d * d;
  }
  gap = std::sqrt(gap);
  for (uint64_t i = 0; i <= iterations; ++i) {
    if (h_loss) h_loss[i] = h[2 * i];
    if (h_dist) h_dist[i] = gap > 0.0 ? std::sqrt(h[2 * i + 1]) / gap : 0.0;
    if (!std::isfinite(h[2 * i]))
      throw RefError("optimization diverged at iteration " + std::to_string(i) +
                     " (loss is not finite); lower the learning rate");
  }
}

// host-buffer forms of the loop: one upload, the device loop, one download
template <typename Run>
tg_status tv_host(int device, uint64_t n_sino, uint64_t n_vox, const float* h_sino, float* h_x,
                  Run run) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaStream_t st;
    TG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    tg_status r = TG_OK;
    std::string msg;
    {
      AsyncBuf<float> s(n_sino, st), x(n_vox, st);
      TG_CUDA(cudaMemcpyAsync(s.p, h_sino, n_sino * sizeof(float), cudaMemcpyHostToDevice, st));
      TG_CUDA(cudaMemcpyAsync(x.p, h_x, n_vox * sizeof(float), cudaMemcpyHostToDevice, st));
      r = run(s.p, x.p, st);
      if (r == TG_OK)
        TG_CUDA(cudaMemcpyAsync(h_x, x.p, n_vox * sizeof(float), cudaMemcpyDeviceToHost, st));
      else
        msg = tg_last_error();
    }  // stream-ordered frees enqueued before the stream goes away
    TG_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    if (r != TG_OK) throw RefError(msg);
  });
}

}  // namespace iter
}  // namespace tgb

using namespace tgb;

extern "C" {

tg_status tg_l2_residual(const float* d_a, const float* d_b, float* d_grad, uint64_t n,
                         double* d_sum, void* stream) {
  return guarded([&] {
    check(n >= 1, "l2_loss expects matching shapes");
    const cudaStream_t st = as_stream(stream);
    iter::Scratch sc(st);
    iter::l2_residual(d_a, d_b, d_grad, n, d_sum, st, sc);
  });
}

tg_status tg_tv_step(const float* d_x, const float* d_grad, float* d_x_out, uint64_t nx,
                     uint64_t ny, uint64_t nz, int has_lo, int has_hi, double tv_lambda,
                     double learning_rate, double* d_tv, void* stream) {
  return guarded([&] {
    check(nx >= 1 && ny >= 1 && nz >= 1, "tv_loss needs a non-scalar input");
    check((d_x_out == nullptr) == (d_grad == nullptr), "tv_step: x_out and grad go together");
    check(d_x_out == nullptr || d_x_out != d_x, "tv_step: x_out must not alias x");
    const cudaStream_t st = as_stream(stream);
    iter::Scratch sc(st);
    iter::tv_step(d_x, d_grad, iter::one_out(d_x_out), nx, ny, nz, has_lo != 0, has_hi != 0,
                  tv_lambda, learning_rate, d_tv, st, sc);
  });
}

tg_status tg_tv_grad(const float* d_x, float* d_gx, uint64_t nx, uint64_t ny, uint64_t nz,
                     double gs, double* d_tv, void* stream) {
  return guarded([&] {
    check(nx >= 1 && ny >= 1 && nz >= 1, "tv_loss needs a non-scalar input");
    check(d_gx != nullptr && d_gx != d_x, "tv_grad: the gradient must not alias x");
    const cudaStream_t st = as_stream(stream);
    iter::Scratch sc(st);
    iter::tv_grad_kernel<<<iter::kRedBlocks, iter::kRedThreads, 0, st>>>(
        d_x, d_gx, int(nx), int(ny), int(nz), gs, sc.partial);
    iter::sum_partials_kernel<<<1, iter::kRedThreads, 0, st>>>(sc.partial, iter::kRedBlocks,
                                                               d_tv);
    TG_LAUNCHED(2);
  });
}

tg_status tg_l2_grad(const float* d_a, const float* d_b, float* d_ga, float* d_gb, uint64_t n,
                     double gs, void* stream) {
  return guarded([&] {
    if (n == 0 || (!d_ga && !d_gb)) return;
    const cudaStream_t st = as_stream(stream);
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148 * 16);
    iter::l2_grad_kernel<<<unsigned(blocks), 256, 0, st>>>(d_a, d_b, d_ga, d_gb, n, 2.0 * gs);
    TG_LAUNCHED(1);
  });
}

tg_status tg_tv_step_multi(const float* d_x, const float* d_grad, float* const* d_x_outs, int n_out,
                           uint64_t nx, uint64_t ny, uint64_t nz, int has_lo, int has_hi,
                           double tv_lambda, double learning_rate, double* d_tv, void* stream) {
  return guarded([&] {
    check(nx >= 1 && ny >= 1 && nz >= 1, "tv_loss needs a non-scalar input");
    check(n_out >= 1 && n_out <= iter::kMaxDest && d_grad != nullptr,
          "tv_step_multi: 1..16 destinations and a gradient");
    iter::OutList o;
    o.n = n_out;
    for (int d = 0; d < n_out; ++d) {
      check(d_x_outs[d] != nullptr && d_x_outs[d] != d_x, "tv_step: x_out must not alias x");
      o.p[d] = d_x_outs[d];
    }
    const cudaStream_t st = as_stream(stream);
    iter::Scratch sc(st);
    iter::tv_step(d_x, d_grad, o, nx, ny, nz, has_lo != 0, has_hi != 0, tv_lambda, learning_rate,
                  d_tv, st, sc);
  });
}

tg_status tg_l2_residual_scatter(const float* d_fp, const float* d_p, uint64_t n_views,
                                 uint64_t n_v, uint64_t n_u, uint64_t view0,
                                 const tg_band_dest* dests, int n_dests, double* d_sum,
                                 void* stream) {
  return guarded([&] {
    check(n_views >= 1 && n_v >= 1 && n_u >= 1, "l2_loss expects matching shapes");
    check(n_dests >= 1 && n_dests <= iter::kMaxDest, "residual scatter: 1..16 destinations");
    iter::BandList b;
    b.n = n_dests;
    for (int d = 0; d < n_dests; ++d) {
      check(dests[d].band != nullptr && dests[d].v0 + dests[d].n_rows <= n_v,
            "detector row band lies outside the detector");
      b.p[d] = dests[d].band;
      b.v0[d] = int(dests[d].v0);
      b.n_rows[d] = int(dests[d].n_rows);
    }
    const cudaStream_t st = as_stream(stream);
    iter::Scratch sc(st);
    iter::l2_scatter_kernel<<<iter::kRedBlocks, iter::kRedThreads, 0, st>>>(
        d_fp, d_p, n_views * n_v * n_u, int(n_v), int(n_u), int(view0), b, sc.partial);
    iter::sum_partials_kernel<<<1, iter::kRedThreads, 0, st>>>(sc.partial, iter::kRedBlocks, d_sum);
    TG_LAUNCHED(2);
  });
}

tg_status tg_cone_tv_reconstruct_host(tg_cone_plan* plan, const float* h_sino, float* h_x,
                                      uint64_t iterations, double learning_rate, double tv_lambda,
                                      double* h_loss_history) {
  tg_volume_spec vol;
  tg_detector2d det;
  uint64_t n_proj = 0;
  const tg_status s0 = tg_cone_plan_shape(plan, &vol, &det, &n_proj);
  if (s0 != TG_OK) return s0;
  int dev = 0;
  cudaGetDevice(&dev);
  return iter::tv_host(dev, n_proj * det.n_u * det.n_v, vol.shape[0] * vol.shape[1] * vol.shape[2],
                 h_sino, h_x, [&](const float* s, float* x, cudaStream_t st) {
                   return tg_cone_tv_reconstruct(plan, s, x, iterations, learning_rate, tv_lambda,
                                                 h_loss_history, st);
                 });
}

tg_status tg_planar_tv_reconstruct_host(tg_planar_plan* plan, const float* h_sino, float* h_x,
                                        uint64_t iterations, double learning_rate,
                                        double tv_lambda, double* h_loss_history) {
  tg_volume_spec vol;
  tg_detector1d det;
  uint64_t n_proj = 0;
  const tg_status s0 = tg_planar_plan_shape(plan, &vol, &det, &n_proj);
  if (s0 != TG_OK) return s0;
  int dev = 0;
  cudaGetDevice(&dev);
  return iter::tv_host(dev, n_proj * det.n_bins, vol.shape[0] * vol.shape[1], h_sino, h_x,
                 [&](const float* s, float* x, cudaStream_t st) {
                   return tg_planar_tv_reconstruct(plan, s, x, iterations, learning_rate,
                                                   tv_lambda, h_loss_history, st);
                 });
}

// ---- peer memory (CUDA IPC) for the fused multi-GPU exchanges -------------

tg_status tg_device_alloc(uint64_t bytes, int device, void** d_ptr) {
  return guarded([&] {
    DeviceGuard dg(device);
    *d_ptr = nullptr;
    TG_CUDA(cudaMalloc(d_ptr, bytes));
    TG_CUDA(cudaMemset(*d_ptr, 0, bytes));
  });
}

tg_status tg_device_free(void* d_ptr) {
  return guarded([&] { TG_CUDA(cudaFree(d_ptr)); });
}

tg_status tg_ipc_get_handle(const void* d_base, unsigned char* out64) {
  return guarded([&] {
    cudaIpcMemHandle_t h;
    TG_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_base)));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(out64, &h, 64);
  });
}

tg_status tg_ipc_open_handle(const unsigned char* in64, int device, void** d_ptr) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, in64, 64);
    TG_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

tg_status tg_ipc_close_handle(void* d_ptr) {
  return guarded([&] { TG_CUDA(cudaIpcCloseMemHandle(d_ptr)); });
}

tg_status tg_cone_tv_reconstruct(tg_cone_plan* plan, const float* d_sino, float* d_x,
                                 uint64_t iterations, double learning_rate, double tv_lambda,
                                 double* h_loss_history, void* stream) {
  return guarded([&] {
    const cudaStream_t st = as_stream(stream);
    tg_volume_spec vol;
    tg_detector2d det;
    uint64_t n_proj = 0;
    tg_cone_plan_shape(plan, &vol, &det, &n_proj);
    auto ok = [](tg_status s) {
      if (s != TG_OK) throw RefError(tg_last_error());
    };
    iter::tv_loop(
        [&](const float* x, float* s, cudaStream_t q) { ok(tg_cone_forward(plan, x, s, q)); },
        [&](const float* s, float* x, cudaStream_t q) {
          ok(tg_cone_backproject(plan, s, x, 1.0f, 0, q));
        },
                  n_proj * det.n_u * det.n_v, vol.shape[0], vol.shape[1], vol.shape[2], d_sino,
                  d_x, iterations, learning_rate, tv_lambda, h_loss_history, st);
  });
}

tg_status tg_planar_learn_filter(tg_planar_plan* plan, const float* d_sino, const float* d_target,
                                 float* d_k, uint64_t P, const double* h_init,
                                 const double* h_ramlak, double learning_rate, uint64_t iterations,
                                 double* h_loss, double* h_dist, float* d_recon, void* stream) {
  return guarded([&] {
    const cudaStream_t st = as_stream(stream);
    tg_volume_spec vol;
    tg_detector1d det;
    uint64_t n_proj = 0;
    tg_planar_plan_shape(plan, &vol, &det, &n_proj);
    auto ok = [](tg_status s) {
      if (s != TG_OK) throw RefError(tg_last_error());
    };
    // graph: scale(backproject(.), pi / n_projections) (pipelines.hpp:228-229)
    const double factor = kPi / double(n_proj);
    iter::learn_filter_loop(
        [&](const float* x, float* s, cudaStream_t q) { ok(tg_planar_forward(plan, x, s, q)); },
        [&](const float* s, float* x, float scale, cudaStream_t q) {
          ok(tg_planar_backproject(plan, s, x, scale, 0, q));
        },
        n_proj, det.n_bins, vol.shape[0] * vol.shape[1], d_sino, d_target, d_k, P, h_init,
        h_ramlak, learning_rate, iterations, factor, h_loss, h_dist, d_recon, st);
  });
}

tg_status tg_planar_learn_filter_host(tg_planar_plan* plan, const float* h_sino,
                                      const float* h_target, float* h_k, uint64_t P,
                                      const double* h_init, const double* h_ramlak,
                                      double learning_rate, uint64_t iterations, double* h_loss,
                                      double* h_dist, float* h_recon) {
  return guarded([&] {
    tg_volume_spec vol;
    tg_detector1d det;
    uint64_t n_proj = 0;
    if (tg_planar_plan_shape(plan, &vol, &det, &n_proj) != TG_OK) throw RefError(tg_last_error());
    const uint64_t n_sino = n_proj * det.n_bins, n_vox = vol.shape[0] * vol.shape[1];
    cudaStream_t st;
    TG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    tg_status r = TG_OK;
    std::string msg;
    {
      iter::AsyncBuf<float> s(n_sino, st), t(n_vox, st), k(P, st), rec(n_vox, st);
      TG_CUDA(cudaMemcpyAsync(s.p, h_sino, n_sino * sizeof(float), cudaMemcpyHostToDevice, st));
      TG_CUDA(cudaMemcpyAsync(t.p, h_target, n_vox * sizeof(float), cudaMemcpyHostToDevice, st));
      TG_CUDA(cudaMemcpyAsync(k.p, h_k, P * sizeof(float), cudaMemcpyHostToDevice, st));
      r = tg_planar_learn_filter(plan, s.p, t.p, k.p, P, h_init, h_ramlak, learning_rate,
                                 iterations, h_loss, h_dist, h_recon ? rec.p : nullptr, st);
      if (r == TG_OK) {
        TG_CUDA(cudaMemcpyAsync(h_k, k.p, P * sizeof(float), cudaMemcpyDeviceToHost, st));
        if (h_recon)
          TG_CUDA(cudaMemcpyAsync(h_recon, rec.p, n_vox * sizeof(float), cudaMemcpyDeviceToHost,
                                  st));
      } else {
        msg = tg_last_error();
      }
    }
    TG_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    if (r != TG_OK) throw RefError(msg);
  });
}

tg_status tg_planar_tv_reconstruct(tg_planar_plan* plan, const float* d_sino, float* d_x,
                                   uint64_t iterations, double learning_rate, double tv_lambda,
                                   double* h_loss_history, void* stream) {
  return guarded([&] {
    const cudaStream_t st = as_stream(stream);
    tg_volume_spec vol;
    tg_detector1d det;
    uint64_t n_proj = 0;
    tg_planar_plan_shape(plan, &vol, &det, &n_proj);
    auto ok = [](tg_status s) {
      if (s != TG_OK) throw RefError(tg_last_error());
    };
    // the planar pair is graph-capturable (K4/K6 build their view maps from
    // the plan's FP64 ray table; no constant-bank upload)
    iter::tv_loop(
        [&](const float* x, float* s, cudaStream_t q) { ok(tg_planar_forward(plan, x, s, q)); },
        [&](const float* s, float* x, cudaStream_t q) {
          ok(tg_planar_backproject(plan, s, x, 1.0f, 0, q));
        },
        n_proj * det.n_bins, vol.shape[0], vol.shape[1], 1, d_sino, d_x, iterations,
        learning_rate, tv_lambda, h_loss_history, st, true);
  });
}

}  // extern "C"
