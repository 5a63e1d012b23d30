// filter.cu — K3 row filter: register-resident radix-16 Stockham FFT
// (fft16.cuh), two real rows per complex transform when the weights are
// symmetric, FDK pre-weights, fused truncation.
//
// The reference (filtering.hpp:95-110) zero-pads each row to P, runs a
// complex-double FFT, multiplies by the real weights, inverse-transforms
// and keeps the first n samples.  This kernel computes the same linear map
// in fp32 with FP64-derived twiddles; the parity tolerance is stated in
// tests/_helpers.py (REL_RMSE / FILTER_REL_RMSE) and exercised by
// tests/test_gpu_fdk.py and tests/test_gpu_fullsize.py.
#include <cstdlib>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "fft16.cuh"
#include "filter.cuh"

namespace tgb {
namespace filt {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 conj_if(float2 a, bool inv) { return inv ? make_float2(a.x, -a.y) : a; }

// One Stockham pass set over smem buffers x <-> y; returns the buffer holding
// the result.  Twiddles w_P(m) = exp(-2 pi i m / P); the inverse conjugates.
__device__ float2* fft_smem(float2* x, float2* y, int P, const float2* __restrict__ tw, bool inv) {
  int Ns = 1;
  const int q = P >> 2;
  while (Ns * 4 <= P) {
    for (int j = threadIdx.x; j < q; j += blockDim.x) {
      const int k = j & (Ns - 1);
      float2 v0 = x[j], v1 = x[j + q], v2 = x[j + 2 * q], v3 = x[j + 3 * q];
      if (Ns > 1) {
        const int m = k * (P / (4 * Ns));
        v1 = cmul(v1, conj_if(__ldg(tw + m), inv));
        v2 = cmul(v2, conj_if(__ldg(tw + 2 * m), inv));
        v3 = cmul(v3, conj_if(__ldg(tw + 3 * m), inv));
      }
      const float2 a0 = cadd(v0, v2), a1 = csub(v0, v2), a2 = cadd(v1, v3);
      const float2 d = csub(v1, v3);
      // forward: -i*d, inverse: +i*d
      const float2 a3 = inv ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
      const int o = (j - k) * 4 + k;
      y[o] = cadd(a0, a2);
      y[o + Ns] = cadd(a1, a3);
      y[o + 2 * Ns] = csub(a0, a2);
      y[o + 3 * Ns] = csub(a1, a3);
    }
    __syncthreads();
    float2* t = x;
    x = y;
    y = t;
    Ns *= 4;
  }
  if (Ns < P) {  // radix-2 tail, Ns == P / 2
    const int h = P >> 1;
    for (int j = threadIdx.x; j < h; j += blockDim.x) {
      const float2 v0 = x[j];
      const float2 v1 = cmul(x[j + h], conj_if(__ldg(tw + j), inv));
      y[j] = cadd(v0, v1);
      y[j + h] = csub(v0, v1);
    }
    __syncthreads();
    x = y;
  }
  return x;
}

__device__ __forceinline__ float pre_weight(float v, const PreWeights& pw, uint64_t row, int j,
                                            int n) {
  if (pw.cos) {
    const uint64_t vrow = pw.cos_row0 + row % pw.rows_per_view;
    v = float(double(v) * __ldg(pw.cos + vrow * n + j));
  }
  if (pw.parker) {
    const uint64_t view = row / pw.rows_per_view;
    v = float(double(v) * __ldg(pw.parker + view * n + j));
  }
  return v;
}

// blockIdx.x -> rows (2b, 2b+1) when packed, row b otherwise
__global__ void __launch_bounds__(kThreads) row_filter_kernel(const float* in, float* out, int n,
                                                             int P, uint64_t n_rows, bool packed,
                                                             const float* __restrict__ w,
                                                             const float2* __restrict__ tw,
                                                             PreWeights pw) {
  extern __shared__ float2 buf[];
  float2* x = buf;
  float2* y = buf + P;
  const uint64_t ra = packed ? 2 * uint64_t(blockIdx.x) : uint64_t(blockIdx.x);
  const bool has_b = packed && ra + 1 < n_rows;
  const float* pa = in + ra * uint64_t(n);
  const float* pb = in + (ra + 1) * uint64_t(n);
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    float2 z = make_float2(0.f, 0.f);
    if (j < n) {
      z.x = pre_weight(pa[j], pw, ra, j, n);
      if (has_b) z.y = pre_weight(pb[j], pw, ra + 1, j, n);
    }
    x[j] = z;
  }
  __syncthreads();
  float2* X = fft_smem(x, y, P, tw, false);
  float2* other = (X == x) ? y : x;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const float wk = __ldg(w + k);
    X[k] = make_float2(X[k].x * wk, X[k].y * wk);
  }
  __syncthreads();
  float2* Z = fft_smem(X, other, P, tw, true);
  const float inv = 1.0f / float(P);
  float* oa = out + ra * uint64_t(n);
  float* ob = out + (ra + 1) * uint64_t(n);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    oa[j] = Z[j].x * inv;
    if (has_b) ob[j] = Z[j].y * inv;
  }
}

__global__ void apply_weights_kernel(const float* in, float* out, uint64_t n, const double* map,
                                     uint64_t map_n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = float(double(in[i]) * __ldg(map + i % map_n));
}

__global__ void apply_row_weights_kernel(const float* in, float* out, uint64_t total,
                                         uint64_t n_rows, uint64_t n, const double* map) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t view = i / (n_rows * n), j = i % n;
    out[i] = float(double(in[i]) * __ldg(map + view * n + j));
  }
}

}  // namespace

RowFilter* create(uint64_t n, uint64_t P, const double* weights, int device) {
  check(P >= 2 && is_pow2(P), "filter window must be a power of two");
  check(P <= 8192, "filter window exceeds the device filter's 8192-sample limit");
  auto f = std::make_unique<RowFilter>();
  f->device = device;
  f->n = n;
  f->P = P;
  // filter_rows keeps Re(IFFT(W X)) of a real row (filtering.hpp:104-107),
  // which equals IFFT(W_s X) with the symmetrised weights
  // W_s[k] = (W[k] + W[P-k]) / 2 for any real W.  Symmetrising in FP64 makes
  // every filter eligible for the two-rows-per-complex-FFT packing; without
  // it the Ram-Lak window, symmetric in exact arithmetic but not bitwise after
  // its FP64 FFT, fell back to one row per transform (2x the K3 work).
  f->symmetric = true;
  std::vector<float> w(P);
  // same rounding as symmetrize_kernel (the graph's trainable weights): the
  // fp32 weights averaged in FP64
  for (uint64_t k = 0; k < P; ++k)
    w[k] = float(0.5 * (double(float(weights[k])) + double(float(weights[(P - k) & (P - 1)]))));
  std::vector<float2> tw(P);
  for (uint64_t k = 0; k < P; ++k) {
    const double ang = -2.0 * kPi * double(k) / double(P);
    tw[k] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
  }
  DeviceGuard dg(device);
  TG_CUDA(cudaMalloc(&f->d_w, P * sizeof(float)));
  TG_CUDA(cudaMalloc(&f->d_tw, P * sizeof(float2)));
  TG_CUDA(cudaMemcpy(f->d_w, w.data(), P * sizeof(float), cudaMemcpyHostToDevice));
  TG_CUDA(cudaMemcpy(f->d_tw, tw.data(), P * sizeof(float2), cudaMemcpyHostToDevice));
  std::vector<float2> t16;
  switch (P) {
    case 512: t16 = fft16::make_tw_table<512>(); break;
    case 1024: t16 = fft16::make_tw_table<1024>(); break;
    case 2048: t16 = fft16::make_tw_table<2048>(); break;
    case 4096: t16 = fft16::make_tw_table<4096>(); break;
    case 8192: t16 = fft16::make_tw_table<8192>(); break;
    default: break;
  }
  if (!t16.empty()) {
    TG_CUDA(cudaMalloc(&f->d_tw16, t16.size() * sizeof(float2)));
    TG_CUDA(cudaMemcpy(f->d_tw16, t16.data(), t16.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  return f.release();
}

void destroy(RowFilter* f) {
  if (!f) return;
  cudaFree(f->d_w);
  cudaFree(f->d_tw);
  cudaFree(f->d_tw16);
  delete f;
}

// FDK pre-weights as one elementwise pass: one warp per detector row (no
// per-element index division; 8 rows per CTA); the FP64
// products and their two fp32 roundings are the reference's
// (filtering.hpp:136-154, applied cosine then Parker).
constexpr int kPwRows = 8;
__global__ void __launch_bounds__(32 * kPwRows) preweight_kernel(const float* in, float* out, int n,
                                                                 uint64_t n_rows, PreWeights pw,
                                                                 RowLayout lay) {
  // (PDL launches) the grid completes only after the stream's previous kernel
  struct WaitPrev {
    __device__ ~WaitPrev() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
  } wait_prev;
  const uint64_t row = uint64_t(blockIdx.x) * kPwRows + (threadIdx.x >> 5);
  if (row >= n_rows) return;
  const int lane = threadIdx.x & 31;
  const float* src = in + row_offset(row, n, lay);
  float* dst = out + row_offset(row, n, lay);
  const double* cw = pw.cos ? pw.cos + (pw.cos_row0 + row % pw.rows_per_view) * uint64_t(n) : nullptr;
  const double* pk = pw.parker ? pw.parker + (row / pw.rows_per_view) * uint64_t(n) : nullptr;
  auto weigh = [&](float v, int j) {
    if (cw) v = float(double(v) * __ldg(cw + j));
    if (pk) v = float(double(v) * __ldg(pk + j));
    return v;
  };
  // lane j of every 32: the FP64 weight rows are read as 256-byte warp
  // segments (2 L1 wavefronts per 32 elements; per-lane float4 with 32-byte
  // lane strides cost 8 per instruction: 4.35 -> 4.23 ms for K3 at c4), four
  // elements in flight per lane
  int j = lane;
  for (; j + 96 < n; j += 128) {
    const float a0 = __ldcs(src + j), a1 = __ldcs(src + j + 32), a2 = __ldcs(src + j + 64),
                a3 = __ldcs(src + j + 96);
    __stcs(dst + j, weigh(a0, j));
    __stcs(dst + j + 32, weigh(a1, j + 32));
    __stcs(dst + j + 64, weigh(a2, j + 64));
    __stcs(dst + j + 96, weigh(a3, j + 96));
  }
  for (; j < n; j += 32) __stcs(dst + j, weigh(__ldcs(src + j), j));
}

void apply(const RowFilter& f, const float* d_in, float* d_out, uint64_t n_rows,
           const PreWeights* pw, cudaStream_t st, RowLayout lay, bool pdl) {
  if (n_rows == 0) return;
  DeviceGuard dg(f.device);
  PreWeights w = pw ? *pw : PreWeights{};
  check(lay.rows_per_view == 0 || (f.P >= 512 && f.P <= 8192),
        "strided row layouts need a filter window in [512, 8192]");
  const bool packed = f.symmetric;
  const uint64_t blocks = packed ? (n_rows + 1) / 2 : n_rows;
  check(blocks <= 2147483647ull, "too many detector rows for one filter launch");
  KernelTimer timer;
  timer.start(st);
  const int n = int(f.n);
  // The FP64 cosine / Parker pre-weights run as their own elementwise pass
  // (HBM-bound, exact double products rounded to fp32 per map) so the FFT
  // kernel keeps its registers for the transform (P = 4096: 3 CTAs / SM).
  const bool sep = (w.cos || w.parker) && f.P >= 512 && f.P <= 8192;
  const float* src = d_in;
  if (sep) {
    check(n_rows <= 2147483647ull, "too many detector rows for one filter launch");
    const uint64_t pw_blocks = (n_rows + kPwRows - 1) / kPwRows;
    check(pw_blocks <= 2147483647ull, "too many detector rows for one filter launch");
    if (pdl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(unsigned(pw_blocks));
      cfg.blockDim = dim3(32 * kPwRows);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      TG_CUDA(cudaLaunchKernelEx(&cfg, preweight_kernel, d_in, d_out, n, n_rows, w, lay));
    } else {
      preweight_kernel<<<unsigned(pw_blocks), 32 * kPwRows, 0, st>>>(d_in, d_out, n, n_rows, w, lay);
    }
    TG_LAUNCHED(1);
    src = d_out;
    w = PreWeights{};
  }
  auto launch16 = [&](auto kern, int P, size_t smem) {
    TG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<unsigned(blocks), P / 16, smem, st>>>(src, d_out, n, n_rows, int(packed), f.d_w, f.d_tw16,
                                                  w, lay);
  };
  const bool half = 2 * f.n <= f.P;  // the row fills at most half the window
  // rows of at most 1280 samples (c4's 1248) in the 4096 window: NZR = 5
  // pruned first / last passes (4.45 -> 4.36 ms for c4's band)
  if (f.P == 4096 && f.n <= 5 * 256) {
    launch16(fft16::filter_kernel<4096, false, true, 5>, 4096, fft16::smem_bytes<4096>());
    TG_LAUNCHED(1);
    timer.stop();
    return;
  }
#define TG_LAUNCH16(PP)                                                                   \
  case PP:                                                                                \
    if (half)                                                                             \
      launch16(fft16::filter_kernel<PP, false, true>, PP, fft16::smem_bytes<PP>());       \
    else                                                                                  \
      launch16(fft16::filter_kernel<PP, false, false>, PP, fft16::smem_bytes<PP>());      \
    break;
  switch (f.P) {
    TG_LAUNCH16(512)
    TG_LAUNCH16(1024)
    TG_LAUNCH16(2048)
    TG_LAUNCH16(4096)
    TG_LAUNCH16(8192)
#undef TG_LAUNCH16
    default: {  // small windows: generic radix-4 shared-memory transform
      const size_t smem = 2 * f.P * sizeof(float2);
      TG_CUDA(cudaFuncSetAttribute(row_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
      row_filter_kernel<<<unsigned(blocks), kThreads, smem, st>>>(d_in, d_out, n, int(f.P), n_rows,
                                                                  packed, f.d_w, f.d_tw, w);
    }
  }
  TG_LAUNCHED(1);
  timer.stop();
}

// ---- graph fourier_filter node with device-resident (trainable) weights ----
// graph.hpp:152-164 / 312-316 forward, 470-497 gradients.
//
// Re(IFFT(k X)) of a real row equals IFFT(k_s X) with the symmetrised
// weights k_s[f] = (k[f] + k[P-f]) / 2 (the antisymmetric part only feeds the
// discarded imaginary part), so every call takes the packed two-rows-per-FFT
// path of K3 whatever the weights are.
__global__ void symmetrize_kernel(const float* __restrict__ k, float* __restrict__ ks, int P) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < P; f += gridDim.x * blockDim.x)
    ks[f] = float(0.5 * (double(k[f]) + double(k[(P - f) & (P - 1)])));
}

// d loss / d k_f = sum over rows Re(X_f conj(G_f)) / P (graph.hpp:478-496).
// One complex FFT per row pairs x (real part) with g (imaginary part):
// X_f = (Z_f + conj Z_{P-f}) / 2, G_f = (Z_f - conj Z_{P-f}) / (2i).
// Each CTA walks rows blockIdx.x, +gridDim.x, ... and keeps per-frequency
// FP64 sums in shared memory; partial[cta][f] are reduced in a fixed order.
__global__ void __launch_bounds__(kThreads) filter_weight_grad_kernel(
    const float* __restrict__ x, const float* __restrict__ g, int n, int P, uint64_t n_rows,
    const float2* __restrict__ tw, double* __restrict__ partial) {
  extern __shared__ float2 buf[];
  float2* zx = buf;
  float2* zy = buf + P;
  double* acc = reinterpret_cast<double*>(buf + 2 * P);
  for (int f = threadIdx.x; f < P; f += blockDim.x) acc[f] = 0.0;
  for (uint64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const float* xr = x + r * uint64_t(n);
    const float* gr = g + r * uint64_t(n);
    for (int j = threadIdx.x; j < P; j += blockDim.x)
      zx[j] = j < n ? make_float2(xr[j], gr[j]) : make_float2(0.f, 0.f);
    __syncthreads();
    const float2* Z = fft_smem(zx, zy, P, tw, false);
    for (int f = threadIdx.x; f < P; f += blockDim.x) {
      const float2 a = Z[f];
      const float2 c = Z[(P - f) & (P - 1)];  // b = conj(c)
      const double xr_ = 0.5 * (double(a.x) + double(c.x)), xi_ = 0.5 * (double(a.y) - double(c.y));
      const double dr = double(a.x) - double(c.x), di = double(a.y) + double(c.y);
      const double gr_ = 0.5 * di, gi_ = -0.5 * dr;  // (a - b) / (2i)
      acc[f] += xr_ * gr_ + xi_ * gi_;
    }
    __syncthreads();  // the next row reuses the buffers
  }
  for (int f = threadIdx.x; f < P; f += blockDim.x) partial[uint64_t(blockIdx.x) * P + f] = acc[f];
}

__global__ void filter_weight_grad_reduce(const double* __restrict__ partial, int parts, int P,
                                          double inv_p, float* gk, int accumulate) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < P; f += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < parts; ++c) s += partial[uint64_t(c) * P + f];
    gk[f] = accumulate ? float(double(gk[f]) + inv_p * s) : float(inv_p * s);
  }
}

// per-(device, P) twiddle tables, built once and kept for the process
const RowFilter& tables(int device, uint64_t P) {
  static std::mutex mu;
  static std::map<std::pair<int, uint64_t>, RowFilter*> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({device, P});
  if (it != cache.end()) return *it->second;
  std::vector<double> ones(P, 1.0);
  RowFilter* f = create(P, P, ones.data(), device);
  cache[{device, P}] = f;
  return *f;
}

void check_fourier(uint64_t n, uint64_t P) {
  // graph.hpp:156-161 in the reference's order
  check(n >= 1, "fourier_filter input must have at least one axis");
  check(is_pow2(P), "filter window must be a power of two");
  check(P >= n, "filter window is smaller than the detector row");
  check(P <= 8192, "filter window exceeds the device filter's 8192-sample limit");
}

void fourier_filter(const float* d_x, const float* d_k, float* d_ks, float* d_out,
                    uint64_t n_rows, uint64_t n, uint64_t P, cudaStream_t st) {
  check_fourier(n, P);
  if (n_rows == 0) return;
  int dev = 0;
  TG_CUDA(cudaGetDevice(&dev));
  RowFilter f = tables(dev, P);
  f.n = n;
  f.symmetric = true;
  symmetrize_kernel<<<unsigned((P + 255) / 256), 256, 0, st>>>(d_k, d_ks, int(P));
  TG_LAUNCHED(1);
  f.d_w = d_ks;
  apply(f, d_x, d_out, n_rows, nullptr, st);
}

int weight_grad_parts(uint64_t n_rows) { return int(std::min<uint64_t>(n_rows, 2 * 148)); }

void weight_grad(const float* d_x, const float* d_g, float* d_gk, double* d_partial,
                 uint64_t n_rows, uint64_t n, uint64_t P, bool accumulate, cudaStream_t st) {
  check_fourier(n, P);
  if (n_rows == 0) return;
  int dev = 0;
  TG_CUDA(cudaGetDevice(&dev));
  const RowFilter& f = tables(dev, P);
  const int parts = weight_grad_parts(n_rows);
  const size_t smem = 2 * P * sizeof(float2) + P * sizeof(double);
  TG_CUDA(cudaFuncSetAttribute(filter_weight_grad_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  filter_weight_grad_kernel<<<parts, 256, smem, st>>>(d_x, d_g, int(n), int(P), n_rows, f.d_tw,
                                                      d_partial);
  filter_weight_grad_reduce<<<unsigned((P + 255) / 256), 256, 0, st>>>(
      d_partial, parts, int(P), 1.0 / double(P), d_gk, int(accumulate));
  TG_LAUNCHED(2);
}

}  // namespace filt
}  // namespace tgb

// ---------------------------------------------------------------------------
// C ABI

using namespace tgb;

struct tg_filter_plan {
  filt::RowFilter* f = nullptr;
};

extern "C" {

tg_status tg_filter_plan_create(uint64_t row_len, double row_spacing, uint64_t filt_n_bins,
                                uint64_t padded_n, double filt_spacing, const double* weights,
                                uint64_t n_weights, int device, tg_filter_plan** out) {
  return guarded([&] {
    *out = nullptr;
    // filtering.hpp:117-121 then 97-99, in the reference's order
    check(filt_n_bins == row_len, "filter was built for a different detector width");
    check(std::abs(filt_spacing - row_spacing) <= 1e-12 * std::max(1.0, std::abs(row_spacing)),
          "filter spacing does not match the detector spacing");
    check(n_weights == padded_n && is_pow2(padded_n),
          "filter window is inconsistent with its weight vector");
    check(padded_n >= row_len, "filter window is smaller than the detector row");
    auto p = std::make_unique<tg_filter_plan>();
    p->f = filt::create(row_len, padded_n, weights, device);
    *out = p.release();
  });
}

tg_status tg_filter_plan_destroy(tg_filter_plan* p) {
  return guarded([&] {
    if (!p) return;
    filt::destroy(p->f);
    delete p;
  });
}

tg_status tg_filter_apply(tg_filter_plan* p, const float* d_in, float* d_out, uint64_t n_rows,
                          void* stream) {
  return guarded([&] { filt::apply(*p->f, d_in, d_out, n_rows, nullptr, as_stream(stream)); });
}

tg_status tg_filter_apply_host(tg_filter_plan* p, const float* h_in, float* h_out, uint64_t n_rows) {
  return guarded([&] {
    DeviceGuard dg(p->f->device);
    const size_t bytes = n_rows * p->f->n * sizeof(float);
    float* d = nullptr;
    TG_CUDA(cudaMalloc(&d, bytes ? bytes : 4));
    TG_CUDA(cudaMemcpy(d, h_in, bytes, cudaMemcpyHostToDevice));
    filt::apply(*p->f, d, d, n_rows, nullptr, 0);
    TG_CUDA(cudaMemcpy(h_out, d, bytes, cudaMemcpyDeviceToHost));
    TG_CUDA(cudaFree(d));
  });
}

tg_status tg_apply_weights(const float* d_in, float* d_out, uint64_t n_total, const double* d_map,
                           uint64_t map_n, void* stream) {
  return guarded([&] {
    check(map_n >= 1, "weight map shape matches neither the sinogram nor its detector");
    if (n_total == 0) return;
    const uint64_t blocks = std::min<uint64_t>((n_total + 255) / 256, 148 * 32);
    filt::apply_weights_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(d_in, d_out, n_total, d_map,
                                                                         map_n);
    TG_LAUNCHED(1);
  });
}

tg_status tg_apply_row_weights(const float* d_in, float* d_out, uint64_t n_views, uint64_t n_rows,
                               uint64_t n, const double* d_map, void* stream) {
  return guarded([&] {
    const uint64_t total = n_views * n_rows * n;
    if (total == 0) return;
    const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148 * 32);
    filt::apply_row_weights_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(
        d_in, d_out, total, n_rows, n, d_map);
    TG_LAUNCHED(1);
  });
}

/* graph fourier_filter node: rows of n at window P, device weights k[P] */
tg_status tg_fourier_filter(const float* d_x, const float* d_k, float* d_out, uint64_t n_rows,
                            uint64_t n, uint64_t P, void* stream) {
  return guarded([&] {
    filt::check_fourier(n, P);
    if (n_rows == 0) return;
    const cudaStream_t st = as_stream(stream);
    float* ks = nullptr;
    TG_CUDA(cudaMallocAsync(&ks, P * sizeof(float), st));
    filt::fourier_filter(d_x, d_k, ks, d_out, n_rows, n, P, st);
    TG_CUDA(cudaFreeAsync(ks, st));
  });
}

tg_status tg_fourier_filter_weight_grad(const float* d_x, const float* d_g, float* d_gk,
                                        uint64_t n_rows, uint64_t n, uint64_t P, void* stream) {
  return guarded([&] {
    filt::check_fourier(n, P);
    if (n_rows == 0) return;
    const cudaStream_t st = as_stream(stream);
    double* partial = nullptr;
    TG_CUDA(cudaMallocAsync(&partial, sizeof(double) * P * filt::weight_grad_parts(n_rows), st));
    filt::weight_grad(d_x, d_g, d_gk, partial, n_rows, n, P, true, st);
    TG_CUDA(cudaFreeAsync(partial, st));
  });
}

}  // extern "C"
