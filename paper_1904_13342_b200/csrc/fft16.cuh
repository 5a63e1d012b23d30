// fft16.cuh — K3 fast path: register radix-16 Stockham FFT row filter for
// windows P in {512, 1024, 2048, 4096, 8192} (the BASELINE configs use 1024,
// 2048 and 4096).
//
// One CTA transforms one complex row z = a + i b (two real detector rows when
// the filter is symmetric), with P/16 threads each holding 16 complex values
// in registers per pass:
//   forward : [global rows (+ FDK pre-weights) -> R16] -> R16 -> R_last (x W)
//   inverse : R16 -> R16 -> [R_last -> global, first n samples only]
// so the zero-padding load and the truncating store are fused into the
// first / last pass and the filter multiply into the forward's last store.
// Shared memory is indexed with one pad word per 16 entries (bank-conflict
// free radix-16 stores).  Twiddles come from an FP64-derived table.
#pragma once

#include <cmath>
#include <vector>

#include "filter.cuh"

namespace tgb {
namespace filt {
namespace fft16 {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 operator-(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 rot(float2 d) {
  return INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
  const float2 t0 = v0 + v2, t1 = v0 - v2, t2 = v1 + v3, t3 = rot<INV>(v1 - v3);
  v0 = t0 + t2;
  v1 = t1 + t3;
  v2 = t0 - t2;
  v3 = t1 - t3;
}

// cos / sin of 2 pi m / 16 for m = 0..15 (exact decimal expansions)
__host__ __device__ constexpr float cos16(int m) {
  constexpr float c[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                           0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                           -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                           0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
  return c[m & 15];
}
__host__ __device__ constexpr float sin16(int m) { return cos16(m - 4); }

// W_R^m = exp(-+ 2 pi i m / R) for R | 16; m is a compile-time constant after unrolling
template <int R, bool INV>
__device__ __forceinline__ float2 wconst(int m) {
  const int q = m * (16 / R);
  return make_float2(cos16(q), INV ? sin16(q) : -sin16(q));
}

// In-place DFT of length R (2, 4, 8, 16) without temporaries: R = 4 * R2,
// n = R2 n1 + n2, k = k1 + 4 k2.  Four-point transforms over n1 for each n2,
// twiddle W_R^(n2 k1), then R2-point transforms over n2 for each k1.  The
// result X[m] is left in register slot(m) = R2 (m % 4) + m / 4.
template <int R>
__host__ __device__ constexpr int slot(int m) {
  return R <= 4 ? m : (R / 4) * (m % 4) + m / 4;
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 2) {
    const float2 t = v[0];
    v[0] = t + v[1];
    v[1] = t - v[1];
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else {
    constexpr int R2 = R / 4;
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
      dft4<INV>(v[n2], v[R2 + n2], v[2 * R2 + n2], v[3 * R2 + n2]);
      // Y[n2][k1] now sits in v[R2 k1 + n2]
      if (n2) {
        v[R2 + n2] = cmul(v[R2 + n2], wconst<R, INV>(n2));
        v[2 * R2 + n2] = cmul(v[2 * R2 + n2], wconst<R, INV>(2 * n2));
        v[3 * R2 + n2] = cmul(v[3 * R2 + n2], wconst<R, INV>(3 * n2));
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      if constexpr (R2 == 2) {
        const float2 t = v[2 * k1];
        v[2 * k1] = t + v[2 * k1 + 1];
        v[2 * k1 + 1] = t - v[2 * k1 + 1];
      } else {
        dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
      }
    }
  }
}

enum { SRC_SMEM = 0, SRC_GLOBAL = 1 };
enum { DST_SMEM = 0, DST_SMEM_FILTER = 1, DST_GLOBAL = 2 };

struct RowIO {
  const float* pa;
  const float* pb;  // nullptr when the CTA has a single row
  float* oa;
  float* ob;
  int n;
  uint64_t ra;  // launch-relative index of row a (for pre-weights)
  PreWeights pw;
  const float* w;  // filter weights (DST_SMEM_FILTER)
  float out_scale;
};

__device__ __forceinline__ float preweight(float v, const PreWeights& pw, uint64_t row, int j, int n) {
  if (pw.cos) v = float(double(v) * __ldg(pw.cos + (pw.cos_row0 + row % pw.rows_per_view) * n + j));
  if (pw.parker) v = float(double(v) * __ldg(pw.parker + (row / pw.rows_per_view) * n + j));
  return v;
}

// One Stockham radix-R pass (Bainville): butterfly j reads src[j + r P/R],
// twiddles by w_P(r k P/(Ns R)) with k = j mod Ns, writes dst[(j-k) R + k + r Ns].
// HALF: the row occupies at most the first P/2 samples (P >= 2 n, always
// true for the FDK window next_pow2(2 n)): in the first pass inputs r >= R/2
// are zero and in the last pass outputs r >= R/2 are discarded, so the
// compiler prunes that half of the butterfly arithmetic.
// NZR < 16 (P = 4096 only, where the first and the last pass both have radix
// 16 and stride 256): the row occupies the first 256 * NZR samples, so only
// NZR of each first-pass butterfly's inputs are non-zero and only NZR of each
// last-pass butterfly's outputs are kept — the compiler drops the rest of
// the DFT16 arithmetic (c4: 1248 samples, NZR = 5 instead of HALF's 8).
template <int P, int R, bool INV, int SRC, int DST, bool PW = true, bool HALF = false, int NZR = 16>
__device__ __forceinline__ void pass(const float2* __restrict__ x, float2* __restrict__ y, int Ns,
                                     const float2* __restrict__ tw, const RowIO& io) {
  constexpr int NB = P / R;          // butterflies
  constexpr int T = P / 16;          // threads
  constexpr int PER = NB / T;        // butterflies per thread (16 / R)
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = threadIdx.x + q * T;
    const int k = j & (Ns - 1);
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = j + r * NB;
      if constexpr (SRC == SRC_GLOBAL) {
        float2 z = make_float2(0.f, 0.f);
        if ((NZR < 16 ? r < NZR : (!HALF || r < R / 2)) && i < io.n) {
          if (PW) {
            z.x = preweight(io.pa[i], io.pw, io.ra, i, io.n);
            if (io.pb) z.y = preweight(io.pb[i], io.pw, io.ra + 1, i, io.n);
          } else {
            z.x = io.pa[i];
            if (io.pb) z.y = io.pb[i];
          }
        }
        v[r] = z;
      } else {
        v[r] = x[pad(i)];
      }
    }
    if (Ns > 1) {
      // per-pass table [r][k] = w_P(r k P / (Ns R)): consecutive lanes read
      // consecutive entries
#pragma unroll
      for (int r = 1; r < R; ++r) {
        float2 t = __ldg(tw + r * Ns + k);
        if (INV) t.y = -t.y;
        v[r] = cmul(v[r], t);
      }
    }
    dft<R, INV>(v);
    const int o = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = o + r * Ns;
      const float2 x_r = v[slot<R>(r)];
      if constexpr (DST == DST_GLOBAL) {
        if ((NZR < 16 ? r < NZR : (!HALF || r < R / 2)) && i < io.n) {
          io.oa[i] = x_r.x * io.out_scale;
          if (io.ob) io.ob[i] = x_r.y * io.out_scale;
        }
      } else if constexpr (DST == DST_SMEM_FILTER) {
        const float wk = __ldg(io.w + i);
        y[pad(i)] = make_float2(x_r.x * wk, x_r.y * wk);
      } else {
        y[pad(i)] = x_r;
      }
    }
  }
}

// P = 4096 middle: the forward's last radix-16 pass (span 256) leaves thread
// j holding X[j + 256 r], r = 0..15 — exactly the inputs of the inverse's
// first pass (span 1, no twiddles).  Filter multiply and the inverse DFT16
// therefore run in registers: one shared-memory round trip and one barrier
// fewer per row pair.
template <int P>
__device__ __forceinline__ void fused_middle(const float2* __restrict__ x, float2* __restrict__ y,
                                             const float2* __restrict__ tw, const float* __restrict__ w) {
  static_assert(P == 4096, "fused middle pass is specific to P = 4096 (radix 16^3)");
  constexpr int NB = P / 16;
  const int j = threadIdx.x;  // one butterfly per thread (k = j for span 256)
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = x[pad(j + r * NB)];
#pragma unroll
  for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], __ldg(tw + r * 256 + j));
  dft<16, false>(v);
  float2 u[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const float wk = __ldg(w + j + r * NB);
    const float2 xr = v[slot<16>(r)];
    u[r] = make_float2(xr.x * wk, xr.y * wk);
  }
  dft<16, true>(u);
#pragma unroll
  for (int r = 0; r < 16; ++r) y[pad(j * 16 + r)] = u[slot<16>(r)];
}

// offset of the twiddle table of the pass with span Ns (Ns = 16, 256, 4096)
template <int P>
__host__ __device__ constexpr int tw_offset(int Ns) {
  return Ns == 16 ? 0 : (Ns == 256 ? 256 : 256 + 16 * 256);
}
// radix of the pass with span Ns
template <int P>
__host__ __device__ constexpr int radix_at(int Ns) {
  return (P == 8192) ? (Ns == 4096 ? 2 : 16) : (Ns == 256 ? P / 256 : 16);
}
template <int P>
__host__ __device__ constexpr int tw_table_size() {
  return P == 8192 ? 256 + 16 * 256 + 2 * 4096 : 256 + (P / 256) * 256;
}

// occupancy target: 16 resident warps per SM (<= 128 registers per thread);
// without fused pre-weights the P = 4096 transform fits 3 CTAs (24 warps)
template <int P, bool PW>
constexpr int min_blocks() {
  return (!PW && P == 4096) ? 2
                            : ((512 / (P / 16)) < 1 ? 1 : ((512 / (P / 16)) > 16 ? 16 : (512 / (P / 16))));
}

template <int P, bool PW, bool HALF, int NZR = 16>
__global__ void __launch_bounds__(P / 16, (min_blocks<P, PW>())) filter_kernel(const float* in, float* out, int n,
                                                        uint64_t n_rows, int packed,
                                                        const float* __restrict__ w,
                                                        const float2* __restrict__ tw,
                                                        PreWeights pw, RowLayout lay) {
  extern __shared__ float2 sm[];
  constexpr int PADDED = P + P / 16;
  float2* A = sm;
  float2* B = sm + PADDED;
  RowIO io;
  io.ra = packed ? 2 * uint64_t(blockIdx.x) : uint64_t(blockIdx.x);
  const bool has_b = packed && io.ra + 1 < n_rows;
  const uint64_t offa = row_offset(io.ra, n, lay);
  const uint64_t offb = has_b ? row_offset(io.ra + 1, n, lay) : 0;
  io.pa = in + offa;
  io.pb = has_b ? in + offb : nullptr;
  io.oa = out + offa;
  io.ob = has_b ? out + offb : nullptr;
  io.n = n;
  io.pw = pw;
  io.w = w;
  io.out_scale = 1.0f / float(P);
  constexpr int RL = (P == 8192) ? 2 : P / 256;  // last radix
  // forward
  static_assert(NZR == 16 || P == 4096, "pruned passes need P = 4096");
  pass<P, 16, false, SRC_GLOBAL, DST_SMEM, PW, HALF, NZR>(nullptr, A, 1, tw, io);
  __syncthreads();
  if constexpr (P == 8192) {
    pass<P, 16, false, SRC_SMEM, DST_SMEM>(A, B, 16, tw + tw_offset<P>(16), io);
    __syncthreads();
    pass<P, 16, false, SRC_SMEM, DST_SMEM>(B, A, 256, tw + tw_offset<P>(256), io);
    __syncthreads();
    pass<P, 2, false, SRC_SMEM, DST_SMEM_FILTER>(A, B, 4096, tw + tw_offset<P>(4096), io);
    __syncthreads();
    // inverse
    pass<P, 16, true, SRC_SMEM, DST_SMEM>(B, A, 1, tw, io);
    __syncthreads();
    pass<P, 16, true, SRC_SMEM, DST_SMEM>(A, B, 16, tw + tw_offset<P>(16), io);
    __syncthreads();
    pass<P, 16, true, SRC_SMEM, DST_SMEM>(B, A, 256, tw + tw_offset<P>(256), io);
    __syncthreads();
    pass<P, 2, true, SRC_SMEM, DST_GLOBAL>(A, nullptr, 4096, tw + tw_offset<P>(4096), io);
  } else if constexpr (P == 4096) {
    pass<P, 16, false, SRC_SMEM, DST_SMEM>(A, B, 16, tw + tw_offset<P>(16), io);
    __syncthreads();
    fused_middle<P>(B, A, tw + tw_offset<P>(256), w);  // fwd pass 3, filter, inv pass 1
    __syncthreads();
    pass<P, 16, true, SRC_SMEM, DST_SMEM>(A, B, 16, tw + tw_offset<P>(16), io);
    __syncthreads();
    pass<P, RL, true, SRC_SMEM, DST_GLOBAL, true, HALF, NZR>(B, nullptr, 256, tw + tw_offset<P>(256), io);
  } else {
    pass<P, 16, false, SRC_SMEM, DST_SMEM>(A, B, 16, tw + tw_offset<P>(16), io);
    __syncthreads();
    pass<P, RL, false, SRC_SMEM, DST_SMEM_FILTER>(B, A, 256, tw + tw_offset<P>(256), io);
    __syncthreads();
    // inverse
    pass<P, 16, true, SRC_SMEM, DST_SMEM>(A, B, 1, tw, io);
    __syncthreads();
    pass<P, 16, true, SRC_SMEM, DST_SMEM>(B, A, 16, tw + tw_offset<P>(16), io);
    __syncthreads();
    pass<P, RL, true, SRC_SMEM, DST_GLOBAL>(A, nullptr, 256, tw + tw_offset<P>(256), io);
  }
}

// host: per-pass twiddle tables [r][k] = exp(-2 pi i r k P/(Ns R) / P) from FP64
template <int P>
inline std::vector<float2> make_tw_table() {
  std::vector<float2> t(tw_table_size<P>());
  const int spans[3] = {16, 256, 4096};
  for (int Ns : spans) {
    if (Ns >= P) break;
    const int R = radix_at<P>(Ns);
    for (int r = 0; r < R; ++r)
      for (int k = 0; k < Ns; ++k) {
        const double m = double(r) * double(k) * double(P / (Ns * R));
        const double ang = -2.0 * kPi * m / double(P);
        t[tw_offset<P>(Ns) + r * Ns + k] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
      }
  }
  return t;
}

template <int P>
inline size_t smem_bytes() {
  return 2 * size_t(P + P / 16) * sizeof(float2);
}

}  // namespace fft16
}  // namespace filt
}  // namespace tgb
