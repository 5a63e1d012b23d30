// Can the texture unit add gather throughput to K1's shared-memory path?
// Times (a) tex2Dgather (tld4: the exact 2x2 fp32 footprint, lerped in fp32),
// (b) K1-style 4 LDS + lerps from shared memory, and (c) both interleaved
// in one loop (half the fetches each), all at one SM load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tld4_bench scripts/tld4_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 256, H = 256, F = 8;

template <int MODE>  // 0 = tld4, 1 = lds, 2 = mixed
__global__ void k(cudaTextureObject_t t, float* out, int iters, float du, float dv) {
  __shared__ float box[64 * 48];
  for (int i = threadIdx.x; i < 64 * 48; i += blockDim.x) box[i] = i * 0.001f;
  __syncthreads();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  float u[F], v[F], acc[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    u[f] = 3.37f + (threadIdx.x & 7) * 1.25f + f * 0.9f;
    v[f] = 2.71f + (threadIdx.x >> 3) * 0.7f + f * 1.3f;
    acc[f] = 0.f;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const float fu = floorf(u[f]), fv = floorf(v[f]);
      const float wu = u[f] - fu, wv = v[f] - fv;
      float a0, a1, b0, b1;
      if (MODE == 0 || (MODE == 2 && (f & 1))) {
        // coordinate at the midpoint between texel centres fu+0.5 and fu+1.5:
        // the gathered footprint is (fu, fu+1) x (fv, fv+1) independent of
        // the unit's 8-bit sub-texel rounding
        const float4 g = tex2Dgather<float4>(t, fu + 1.0f, fv + 1.0f, 0);
        a0 = g.w; a1 = g.z; b0 = g.x; b1 = g.y;
      } else {
        const int i = int(fv) * 48 + int(fu);
        a0 = box[i]; a1 = box[i + 1]; b0 = box[i + 48]; b1 = box[i + 49];
      }
      const float top = fmaf(wu, a1 - a0, a0), bot = fmaf(wu, b1 - b0, b0);
      acc[f] += fmaf(wv, bot - top, top);
      u[f] += du;
      v[f] += dv;
      if (u[f] > 40.f) u[f] -= 30.f;
      if (v[f] > 55.f) v[f] -= 45.f;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int f = 0; f < F; ++f) s += acc[f];
  out[tid] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
  cudaArray_t arr;
  cudaMallocArray(&arr, &cd, W, H);
  float* h = new float[W * H];
  for (int i = 0; i < W * H; ++i) h[i] = (i % 97) * 0.01f;
  cudaMemcpy2DToArray(arr, 0, 0, h, W * 4, W * 4, H, cudaMemcpyHostToDevice);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = arr;
  cudaTextureDesc td = {};
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t t;
  cudaCreateTextureObject(&t, &rd, &td, nullptr);
  const int blocks = sms * 8, threads = 256, iters = 2000;
  float* out;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"tld4_gather_lerp", "smem_4lds_lerp", "mixed_half_each"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 3; ++m) {
      auto fn = m == 0 ? k<0> : (m == 1 ? k<1> : k<2>);
      fn<<<blocks, threads>>>(t, out, 10, 0.37f, 0.11f);
      cudaEventRecord(a);
      fn<<<blocks, threads>>>(t, out, iters, 0.37f, 0.11f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double n = double(blocks) * threads * iters * F;
      printf("{\"kind\": \"%s\", \"g_updates_s\": %.1f, \"per_clk_per_sm_at_max\": %.3f}\n", names[m],
             n / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
