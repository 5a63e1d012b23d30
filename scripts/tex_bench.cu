// tex2D bilinear-fetch throughput microbenchmark ("the builder
// records a tex2D microbenchmark peak on the box next to [the theoretical
// 4 bilinear/clk/SM]").  fp32 single-channel 2D texture, linear filtering,
// border addressing, L1-resident footprint; each thread issues FETCHES
// independent fetches per iteration.  Also times the shared-memory lerp
// equivalent (4 LDS + 3 lerps, K1's inner step) for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tex_bench scripts/tex_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 256, H = 256, FETCHES = 8;

__global__ void tex_kernel(cudaTextureObject_t t, float* out, int iters, float du, float dv) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  float u[FETCHES], v[FETCHES], acc[FETCHES];
#pragma unroll
  for (int f = 0; f < FETCHES; ++f) {
    u[f] = 16.37f + (threadIdx.x & 31) * 1.25f + f * 3.1f;
    v[f] = 20.71f + (threadIdx.x >> 5) * 1.7f + f * 2.3f + (blockIdx.x & 63);
    acc[f] = 0.f;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int f = 0; f < FETCHES; ++f) {
      acc[f] += tex2D<float>(t, u[f], v[f]);
      u[f] += du;
      v[f] += dv;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int f = 0; f < FETCHES; ++f) s += acc[f];
  out[tid] = s;
}

__global__ void lds_lerp_kernel(float* out, int iters, float du, float dv) {
  __shared__ float box[64 * 48];
  for (int i = threadIdx.x; i < 64 * 48; i += blockDim.x) box[i] = i * 0.001f;
  __syncthreads();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  float u[FETCHES], v[FETCHES], acc[FETCHES];
#pragma unroll
  for (int f = 0; f < FETCHES; ++f) {
    u[f] = 3.37f + (threadIdx.x & 7) * 1.25f + f * 0.9f;
    v[f] = 2.71f + (threadIdx.x >> 3) * 0.7f + f * 1.3f;
    acc[f] = 0.f;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int f = 0; f < FETCHES; ++f) {
      const float fu = floorf(u[f]), fv = floorf(v[f]);
      const int i = int(fv) * 48 + int(fu);
      const float wu = u[f] - fu, wv = v[f] - fv;
      const float a0 = box[i], a1 = box[i + 1], b0 = box[i + 48], b1 = box[i + 49];
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
  for (int f = 0; f < FETCHES; ++f) s += acc[f];
  out[tid] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max)
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
  td.filterMode = cudaFilterModeLinear;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  cudaTextureObject_t t;
  cudaCreateTextureObject(&t, &rd, &td, nullptr);
  const int blocks = sms * 8, threads = 256, iters = 2000;
  float* out;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    tex_kernel<<<blocks, threads>>>(t, out, 10, 0.37f, 0.11f);
    cudaEventRecord(a);
    tex_kernel<<<blocks, threads>>>(t, out, iters, 0.37f, 0.11f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fetches = double(blocks) * threads * iters * FETCHES;
    printf("{\"kind\": \"tex2D_bilinear_f32\", \"gfetch_s\": %.1f, \"per_clk_per_sm_at_max\": %.3f, \"sms\": %d, \"max_mhz\": %.0f}\n",
           fetches / (ms * 1e-3) / 1e9, fetches / (ms * 1e-3) / sms / (clk * 1e3), sms, clk / 1e3);
    lds_lerp_kernel<<<blocks, threads>>>(out, 10, 0.37f, 0.11f);
    cudaEventRecord(a);
    lds_lerp_kernel<<<blocks, threads>>>(out, iters, 0.37f, 0.11f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"smem_4lds_lerp_f32\", \"gfetch_s\": %.1f, \"per_clk_per_sm_at_max\": %.3f}\n",
           fetches / (ms * 1e-3) / 1e9, fetches / (ms * 1e-3) / sms / (clk * 1e3));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
