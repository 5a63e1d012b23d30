// K1-like inner loop (voxel pairs on the FP32x2 pipe, pipelined 4-LDS taps)
// with a fraction of the pairs fetched by exact tld4 gathers instead:
// does the texture path add throughput to the shared-memory path?
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 256, H = 256, NP = 16;

template <int TEXMOD>  // pair k uses tld4 when TEXMOD && k % TEXMOD == TEXMOD - 1
__global__ void __launch_bounds__(256, 3) k1like(cudaTextureObject_t t, float* out, int views) {
  __shared__ float box[64 * 48];
  for (int i = threadIdx.x; i < 64 * 48; i += blockDim.x) box[i] = (i % 97) * 0.001f;
  __syncthreads();
  float2 acc[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = make_float2(0.f, 0.f);
  const float u = 3.3f + (threadIdx.x & 7) * 1.25f, dv = 1.25f;
  for (int it = 0; it < views; ++it) {
    const float v0 = 1.7f + (threadIdx.x >> 3) * 0.05f + (it & 3) * 0.3f;
    const float fu = floorf(u), wu = u - fu;
    const float2 wu2 = make_float2(wu, wu), iw2 = make_float2(1.01f, 1.01f);
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const float2 vk = make_float2(v0 + k * dv * 0.1f, v0 + (k + NP) * dv * 0.1f);
      const float2 fl = make_float2(floorf(vk.x), floorf(vk.y));
      const float2 wv = make_float2(vk.x - fl.x, vk.y - fl.y);
      float a0, a1, b0, b1, c0, c1, d0, d1;
      if (TEXMOD && (k % TEXMOD) == TEXMOD - 1) {
        const float4 g = tex2Dgather<float4>(t, fu + 1.0f, fl.x + 1.0f, 0);
        const float4 h = tex2Dgather<float4>(t, fu + 1.0f, fl.y + 1.0f, 0);
        a0 = g.w; a1 = g.z; b0 = g.x; b1 = g.y; c0 = h.w; c1 = h.z; d0 = h.x; d1 = h.y;
      } else {
        const int ia = int(fl.x) * 48 + int(fu), ib = int(fl.y) * 48 + int(fu);
        a0 = box[ia]; a1 = box[ia + 1]; b0 = box[ia + 48]; b1 = box[ia + 49];
        c0 = box[ib]; c1 = box[ib + 1]; d0 = box[ib + 48]; d1 = box[ib + 49];
      }
      const float2 p0 = make_float2(a0, c0), p1 = make_float2(a1, c1);
      const float2 q0 = make_float2(b0, d0), q1 = make_float2(b1, d1);
      const float2 top = __ffma2_rn(wu2, __fadd2_rn(p1, make_float2(-p0.x, -p0.y)), p0);
      const float2 bot = __ffma2_rn(wu2, __fadd2_rn(q1, make_float2(-q0.x, -q0.y)), q0);
      const float2 mid = __ffma2_rn(wv, __fadd2_rn(bot, make_float2(-top.x, -top.y)), top);
      acc[k] = __ffma2_rn(mid, iw2, acc[k]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NP; ++k) s += acc[k].x + acc[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
  const int blocks = sms * 3, threads = 256, views = 4000;
  float* out;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto fn, const char* name) {
    fn<<<blocks, threads>>>(t, out, 10);
    cudaEventRecord(a);
    fn<<<blocks, threads>>>(t, out, views);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = double(blocks) * threads * views * NP * 2;
    printf("{\"kind\": \"%s\", \"g_updates_s\": %.1f, \"per_clk_per_sm\": %.3f}\n", name,
           n / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
  };
  for (int rep = 0; rep < 2; ++rep) {
    run(k1like<0>, "smem_only");
    run(k1like<4>, "tex_1_of_4_pairs");
    run(k1like<3>, "tex_1_of_3_pairs");
    run(k1like<2>, "tex_1_of_2_pairs");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
