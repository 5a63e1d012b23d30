// K2-like gathers: per sample two 16-byte quads (slices z and z+1) from a
// quad volume via LDG.128, vs one LDG.128 + one exact tld4 gather (layered
// 2D texture, midpoint coordinates), vs two tld4 — do the LSU and texture
// paths add up for ray-marching gathers?
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NX = 256, NY = 256, NZ = 64;

template <int MODE>  // 0: 2 x LDG.128, 1: LDG.128 + tld4, 2: 2 x tld4
__global__ void __launch_bounds__(256, 4) k(const float4* __restrict__ q, cudaTextureObject_t t, float* out,
                                            int steps) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float px = 20.3f + (lane & 7) * 0.8f + (blockIdx.x % 16) * 12.f;
  float py = 30.7f + (lane >> 3) * 0.8f + w * 3.3f + (blockIdx.x / 16 % 8) * 20.f;
  float pz = 5.1f + (blockIdx.x % 7) * 3.f;
  const float dx = 0.45f, dy = 0.12f, dz = 0.05f;
  float sum = 0.f;
  for (int s = 0; s < steps; ++s) {
    const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
    const float wx = px - fx, wy = py - fy, wz = pz - fz;
    const int ix = int(fx), iy = int(fy), iz = int(fz);
    float4 a, b;
    if (MODE == 2) {
      const float4 g = tex2DLayered<float4>(t, fx + 1.0f, fy + 1.0f, iz);
      a = make_float4(g.w, g.z, g.x, g.y);
    } else {
      a = __ldg(q + (iz * NY + iy) * NX + ix);
    }
    if (MODE >= 1) {
      const float4 g = tex2DLayered<float4>(t, fx + 1.0f, fy + 1.0f, iz + 1);
      b = make_float4(g.w, g.z, g.x, g.y);
    } else {
      b = __ldg(q + ((iz + 1) * NY + iy) * NX + ix);
    }
    const float c0 = fmaf(wy, fmaf(wx, a.w - a.z, a.z) - fmaf(wx, a.y - a.x, a.x), fmaf(wx, a.y - a.x, a.x));
    const float c1 = fmaf(wy, fmaf(wx, b.w - b.z, b.z) - fmaf(wx, b.y - b.x, b.x), fmaf(wx, b.y - b.x, b.x));
    sum += fmaf(wz, c1 - c0, c0);
    px += dx; py += dy; pz += dz;
    if (px > NX - 30) px -= 200.f;
    if (py > NY - 30) py -= 150.f;
    if (pz > NZ - 4) pz -= 50.f;
  }
  out[tid] = sum;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float4* q;
  cudaMalloc(&q, size_t(NX) * NY * NZ * sizeof(float4));
  cudaMemset(q, 0, size_t(NX) * NY * NZ * sizeof(float4));
  cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
  cudaArray_t arr;
  cudaExtent ext = make_cudaExtent(NX, NY, NZ);
  cudaMalloc3DArray(&arr, &cd, ext, cudaArrayLayered);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = arr;
  cudaTextureDesc td = {};
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t t;
  cudaCreateTextureObject(&t, &rd, &td, nullptr);
  const int blocks = sms * 4 * 4, threads = 256, steps = 3000;
  float* out;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"2x_ldg128", "ldg128_plus_tld4", "2x_tld4"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 3; ++m) {
      auto fn = m == 0 ? k<0> : (m == 1 ? k<1> : k<2>);
      fn<<<blocks, threads>>>(q, t, out, 10);
      cudaEventRecord(e0);
      fn<<<blocks, threads>>>(q, t, out, steps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n = double(blocks) * threads * steps;
      printf("{\"kind\": \"%s\", \"gsamples_s\": %.1f, \"per_clk_per_sm\": %.3f}\n", names[m],
             n / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / sms / (clk * 1e3));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
