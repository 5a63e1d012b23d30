// LDS.32 / LDS.64 wavefront microbenchmark (B200): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bench scripts/lds_bench.cu
// results: profiles/r1_lds_microbench.txt (pat 0 = 32 distinct words, 1 = pairs share, 2 = ~20 unique contiguous, 3 = spacing 1.25 (40-word span), 4 = 4 rows with a 64-word pitch)
// microbenchmark: shared-memory wavefronts of LDS.32 / LDS.64 under lane-address patterns
#include <cstdio>
#include <cuda_runtime.h>
template <int W, int PAT>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 0.5f;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int word;  // index in units of W floats
  if (PAT == 0) word = lane;                       // all distinct, contiguous
  else if (PAT == 1) word = lane >> 1;             // pairs share
  else if (PAT == 2) word = (lane * 5) >> 3;       // ~20 unique contiguous (spacing 0.625)
  else if (PAT == 3) word = (lane * 5) >> 2;       // spacing 1.25: 40 span, 32 unique
  else word = ((lane & 7) * 5 >> 2) + (lane >> 3) * 64;  // 8x4: 4 rows (pitch 64 words) of ~10
  float acc = 0.f;
  unsigned base = (unsigned)__cvta_generic_to_shared(s) + word * 4 * W + w * 16;
  for (int it = 0; it < iters; ++it) {
    unsigned ad = base + ((it & 3) << 7);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (W == 1) { float v; asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(ad + j * 1024)); acc += v; }
      else { float v0, v1; asm volatile("ld.volatile.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v0), "=f"(v1) : "r"((ad + j * 1024) & ~7u)); acc += v0 + v1; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int W, int PAT> void run(float* d) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096, blocks = 148 * 4, th = 256;
  k<W, PAT><<<blocks, th>>>(d, 16);
  cudaEventRecord(a);
  k<W, PAT><<<blocks, th>>>(d, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double inst = double(blocks) * (th / 32) * iters * 16;
  printf("W=%d pat=%d: %.3f ms, %.3f warp-LDS per clk per SM (at 1.965 GHz)\n", W, PAT, ms, inst / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 4 * 256 * 4);
  run<1,0>(d); run<1,1>(d); run<1,2>(d); run<1,3>(d); run<1,4>(d);
  run<2,0>(d); run<2,1>(d); run<2,2>(d); run<2,3>(d); run<2,4>(d);
  return 0;
}
