// One 3D TMA box load with given tensor dims / pitch / box / coordinates:
// prints "ok <sum>" or the CUDA error.  Used to pin TMA constraints for the
// slab-staged K2 (box extents vs tensor extents, coordinates).
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_1904_13342_b200/csrc tma_box_test.cu
//   ./a.out d0 d1 d2 pitch box0 box1 box2 c0 c1 c2
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(su32(sm)), "l"((uint64_t)&m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar)) : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
  }
  float s = 0;
  const float* f = (const float*)sm;
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) s += f[i];
  atomicAdd(out, s);
}

int main(int argc, char** argv) {
  if (argc < 11) return 2;
  long d0 = atol(argv[1]), d1 = atol(argv[2]), d2 = atol(argv[3]), pitch = atol(argv[4]);
  unsigned b0 = atoi(argv[5]), b1 = atoi(argv[6]), b2 = atoi(argv[7]);
  int c0 = atoi(argv[8]), c1 = atoi(argv[9]), c2 = atoi(argv[10]);
  float* g;
  cudaMalloc(&g, pitch * d1 * d2 * 4);
  float* h = (float*)malloc(pitch * d1 * d2 * 4);
  for (long i = 0; i < pitch * d1 * d2; ++i) h[i] = 1.0f;
  cudaMemcpy(g, h, pitch * d1 * d2 * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)pitch * d1 * 4};
  cuuint32_t box[3] = {b0, b1, b2}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  float* out;
  cudaMalloc(&out, 4);
  cudaMemset(out, 0, 4);
  int bytes = b0 * b1 * b2 * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 128);
  k<<<1, 128, bytes + 128>>>(m, c0, c1, c2, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  float s = 0;
  cudaMemcpy(&s, out, 4, cudaMemcpyDeviceToHost);
  printf("%s d=(%ld,%ld,%ld) p=%ld box=(%u,%u,%u) c=(%d,%d,%d) sum=%g\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e),
         d0, d1, d2, pitch, b0, b1, b2, c0, c1, c2, s);
  return 0;
}
