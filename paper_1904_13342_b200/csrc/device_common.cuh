// device_common.cuh — CUDA plumbing shared by the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "tg_internal.h"

namespace tgb {

#define TG_CUDA(expr)                                                                         \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      throw ::tgb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
  } while (0)

#define TG_LAUNCHED(n)                                                                        \
  do {                                                                                        \
    cudaError_t _e = cudaGetLastError();                                                      \
    if (_e != cudaSuccess)                                                                    \
      throw ::tgb::CudaError(std::string("kernel launch: ") + cudaGetErrorString(_e));        \
    ::tgb::count_launch(n);                                                                   \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    TG_CUDA(cudaGetDevice(&prev));
    if (prev != dev) TG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Device time of kernels between start()/stop() on one stream (enabled by
// tg_set_timing); feeds tg_last_kernel_ms() for bench.py's roofline.
struct KernelTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s = nullptr;
  bool on = false;
  void start(cudaStream_t st);
  void stop();
};
bool timing_enabled();
void record_kernel_ms(double ms);

// A __constant__ bank shared by all plans of one kernel family on one
// device.  Uploads are stream-ordered: before a plan overwrites the bank,
// its stream waits for every kernel that read the previous contents — one
// reader event per stream that launched a reader since then (a plan may
// launch on several streams).
struct ConstBank {
  struct Reader {
    cudaStream_t stream;
    cudaEvent_t ev;
  };
  static constexpr int kMaxDev = 64;
  static constexpr size_t kMaxReaders = 32;
  std::mutex mu;
  uint64_t owner[kMaxDev] = {};
  std::vector<Reader> readers[kMaxDev];
  // Call with mu held, right before launching on `stream`.
  void acquire(int dev, uint64_t plan_id, cudaStream_t stream, const void* symbol,
               const void* d_src, size_t bytes) {
    if (owner[dev] != plan_id) {
      for (const Reader& r : readers[dev])
        if (r.stream != stream) TG_CUDA(cudaStreamWaitEvent(stream, r.ev, 0));
      TG_CUDA(cudaMemcpyToSymbolAsync(symbol, d_src, bytes, 0, cudaMemcpyDeviceToDevice, stream));
      owner[dev] = plan_id;
    }
  }
  // After the reader launch.  Inside a CUDA-graph capture the owner cannot
  // change (callers capture only work whose bank upload happened before the
  // capture), so no ordering event is recorded there.
  void release(int dev, cudaStream_t stream) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TG_CUDA(cudaStreamIsCapturing(stream, &cs));
    if (cs == cudaStreamCaptureStatusActive) return;
    std::vector<Reader>& rs = readers[dev];
    for (Reader& r : rs)
      if (r.stream == stream) {
        TG_CUDA(cudaEventRecord(r.ev, stream));
        return;
      }
    if (rs.size() >= kMaxReaders) {
      // bound the list: the oldest readers are waited for on the host
      for (Reader& r : rs) TG_CUDA(cudaEventSynchronize(r.ev));
      for (Reader& r : rs) cudaEventDestroy(r.ev);
      rs.clear();
    }
    Reader r{stream, nullptr};
    TG_CUDA(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
    TG_CUDA(cudaEventRecord(r.ev, stream));
    rs.push_back(r);
  }
  void forget(uint64_t plan_id) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& o : owner)
      if (o == plan_id) o = 0;
  }
};

// Orders the uses of one plan-owned scratch buffer across streams: a call
// about to overwrite it first makes its own stream wait for the last stream
// that used it (the ConstBank pattern for device memory).  Call enter()
// before the first launch touching the buffer and leave() after the last,
// both with the owning plan's mutex held.  Inside a CUDA-graph capture the
// ordering is the capture's own (nothing recorded or waited on).
struct ScratchOrder {
  cudaEvent_t ev = nullptr;
  cudaStream_t last = nullptr;
  bool used = false;
  static bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TG_CUDA(cudaStreamIsCapturing(st, &cs));
    return cs == cudaStreamCaptureStatusActive;
  }
  void enter(cudaStream_t st) {
    if (used && last != st && !capturing(st)) TG_CUDA(cudaStreamWaitEvent(st, ev, 0));
  }
  void leave(cudaStream_t st) {
    if (capturing(st)) return;
    if (!ev) TG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TG_CUDA(cudaEventRecord(ev, st));
    last = st;
    used = true;
  }
  ~ScratchOrder() {
    if (ev) cudaEventDestroy(ev);
  }
};

uint64_t next_plan_id();

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
CUresult encode_tensor_map_3d_f32(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1,
                                  uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes,
                                  uint32_t box0, uint32_t box1, uint32_t box2 = 1);

// ---- device-side PTX helpers (sm_90+/sm_100a) --------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// For a producer warp that runs ahead of its consumers: back off between
// polls so the spin does not take issue slots from the consumer warps.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, unsigned ns) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(ns);
}

// TMA: 3D tile load global -> shared, completion counted on `bar` (bytes).
// Out-of-bounds elements (including negative coordinates) are zero-filled,
// which is exactly the reference's zero-padded interpolation
// (projector.hpp:36-40,51-62).
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tensor_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace tgb
