// runtime.cu — library-wide runtime services: launch accounting, kernel
// timing, plan ids and TMA descriptor encoding.
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>

#include "device_common.cuh"

namespace tgb {

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_plan_ids{0};
std::atomic<bool> g_timing{false};
std::mutex g_timer_mu;
cudaEvent_t g_ev_a = nullptr, g_ev_b = nullptr;
bool g_have_timing = false;
double g_last_ms = 0.0;
}  // namespace

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t next_plan_id() { return g_plan_ids.fetch_add(1) + 1; }
bool timing_enabled() { return g_timing.load(); }
void record_kernel_ms(double ms) { g_last_ms = ms; }

void KernelTimer::start(cudaStream_t st) {
  on = timing_enabled();
  if (!on) return;
  s = st;
  std::lock_guard<std::mutex> lk(g_timer_mu);
  if (!g_ev_a) {
    TG_CUDA(cudaEventCreate(&g_ev_a));
    TG_CUDA(cudaEventCreate(&g_ev_b));
  }
  TG_CUDA(cudaEventRecord(g_ev_a, s));
}

void KernelTimer::stop() {
  if (!on) return;
  std::lock_guard<std::mutex> lk(g_timer_mu);
  TG_CUDA(cudaEventRecord(g_ev_b, s));
  g_have_timing = true;
}

CUresult encode_tensor_map_3d_f32(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1,
                                  uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes,
                                  uint32_t box0, uint32_t box1, uint32_t box2) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!fn) return CUDA_ERROR_NOT_SUPPORTED;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {box0, box1, box2};
  const cuuint32_t elem[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box,
            elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace tgb

extern "C" {

uint64_t tg_kernel_launch_count(void) { return tgb::g_launches.load(); }

void tg_set_timing(int enable) { tgb::g_timing.store(enable != 0); }

double tg_last_kernel_ms(void) {
  std::lock_guard<std::mutex> lk(tgb::g_timer_mu);
  if (!tgb::g_have_timing) return -1.0;
  float ms = 0.f;
  if (cudaEventSynchronize(tgb::g_ev_b) != cudaSuccess) return -1.0;
  if (cudaEventElapsedTime(&ms, tgb::g_ev_a, tgb::g_ev_b) != cudaSuccess) return -1.0;
  return double(ms);
}

}  // extern "C"
