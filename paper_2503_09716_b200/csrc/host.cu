// Host-side utilities shared by every launcher in libmgb: tensor-map encoding (through the
// runtime's driver entry point, so the library does not link libcuda directly), SM count, and the
// C-ABI introspection entry points.
#include <cudaTypedefs.h>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

// {code, rows needed, rows_cap, site} of the first capacity overflow since the last read
__device__ int g_capacity_status[4];

namespace mgb_host {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

CUresult encode_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                          const uint64_t* strides_bytes, const uint32_t* box, bool swizzle128, bool l2_promote_256) {
  if (!encoder()) return CUDA_ERROR_NOT_FOUND;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promote_256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

CUresult encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                             uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  if (!encoder()) return CUDA_ERROR_NOT_FOUND;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = mgb::kNumSMsB200;
  }
  return n;
}

int ensure_max_smem(const void* fn, int bytes) {
  // cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute: remember (kernel,
  // device) pairs, not kernels, so a process driving several GPUs configures each one
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return MGB_ECUDA;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({fn, dev})) return MGB_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    launch_status();  // record the error for mgb_last_error
    return MGB_ECUDA;
  }
  done.insert({fn, dev});
  return MGB_OK;
}

int* capacity_status_ptr() {
  static std::mutex mu;
  static int* ptrs[64] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!ptrs[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_capacity_status) != cudaSuccess) return nullptr;
    ptrs[dev] = static_cast<int*>(p);
  }
  return ptrs[dev];
}

namespace {
cudaError_t g_last_err = cudaSuccess;  // first launch error a libmgb entry point returned MGB_ECUDA for
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MGB_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

namespace {
thread_local cudaError_t t_pending = cudaSuccess;  // a cudaLaunchKernelEx failure (mgb_host::launch)
}

void note_launch_error(cudaError_t e) {
  if (t_pending == cudaSuccess) t_pending = e;
}

int launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = t_pending;
  t_pending = cudaSuccess;
  if (e == cudaSuccess) return MGB_OK;
  g_last_err = e;
  return MGB_ECUDA;
}

}  // namespace mgb_host

extern "C" {

// ABI version of include/mgb.h; bumped whenever a signature changes.
int mgb_abi_version(void) { return 2; }

// Name of the last CUDA error seen by the runtime in this library (for loud failures).
// A launch error an entry point already consumed (returned as MGB_ECUDA) is reported, then cleared.
const char* mgb_last_error(void) {
  const cudaError_t e = mgb_host::g_last_err != cudaSuccess ? mgb_host::g_last_err : cudaPeekAtLastError();
  mgb_host::g_last_err = cudaSuccess;
  return cudaGetErrorString(e);
}

// Capacity status of the current device: synchronises the device, copies {code, rows needed,
// rows_cap, site} of the first overflow a grouped GEMM / EP dispatch saw since the last call into
// out4 (may be NULL), clears it when `reset`, and returns MGB_ECAPACITY if one was recorded.
int mgb_capacity_status(int* out4, int reset) {
  int* p = mgb_host::capacity_status_ptr();
  if (!p) return MGB_ECUDA;
  int h[4] = {0, 0, 0, 0};
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(h, p, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess)
    return mgb_host::launch_status(), MGB_ECUDA;
  if (reset && h[0] && cudaMemset(p, 0, sizeof h) != cudaSuccess) return MGB_ECUDA;
  if (out4)
    for (int i = 0; i < 4; ++i) out4[i] = h[i];
  return h[0] ? MGB_ECAPACITY : MGB_OK;
}

// Host-side capacity check in front of a grouped launch whose offsets live on the device (the
// scheduler's pre-flight, exec_sim.py:170-175): copies offsets[E+1] on `stream`, waits, writes the
// per-expert row counts to counts_out[E] (host) and returns MGB_ECAPACITY if the segments need more
// than rows_cap rows (or are not monotone) -- the caller then re-splits the group by b_e.
int mgb_moe_check_capacity(const int* offsets, int E, int rows_cap, int* counts_out, void* stream) {
  if (E < 1 || E > 4096 || rows_cap < 0 || !offsets) return MGB_EINVAL;
  int h[4097];
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(h, offsets, sizeof(int) * (E + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    mgb_host::launch_status();
    return MGB_ECUDA;
  }
  bool ok = h[0] >= 0;
  for (int e = 0; e < E; ++e) {
    const int c = h[e + 1] - h[e];
    ok = ok && c >= 0;
    if (counts_out) counts_out[e] = c;
  }
  return ok && h[E] <= rows_cap ? MGB_OK : MGB_ECAPACITY;
}

// Number of SMs of the current device (148 on B200).
int mgb_num_sms(void) { return mgb_host::num_sms(); }

}  // extern "C"
