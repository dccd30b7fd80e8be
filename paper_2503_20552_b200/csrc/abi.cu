// libadrenaline.so housekeeping: error state, version, device facts, TMA
// descriptor encoding, peer access / peer copies and stream-ordered flags.
#include <cstdio>
#include <cstring>
#include <mutex>

#include "adr_internal.h"

namespace adr {

namespace {
thread_local char g_last_error[512] = {0};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using StreamWriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using StreamWaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using AddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

struct DriverFns {
  EncodeTiledFn encode_tiled = nullptr;
  StreamWriteFn write_value = nullptr;
  StreamWaitFn wait_value = nullptr;
  AddressRangeFn address_range = nullptr;
  bool loaded = false;
};

// Green-context entry points (adr_sm_partition_*), resolved on first use.
using DeviceGetFn = CUresult (*)(CUdevice*, int);
using GetDevResourceFn = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using SmSplitFn = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                               unsigned int, unsigned int);
using GenDescFn = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
using GreenCreateFn = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
using GreenStreamFn = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
using GreenDestroyFn = CUresult (*)(CUgreenCtx);
using StreamDestroyFn = CUresult (*)(CUstream);

template <typename F>
F entry(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

struct Partition {
  CUgreenCtx ctx[2] = {nullptr, nullptr};
  CUstream stream[2] = {nullptr, nullptr};
};

DriverFns& driver() {
  static DriverFns fns;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fns.encode_tiled = reinterpret_cast<EncodeTiledFn>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fns.write_value = reinterpret_cast<StreamWriteFn>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fns.wait_value = reinterpret_cast<StreamWaitFn>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fns.address_range = reinterpret_cast<AddressRangeFn>(fn);
    fns.loaded = true;
  });
  return fns;
}
}  // namespace

void clear_error() { g_last_error[0] = '\0'; }

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

bool cuda_ok(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return true;
  fail(ADR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(err));
  return false;
}

namespace {
// A page tensor map depends only on (base, D, rows): cache the last few per
// thread so steady-state calls skip the driver encode (~µs of host time each).
struct TmapEntry {
  const void* base = nullptr;
  int D = 0;
  uint64_t rows = 0;
  CUtensorMap map;
};
constexpr int kTmapCache = 128;
thread_local TmapEntry g_tmaps[kTmapCache];
thread_local int g_tmap_next = 0;
}  // namespace

int encode_page_tmap(CUtensorMap* map, const void* base, int D, uint64_t rows) {
  for (const TmapEntry& e : g_tmaps) {
    if (e.base == base && e.D == D && e.rows == rows) {
      *map = e.map;
      return ADR_OK;
    }
  }
  DriverFns& d = driver();
  if (d.encode_tiled == nullptr)
    return fail(ADR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 16};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = d.encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ADR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  TmapEntry& slot = g_tmaps[g_tmap_next];
  g_tmap_next = (g_tmap_next + 1) % kTmapCache;
  slot.base = base;
  slot.D = D;
  slot.rows = rows;
  slot.map = *map;
  return ADR_OK;
}

}  // namespace adr

using namespace adr;

extern "C" int32_t adr_version(void) { return (0 << 16) | 1; }

extern "C" const char* adr_last_error(void) { return g_last_error; }

extern "C" int32_t adr_device_info(int32_t device, int32_t* num_sms, int32_t* cc_major,
                                   int32_t* cc_minor) {
  clear_error();
  if (!num_sms || !cc_major || !cc_minor) return fail(ADR_ERR_INVALID, "null output pointer");
  int v = 0;
  if (!cuda_ok(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device),
               "cudaDeviceGetAttribute(SMs)"))
    return ADR_ERR_CUDA;
  *num_sms = v;
  if (!cuda_ok(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device), "cc major"))
    return ADR_ERR_CUDA;
  *cc_major = v;
  if (!cuda_ok(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device), "cc minor"))
    return ADR_ERR_CUDA;
  *cc_minor = v;
  return ADR_OK;
}

extern "C" int32_t adr_peer_open(int32_t dev_a, int32_t dev_b) {
  clear_error();
  if (dev_a == dev_b) return ADR_OK;
  int prev = 0;
  if (!cuda_ok(cudaGetDevice(&prev), "cudaGetDevice")) return ADR_ERR_CUDA;
  const int pairs[2][2] = {{dev_a, dev_b}, {dev_b, dev_a}};
  for (auto& pr : pairs) {
    int can = 0;
    if (!cuda_ok(cudaDeviceCanAccessPeer(&can, pr[0], pr[1]), "cudaDeviceCanAccessPeer"))
      return ADR_ERR_CUDA;
    if (!can) {
      cudaSetDevice(prev);
      return fail(ADR_ERR_UNSUPPORTED, "device %d cannot access peer %d", pr[0], pr[1]);
    }
    cudaSetDevice(pr[0]);
    cudaError_t e = cudaDeviceEnablePeerAccess(pr[1], 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
    } else if (!cuda_ok(e, "cudaDeviceEnablePeerAccess")) {
      cudaSetDevice(prev);
      return ADR_ERR_CUDA;
    }
  }
  cudaSetDevice(prev);
  return ADR_OK;
}

extern "C" int32_t adr_copy_peer(void* dst, int32_t dst_dev, const void* src, int32_t src_dev,
                                 size_t bytes, void* stream) {
  clear_error();
  if (bytes == 0) return ADR_OK;
  if (!dst || !src) return fail(ADR_ERR_INVALID, "null pointer");
  cudaError_t e = dst_dev == src_dev
                      ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice,
                                        static_cast<cudaStream_t>(stream))
                      : cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes,
                                            static_cast<cudaStream_t>(stream));
  return cuda_ok(e, "peer copy") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" int32_t adr_signal(uint32_t* flag, uint32_t value, void* stream) {
  clear_error();
  if (!flag) return fail(ADR_ERR_INVALID, "null flag");
  DriverFns& d = driver();
  if (!d.write_value) return fail(ADR_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  CUresult r = d.write_value(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag),
                             value, CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? ADR_OK : fail(ADR_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
}

extern "C" int32_t adr_wait(const uint32_t* flag, uint32_t value, void* stream) {
  clear_error();
  if (!flag) return fail(ADR_ERR_INVALID, "null flag");
  DriverFns& d = driver();
  if (!d.wait_value) return fail(ADR_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  CUresult r = d.wait_value(static_cast<CUstream>(stream),
                            reinterpret_cast<CUdeviceptr>(const_cast<uint32_t*>(flag)), value,
                            CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? ADR_OK : fail(ADR_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
}

// ---- CUDA IPC: the zero-copy offload across processes -----------------------
// The decode process exports the allocations holding its per-layer q/k/v/out
// rows and its flags; the executor process maps them and passes the mapped
// pointers to adr_paged_decode_attn_rows / adr_signal / adr_wait. Allocators
// sub-allocate, so a handle names the containing allocation plus an offset.

static_assert(sizeof(cudaIpcMemHandle_t) == ADR_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" int32_t adr_ipc_export(const void* ptr, void* handle, uint64_t* offset) {
  clear_error();
  if (!ptr || !handle || !offset) return fail(ADR_ERR_INVALID, "null pointer");
  DriverFns& d = driver();
  if (!d.address_range) return fail(ADR_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = d.address_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) return fail(ADR_ERR_CUDA, "cuMemGetAddressRange failed (%d)", (int)r);
  cudaIpcMemHandle_t h;
  if (!cuda_ok(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle"))
    return ADR_ERR_CUDA;
  std::memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<CUdeviceptr>(ptr) - base;
  return ADR_OK;
}

extern "C" int32_t adr_ipc_import(const void* handle, uint64_t offset, void** ptr, void** base) {
  clear_error();
  if (!handle || !ptr || !base) return fail(ADR_ERR_INVALID, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* b = nullptr;
  if (!cuda_ok(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle"))
    return ADR_ERR_CUDA;
  *base = b;
  *ptr = static_cast<uint8_t*>(b) + offset;
  return ADR_OK;
}

extern "C" int32_t adr_ipc_close(void* base) {
  clear_error();
  if (!base) return fail(ADR_ERR_INVALID, "null pointer");
  return cuda_ok(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" ADR_API int32_t adr_sm_partition_create(int32_t device, int32_t attn_sms,
                                                   int32_t attn_priority, int32_t prefill_priority,
                                                   void** attn_stream, void** prefill_stream,
                                                   int32_t* attn_sms_out, int32_t* prefill_sms_out,
                                                   void** handle) {
  adr::clear_error();
  if (!attn_stream || !prefill_stream || !handle || attn_sms <= 0)
    return adr::fail(ADR_ERR_INVALID, "adr_sm_partition_create: bad arguments");
  static const auto dev_get = adr::entry<adr::DeviceGetFn>("cuDeviceGet");
  static const auto get_res = adr::entry<adr::GetDevResourceFn>("cuDeviceGetDevResource");
  static const auto split = adr::entry<adr::SmSplitFn>("cuDevSmResourceSplitByCount");
  static const auto gen = adr::entry<adr::GenDescFn>("cuDevResourceGenerateDesc");
  static const auto gcreate = adr::entry<adr::GreenCreateFn>("cuGreenCtxCreate");
  static const auto gstream = adr::entry<adr::GreenStreamFn>("cuGreenCtxStreamCreate");
  if (!dev_get || !get_res || !split || !gen || !gcreate || !gstream)
    return adr::fail(ADR_ERR_UNSUPPORTED, "green-context driver entry points unavailable");
  int prev_dev = 0;
  if (!adr::cuda_ok(cudaGetDevice(&prev_dev), "cudaGetDevice")) return ADR_ERR_CUDA;
  // make sure the device's primary context exists, then leave the caller's
  // current device as it was
  const bool ctx_ok = adr::cuda_ok(cudaSetDevice(device), "cudaSetDevice") &&
                      adr::cuda_ok(cudaFree(nullptr), "cudaFree(0)");
  cudaSetDevice(prev_dev);
  if (!ctx_ok) return ADR_ERR_CUDA;
  CUdevice dev;
  CUdevResource all, groups[1], rest;
  if (dev_get(&dev, device) != CUDA_SUCCESS || get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return adr::fail(ADR_ERR_CUDA, "cuDeviceGetDevResource failed");
  unsigned int n = 1;
  if (split(groups, &n, &all, &rest, 0, (unsigned)attn_sms) != CUDA_SUCCESS || n != 1)
    return adr::fail(ADR_ERR_INVALID, "cuDevSmResourceSplitByCount(%d SMs) failed", attn_sms);
  auto* part = new adr::Partition();
  CUdevResource* res[2] = {&groups[0], &rest};
  const int prio[2] = {attn_priority, prefill_priority};
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc desc;
    CUresult r = gen(&desc, res[i], 1);
    if (r == CUDA_SUCCESS) r = gcreate(&part->ctx[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r == CUDA_SUCCESS) r = gstream(&part->stream[i], part->ctx[i], CU_STREAM_NON_BLOCKING, prio[i]);
    if (r != CUDA_SUCCESS) {
      adr_sm_partition_destroy(part);
      return adr::fail(ADR_ERR_CUDA, "green context %d: driver error %d", i, (int)r);
    }
  }
  *attn_stream = part->stream[0];
  *prefill_stream = part->stream[1];
  if (attn_sms_out) *attn_sms_out = (int32_t)groups[0].sm.smCount;
  if (prefill_sms_out) *prefill_sms_out = (int32_t)rest.sm.smCount;
  *handle = part;
  return ADR_OK;
}

extern "C" ADR_API int32_t adr_sm_partition_destroy(void* handle) {
  adr::clear_error();
  if (!handle) return ADR_OK;
  static const auto gdestroy = adr::entry<adr::GreenDestroyFn>("cuGreenCtxDestroy");
  static const auto sdestroy = adr::entry<adr::StreamDestroyFn>("cuStreamDestroy");
  auto* part = static_cast<adr::Partition*>(handle);
  for (int i = 0; i < 2; ++i) {
    if (part->stream[i] && sdestroy) sdestroy(part->stream[i]);
    if (part->ctx[i] && gdestroy) gdestroy(part->ctx[i]);
  }
  delete part;
  return ADR_OK;
}
