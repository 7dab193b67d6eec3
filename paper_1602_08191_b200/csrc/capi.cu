// capi.cu — error state, version and device queries of the C-ABI.
#include <mutex>

#include "ds_common.cuh"
#include "master.cuh"

namespace dsb {

std::string& last_error() {
  thread_local std::string msg;
  return msg;
}

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

int sm_count(int device) {
  static std::mutex mu;
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[device] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    cache[device] = v;
  }
  return cache[device];
}

}  // namespace dsb

extern "C" const char* ds_last_error(void) { return dsb::last_error().c_str(); }

extern "C" const char* ds_version(void) { return "paper_1602_08191_b200 0.1 (sm_100a)"; }

extern "C" int ds_device_count(int* count) {
  if (!count) return dsb::set_error(DS_E_CONTRACT, "device_count: null");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    *count = 0;
    return DS_OK;
  }
  if (e != cudaSuccess) return dsb::set_error(DS_E_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  *count = n;
  return DS_OK;
}

// ------------------------------------------------------------------------------------
// Device plumbing
// ------------------------------------------------------------------------------------
extern "C" int ds_device_alloc(int device, uint64_t bytes, void** out) {
  if (!out) return dsb::set_error(DS_E_CONTRACT, "device_alloc: null");
  dsb::DeviceScope ds(device);
  *out = nullptr;
  if (bytes == 0) bytes = 1;
  DS_CUDA_TRY(cudaMalloc(out, bytes));
  return DS_OK;
}

extern "C" int ds_device_free(void* p) {
  if (p) DS_CUDA_TRY(cudaFree(p));
  return DS_OK;
}

extern "C" int ds_memcpy(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return DS_OK;
  if (!dst || !src) return dsb::set_error(DS_E_CONTRACT, "memcpy: null");
  if (stream) {
    DS_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, dsb::as_stream(stream)));
  } else {
    DS_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  }
  return DS_OK;
}

extern "C" int ds_memset(void* dst, int value, uint64_t bytes, void* stream) {
  if (bytes == 0) return DS_OK;
  if (stream) {
    DS_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, dsb::as_stream(stream)));
  } else {
    DS_CUDA_TRY(cudaMemset(dst, value, bytes));
  }
  return DS_OK;
}

extern "C" int ds_stream_create(int device, void** stream) {
  if (!stream) return dsb::set_error(DS_E_CONTRACT, "stream_create: null");
  dsb::DeviceScope ds(device);
  cudaStream_t s = nullptr;
  DS_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return DS_OK;
}

extern "C" int ds_stream_destroy(void* stream) {
  if (stream) dsb::master_forget_stream(dsb::as_stream(stream));  // no master may record on it later
  if (stream) DS_CUDA_TRY(cudaStreamDestroy(dsb::as_stream(stream)));
  return DS_OK;
}

extern "C" int ds_stream_sync(void* stream) {
  DS_CUDA_TRY(cudaStreamSynchronize(dsb::as_stream(stream)));
  return DS_OK;
}
