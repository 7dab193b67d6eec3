#include "device_ctx.hpp"

#include <cstdlib>
#include <string>
#include <vector>

namespace deepspark {

void throw_status(int status, const char* context) {
  const std::string msg = std::string(context) + ": " + ds_last_error();
  switch (status) {
    case DS_E_CONTRACT: throw ContractError(ds_last_error());
    case DS_E_NUMERIC: throw NumericError(ds_last_error());
    case DS_E_FORMAT: throw FormatError(ds_last_error());
    case DS_E_IO: throw IoError(ds_last_error());
    default: throw CudaError(msg);
  }
}

namespace detail {

int default_device() {
  const char* env = std::getenv("DEEPSPARK_DEVICE");
  return env ? std::atoi(env) : 0;
}

DeviceCtx::DeviceCtx() : device_(default_device()) {
  check_status(ds_stream_create(device_, &stream_), "device context");
}

DeviceCtx::~DeviceCtx() {
  if (stream_) ds_stream_sync(stream_);
  for (void* p : buf_) ds_device_free(p);
  ds_stream_destroy(stream_);
}

DeviceCtx& DeviceCtx::get() {
  thread_local DeviceCtx ctx;
  return ctx;
}

void* DeviceCtx::scratch(int slot, size_t bytes) {
  if (bytes > cap_[slot]) {
    sync();
    ds_device_free(buf_[slot]);
    buf_[slot] = nullptr;
    size_t cap = cap_[slot] * 2 > bytes ? cap_[slot] * 2 : bytes;
    check_status(ds_device_alloc(device_, cap, &buf_[slot]), "device scratch");
    cap_[slot] = cap;
  }
  return buf_[slot];
}

void DeviceCtx::upload(void* dst, const void* src, size_t bytes) {
  check_status(ds_memcpy(dst, src, bytes, stream_), "upload");
}

void DeviceCtx::download(void* dst, const void* src, size_t bytes) {
  check_status(ds_memcpy(dst, src, bytes, stream_), "download");
}

void DeviceCtx::sync() { check_status(ds_stream_sync(stream_), "sync"); }

}  // namespace detail
}  // namespace deepspark
