// device_ctx.hpp — per-thread device scratch used by the synchronous C++ API calls
// (loss_and_grad, sgd_step, easgd_update, MasterState::exchange, accuracy ...).
// Everything goes through the C-ABI (ds_cuda.h); this file links no CUDA runtime.
#pragma once

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "deepspark/errors.hpp"
#include "ds_cuda.h"

namespace deepspark::detail {

int default_device();  // $DEEPSPARK_DEVICE or 0

class DeviceCtx {
 public:
  static DeviceCtx& get();  // thread-local, on default_device()
  ~DeviceCtx();
  int device() const { return device_; }
  void* stream() const { return stream_; }
  // Grow-only scratch buffer `slot` of at least `bytes` bytes.
  void* scratch(int slot, size_t bytes);
  void upload(void* dst, const void* src, size_t bytes);   // async on stream()
  void download(void* dst, const void* src, size_t bytes); // async on stream()
  void sync();

 private:
  DeviceCtx();
  int device_ = 0;
  void* stream_ = nullptr;
  void* buf_[12] = {};
  size_t cap_[12] = {};
};

// ds_model_desc view of a Model (hidden array kept alive by the holder).
struct ModelDesc {
  ds_model_desc d{};
  std::vector<uint32_t> hidden;
};

}  // namespace deepspark::detail

namespace deepspark::detail {

// Owned device allocation on the context's device.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) {
    check_status(ds_device_alloc(DeviceCtx::get().device(), bytes, &p_), "device alloc");
  }
  ~DeviceBuffer() { ds_device_free(p_); }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    return *this;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
};

}  // namespace deepspark::detail
