// shard.cu — DSHD shard ingestion straight into device memory.
//
// The reference reads a whole shard file into a host vector, then decodes it row by row
// into Dataset{features, labels} (shard.cpp:75-125). Here the header is validated on the
// host with the same checks in the same order and the same messages. The body is
// streamed in row-aligned chunks:
//   pread by several host threads -> pinned buffer -> async H2D copy -> a device
//   staging buffer -> dshd_unpack_kernel.
// dshd_unpack_kernel splits the interleaved rows (F x f32, u32 label) into the resident
// row-major X [n x F] and y [n], and range-checks every label on the device. Two
// pinned/staging slots alternate, so file reads overlap the copy engine and the
// unpack. The first out-of-range label is reported like the reference's loop:
// "<path>: label L out of range at sample i".
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ds_common.cuh"

namespace dsb {
namespace {

constexpr uint32_t kMagic = 0x44534844u;  // "DSHD" (shard.hpp:17)
constexpr uint32_t kVersion = 1;
constexpr uint64_t kHeaderBytes = 28;
constexpr uint64_t kChunkBytes = 64ull << 20;  // per slot; two slots in flight
constexpr int kUnpackThreads = 256;

uint32_t rd32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 | static_cast<uint32_t>(p[2]) << 16 |
         static_cast<uint32_t>(p[3]) << 24;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// pread exactly n bytes at off, or fail
bool pread_all(int fd, void* dst, uint64_t n, uint64_t off) {
  auto* p = static_cast<uint8_t*>(dst);
  while (n > 0) {
    const ssize_t got = pread(fd, p, n, static_cast<off_t>(off));
    if (got < 0 && errno == EINTR) continue;
    if (got <= 0) return false;
    p += got;
    off += static_cast<uint64_t>(got);
    n -= static_cast<uint64_t>(got);
  }
  return true;
}

// several threads read disjoint pieces of one chunk (page-cache copy is the host bound)
bool pread_parallel(int fd, void* dst, uint64_t n, uint64_t off) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t nt = std::min<uint64_t>(std::min(hw, 8u), std::max<uint64_t>(1, n >> 22));  // >= 4 MiB each
  if (nt <= 1) return pread_all(fd, dst, n, off);
  std::vector<std::thread> th;
  std::vector<char> ok(nt, 0);
  const uint64_t piece = (n + nt - 1) / nt;
  for (uint64_t t = 0; t < nt; ++t) {
    const uint64_t b = t * piece, e = std::min(n, b + piece);
    th.emplace_back([&, t, b, e] { ok[t] = e <= b || pread_all(fd, static_cast<uint8_t*>(dst) + b, e - b, off + b); });
  }
  for (auto& x : th) x.join();
  return std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; });
}

// Header validation in read_shard's order (shard.cpp:75-99); FormatError -> DS_E_FORMAT,
// IoError -> DS_E_IO, with the reference's messages.
int read_header(const char* path, Fd& f, ds_shard_info* info) {
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return set_error(DS_E_IO, "cannot open %s", path);
  struct stat st {};
  if (fstat(f.fd, &st) != 0) return set_error(DS_E_IO, "read failed for %s", path);
  const uint64_t size = static_cast<uint64_t>(st.st_size);
  if (size < kHeaderBytes) return set_error(DS_E_FORMAT, "%s: truncated header", path);
  uint8_t h[kHeaderBytes];
  if (!pread_all(f.fd, h, kHeaderBytes, 0)) return set_error(DS_E_IO, "read failed for %s", path);
  if (rd32(h) != kMagic) return set_error(DS_E_FORMAT, "%s: bad magic", path);
  if (rd32(h + 4) != kVersion) return set_error(DS_E_FORMAT, "%s: unsupported version", path);
  const uint32_t n = rd32(h + 8), F = rd32(h + 12), C = rd32(h + 16);
  const uint64_t seed = static_cast<uint64_t>(rd32(h + 20)) | static_cast<uint64_t>(rd32(h + 24)) << 32;
  if (n == 0) return set_error(DS_E_FORMAT, "%s: empty shard", path);
  if (F == 0 || C == 0) return set_error(DS_E_FORMAT, "%s: zero dimension", path);
  if (F > (UINT64_MAX - 4) / 4 || n > UINT64_MAX / (4ull * F + 4ull))
    return set_error(DS_E_FORMAT, "%s: dimension overflow", path);
  const uint64_t want = kHeaderBytes + static_cast<uint64_t>(n) * (4ull * F + 4ull);  // dshd::file_size
  if (size != want)
    return set_error(DS_E_FORMAT, "%s: size mismatch (header implies %llu bytes, file has %llu bytes)", path,
                     static_cast<unsigned long long>(want), static_cast<unsigned long long>(size));
  info->n_samples = n;
  info->n_features = F;
  info->n_classes = C;
  info->seed = seed;
  return DS_OK;
}

// One warp per row: the F feature words go to X (coalesced on both sides; rows are
// 4(F+1)-byte strided in the file so no wider vector width is aligned in general), lane 0
// moves the label and range-checks it. HBM-bound: 8(F+1) bytes per row.
__global__ void __launch_bounds__(kUnpackThreads) dshd_unpack_kernel(const uint32_t* __restrict__ raw, uint64_t rows,
                                                                     uint32_t F, uint32_t C, uint64_t row0,
                                                                     float* __restrict__ X, uint32_t* __restrict__ y,
                                                                     unsigned long long* __restrict__ first_bad) {
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kUnpackThreads / 32);
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = blockIdx.x * (kUnpackThreads / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const uint32_t* src = raw + r * (F + 1ull);
    uint32_t* dst = reinterpret_cast<uint32_t*>(X) + (row0 + r) * F;
    for (uint32_t j = lane; j < F; j += 32) dst[j] = __ldcs(src + j);
    if (lane == 0) {
      const uint32_t label = __ldcs(src + F);
      y[row0 + r] = label;
      if (label >= C) atomicMin(first_bad, static_cast<unsigned long long>(row0 + r));
    }
  }
}

}  // namespace
}  // namespace dsb

using dsb::set_error;

extern "C" int ds_shard_info_read(const char* path, ds_shard_info* info) {
  if (!path || !info) return set_error(DS_E_CONTRACT, "shard: null argument");
  dsb::Fd f;
  return dsb::read_header(path, f, info);
}

extern "C" int ds_shard_load(const char* path, float* X_dev, uint32_t* y_dev, uint64_t capacity_rows,
                             ds_shard_info* info_out, void* stream) {
  if (!path || !X_dev || !y_dev) return set_error(DS_E_CONTRACT, "shard: null argument");
  dsb::Fd f;
  ds_shard_info info{};
  DS_TRY(dsb::read_header(path, f, &info));
  if (info.n_samples > capacity_rows)
    return set_error(DS_E_CONTRACT, "shard: %s holds %u rows, destination has room for %llu", path, info.n_samples,
                     static_cast<unsigned long long>(capacity_rows));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t row_bytes = 4ull * info.n_features + 4ull;
  const uint64_t chunk_rows = std::max<uint64_t>(1, dsb::kChunkBytes / row_bytes);
  const uint64_t slot_bytes = std::min<uint64_t>(chunk_rows, info.n_samples) * row_bytes;
  int dev = 0;
  DS_CUDA_TRY(cudaGetDevice(&dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  struct Slots {
    void* host[2] = {nullptr, nullptr};
    void* staging[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    unsigned long long* bad = nullptr;
    ~Slots() {
      for (int k = 0; k < 2; ++k) {
        if (done[k]) cudaEventSynchronize(done[k]), cudaEventDestroy(done[k]);
        if (host[k]) cudaFreeHost(host[k]);
        if (staging[k]) cudaFree(staging[k]);
      }
      if (bad) cudaFree(bad);
    }
  } sl;
  for (int k = 0; k < 2; ++k) {
    DS_CUDA_TRY(cudaHostAlloc(&sl.host[k], slot_bytes, cudaHostAllocDefault));
    DS_CUDA_TRY(cudaMalloc(&sl.staging[k], slot_bytes));
    DS_CUDA_TRY(cudaEventCreateWithFlags(&sl.done[k], cudaEventDisableTiming));
  }
  DS_CUDA_TRY(cudaMalloc(&sl.bad, sizeof(unsigned long long)));
  DS_CUDA_TRY(cudaMemsetAsync(sl.bad, 0xFF, sizeof(unsigned long long), s));
  bool recorded[2] = {false, false};
  uint64_t c = 0;
  for (uint64_t r0 = 0; r0 < info.n_samples; r0 += chunk_rows, ++c) {
    const int k = static_cast<int>(c & 1);
    const uint64_t rows = std::min<uint64_t>(chunk_rows, info.n_samples - r0);
    if (recorded[k]) DS_CUDA_TRY(cudaEventSynchronize(sl.done[k]));  // the slot's previous H2D finished
    if (!dsb::pread_parallel(f.fd, sl.host[k], rows * row_bytes, dsb::kHeaderBytes + r0 * row_bytes))
      return set_error(DS_E_IO, "read failed for %s", path);
    DS_CUDA_TRY(cudaMemcpyAsync(sl.staging[k], sl.host[k], rows * row_bytes, cudaMemcpyHostToDevice, s));
    DS_CUDA_TRY(cudaEventRecord(sl.done[k], s));
    recorded[k] = true;
    const uint64_t want_blocks = (rows + dsb::kUnpackThreads / 32 - 1) / (dsb::kUnpackThreads / 32);
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>(want_blocks, 8ull * sms));
    dsb::dshd_unpack_kernel<<<blocks, dsb::kUnpackThreads, 0, s>>>(static_cast<const uint32_t*>(sl.staging[k]), rows,
                                                                    info.n_features, info.n_classes, r0, X_dev, y_dev,
                                                                    sl.bad);
    DS_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long bad = 0;
  DS_CUDA_TRY(cudaMemcpyAsync(&bad, sl.bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
  DS_CUDA_TRY(cudaStreamSynchronize(s));
  if (bad != ~0ull) {
    uint32_t label = 0;
    DS_CUDA_TRY(cudaMemcpy(&label, y_dev + bad, sizeof(label), cudaMemcpyDeviceToHost));
    return set_error(DS_E_FORMAT, "%s: label %u out of range at sample %llu", path, label, bad);
  }
  if (info_out) *info_out = info;
  return DS_OK;
}
