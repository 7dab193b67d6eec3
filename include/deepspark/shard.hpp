// deepspark/shard.hpp — the DSHD on-disk shard format (reference shard.hpp:9-35):
//   28-byte little-endian header: u32 magic 0x44534844, u32 version 1, u32 n_samples,
//   u32 n_features, u32 n_classes, u64 seed; then n_samples x (f32 x n_features, u32 label).
#pragma once

#include <cstdint>
#include <string>

#include "deepspark/dataset.hpp"

namespace deepspark {

namespace dshd {
constexpr uint32_t kMagic = 0x44534844;
constexpr uint32_t kVersion = 1;
constexpr size_t kHeaderSize = 28;
uint64_t file_size(uint32_t n_samples, uint32_t n_features);
}  // namespace dshd

struct ShardData {
  Dataset data;
  uint64_t seed = 0;
};

// Removes the partial file if writing fails.
void write_shard(const Dataset& shard, const std::string& path, uint64_t seed);
// FormatError on bad magic/version/dimensions/size/labels.
ShardData read_shard(const std::string& path);

}  // namespace deepspark
