// host_rows.cpp — the host half of the tensor-core stream mode: gather_batch
// (model.cpp:12-21) of a step's rows from the host shard, cast to bf16 on the way into the
// zero-copy ring. Compiled by g++ into libds_cuda.so (not nvcc: the AVX-512 path uses
// target-specific intrinsics, dispatched at run time).
//
// Bits: round to nearest even, NaN -> 0x7FFF, denormals kept — exactly the device's
// __float2bfloat16_rn (cvt.rn.bf16.f32). AVX512-BF16's vcvtne2ps2bf16 rounds the same way
// for normal numbers but treats denormal inputs as zero and keeps NaN payloads, so a
// 32-float chunk that holds a zero-exponent or all-ones-exponent value takes the scalar path.
#include <immintrin.h>

#include <cstdint>
#include <cstring>

namespace dsb {

namespace {

inline uint16_t bf16_rn(uint32_t u) {
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFu;
  return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

void row_scalar(const float* src, uint32_t F, uint16_t* dst) {
  for (uint32_t f = 0; f < F; ++f) {
    uint32_t u;
    std::memcpy(&u, src + f, 4);
    dst[f] = bf16_rn(u);
  }
}

__attribute__((target("avx512f,avx512bw,avx512vl,avx512bf16"))) void row_avx512(const float* src, uint32_t F,
                                                                                 uint16_t* dst) {
  const __m512i expmask = _mm512_set1_epi32(0x7F800000);
  uint32_t f = 0;
  for (; f + 32 <= F; f += 32) {
    const __m512 a = _mm512_loadu_ps(src + f), b = _mm512_loadu_ps(src + f + 16);
    const __m512i ea = _mm512_and_si512(_mm512_castps_si512(a), expmask);
    const __m512i eb = _mm512_and_si512(_mm512_castps_si512(b), expmask);
    // special: exponent 0 (zero/denormal: zero is fine either way, denormals are not) or 0xFF
    const __mmask16 sa = _mm512_cmpeq_epi32_mask(ea, _mm512_setzero_si512()) | _mm512_cmpeq_epi32_mask(ea, expmask);
    const __mmask16 sb = _mm512_cmpeq_epi32_mask(eb, _mm512_setzero_si512()) | _mm512_cmpeq_epi32_mask(eb, expmask);
    if ((sa | sb) == 0) {
      _mm512_storeu_si512(reinterpret_cast<void*>(dst + f), reinterpret_cast<__m512i>(_mm512_cvtne2ps_pbh(b, a)));
    } else {
      row_scalar(src + f, 32, dst + f);
    }
  }
  row_scalar(src + f, F - f, dst + f);
}

const bool kAvx512Bf16 = __builtin_cpu_supports("avx512bf16") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("avx512vl");

}  // namespace

// rows x F floats, row r from X + idx[r] * F (idx == nullptr: X is already the batch,
// row r at X + r * F) -> dst rows of `pitch` bf16 (the padding is left as it is)
void gather_rows_bf16_host(const float* X, uint32_t F, const uint32_t* idx, uint32_t rows, uint16_t* dst,
                           uint64_t pitch) {
  for (uint32_t r = 0; r < rows; ++r) {
    const float* src = X + static_cast<uint64_t>(idx ? idx[r] : r) * F;
    if (kAvx512Bf16)
      row_avx512(src, F, dst + r * pitch);
    else
      row_scalar(src, F, dst + r * pitch);
  }
}

}  // namespace dsb

// C-ABI (ds_cuda.h): the host half of the tensor-core stream mode, exported for pipelines
// that stage their own batches (and testable without a GPU)
extern "C" int ds_host_rows_to_bf16(const float* X, uint32_t F, const uint32_t* idx, uint32_t rows, uint16_t* dst,
                                    uint64_t pitch) {
  if (!X || !dst || F == 0 || pitch < F) return 1;  // DS_E_CONTRACT
  dsb::gather_rows_bf16_host(X, F, idx, rows, dst, pitch);
  return 0;
}
