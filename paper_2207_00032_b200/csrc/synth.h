// Synthetic weights: a pure function of (seed, layer, tensor, flat row-major index) so the
// device generator, the host generator and the CPU oracle (oracle/oracle.c) produce the
// same fp16 bits with no checkpoint and no host->device weight copy.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define DSINF_HD __host__ __device__ __forceinline__
#else
#define DSINF_HD inline
#endif

namespace dsinf {

DSINF_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Per-tensor stream base.
DSINF_HD uint64_t synth_base(uint64_t seed, int32_t layer, int32_t tensor) {
  return splitmix64(seed ^ (0x51ED2701ull * static_cast<uint64_t>(layer + 1)) ^
                    (static_cast<uint64_t>(tensor) << 56));
}

// Uniform in [-1, 1) with 24-bit resolution, exact in fp32.
DSINF_HD float synth_unit(uint64_t base, uint64_t flat) {
  const uint64_t h = splitmix64(base + flat);
  const int32_t u24 = static_cast<int32_t>(h >> 40);           // [0, 2^24)
  return static_cast<float>(2 * u24 - (1 << 24)) * (1.0f / 16777216.0f);
}

// Amplitudes a with w = unit * a (std = a / sqrt(3)).
struct SynthScale {
  static constexpr float kWeight = 0.034641016f;  // 0.02 * sqrt(3): std 0.02
  static constexpr float kBias = 0.017320508f;    // 0.01 * sqrt(3): std 0.01
  static constexpr float kLnGamma = 0.1f;         // gamma = 1 + U(-0.1, 0.1)
  static constexpr float kLnBeta = 0.05f;         // beta = U(-0.05, 0.05)
};

// fp32 -> fp16 bits, round to nearest even (host side; the device uses __float2half_rn).
inline uint16_t f32_to_f16_bits(float f) {
  union {
    float f;
    uint32_t u;
  } v{f};
  const uint32_t x = v.u;
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t absx = x & 0x7fffffffu;
  if (absx >= 0x7f800000u) return static_cast<uint16_t>(sign | (absx > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (absx >= 0x477ff000u) return static_cast<uint16_t>(sign | 0x7c00u);  // rounds to inf
  if (absx < 0x38800000u) {  // subnormal half (or zero)
    if (absx < 0x33000000u) return static_cast<uint16_t>(sign);  // < 2^-25 -> 0 (RNE)
    const uint32_t e = absx >> 23;
    const uint32_t m = (absx & 0x7fffffu) | 0x800000u;
    const uint32_t shift = 126 - e;  // 14 - (e - 112) + ...: value = m * 2^(e-150); half sub unit 2^-24
    // half subnormal mantissa = m * 2^(e-150) / 2^-24 = m >> (126 - e)
    uint32_t q = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    return static_cast<uint16_t>(sign | q);
  }
  uint32_t hbits = ((absx >> 23) - 112) << 10 | ((absx >> 13) & 0x3ffu);
  const uint32_t rem = absx & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (hbits & 1u))) ++hbits;
  return static_cast<uint16_t>(sign | hbits);
}

inline float f16_bits_to_f32(uint16_t h) {
  const uint32_t sign = (h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu;
  const uint32_t m = h & 0x3ffu;
  uint32_t out;
  if (e == 0) {
    if (m == 0) {
      out = sign;
    } else {  // subnormal: m * 2^-24
      float f = static_cast<float>(m) * (1.0f / 16777216.0f);
      union {
        float f;
        uint32_t u;
      } v{f};
      out = sign | v.u;
    }
  } else if (e == 31) {
    out = sign | 0x7f800000u | (m << 13);
  } else {
    out = sign | ((e + 112) << 23) | (m << 13);
  }
  union {
    uint32_t u;
    float f;
  } r{out};
  return r.f;
}

}  // namespace dsinf
