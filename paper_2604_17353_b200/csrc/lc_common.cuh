// Shared device primitives for the B200 logits-cache re-sampling path.
//
// Bit-exact 64-bit mixing follows the reference contract
// (pkg/docs/determinism.md:14-92, pkg/src/agentserve/mixing.py:43-105).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/lc_b200.h"

namespace lcb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;   // mixing.py:29
constexpr uint64_t kMult1 = 0xBF58476D1CE4E5B9ull;    // mixing.py:30
constexpr uint64_t kMult2 = 0x94D049BB133111EBull;    // mixing.py:31
constexpr uint64_t kEmptyHash = 0xA0761D6478BD642Full; // mixing.py:34
constexpr uint64_t kPeakSalt = 0x8BB84B93962EACC9ull;  // mixing.py:36
constexpr uint64_t kSamplerSalt = 0x2545F4914F6CDD1Dull; // mixing.py:38

__host__ __device__ __forceinline__ uint64_t avalanche64(uint64_t z) {
  z ^= z >> 30;
  z *= kMult1;
  z ^= z >> 27;
  z *= kMult2;
  z ^= z >> 31;
  return z;
}

__host__ __device__ __forceinline__ uint64_t stream_u64(uint64_t state, uint64_t i) {
  return avalanche64(state + (i + 1) * kGolden);
}

__host__ __device__ __forceinline__ double unit_float(uint64_t u) {
  return (double)(u >> 11) * 0x1.0p-53;  // exact: 53-bit integer times 2^-53
}

// mix2(a, b) = avalanche64(avalanche64(a) ^ b)  (mixing.py:76-78)
__host__ __device__ __forceinline__ uint64_t mix2(uint64_t a, uint64_t b) { return avalanche64(avalanche64(a) ^ b); }

__host__ __device__ __forceinline__ uint64_t fold_token(uint64_t h, int64_t t) {
  return avalanche64(h ^ (uint64_t)(t + 1));
}

// RngStream(seed)'s i-th next_float() (mixing.py:91-98).
__host__ __device__ __forceinline__ double request_uniform(uint64_t seed, uint64_t i) {
  return unit_float(stream_u64(avalanche64(seed ^ kSamplerSalt), i));
}

// ---- small utilities -------------------------------------------------------------

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

// fp32 -> bf16 round-to-nearest-even (NaN kept quiet).
__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// One element of the synthetic producer row (kernels.py:47-60, _mixcore.pyx:27-40):
// base_v = f32((2*unit_float(stream_u64(state, v)) - 1) * r) evaluated in f64 (no FMA
// contraction: __dmul_rn/__dsub_rn keep the reference's two roundings), then the peak
// element += f32(c*r) in f32; bf16 outputs are the RNE of that fp32 value.
template <typename OutT>
__device__ __forceinline__ OutT producer_value(uint64_t st, int64_t v, uint64_t peak, float boost, double range) {
  const double x = unit_float(stream_u64(st, (uint64_t)v));
  float f = (float)__dmul_rn(__dsub_rn(__dmul_rn(2.0, x), 1.0), range);
  if ((uint64_t)v == peak) f = __fadd_rn(f, boost);
  if constexpr (sizeof(OutT) == 4) return f;
  else return f32_to_bf16_bits(f);
}

// One producer row, 8 consecutive elements per thread per step (one 16-byte store per 8 bf16,
// two per 8 f32): the same values as producer_value (bit-identical), cheaper per element --
// the stream counter advances by one 64-bit add per element instead of a 64-bit multiply, and
// f32((2 u - 1) r) is one exact int64 -> f64 conversion of 2k - 2^53 (k = the top 53 bits)
// times the exact power-of-two scaling 2^-53 r: the same real number as the reference's
// fl(fl(2x) - 1) * r (both prior steps exact), so the same single rounding.
template <typename OutT>
__device__ __forceinline__ void produce_row(OutT* __restrict__ o, int64_t vocab, uint64_t st, uint64_t peak,
                                            float boost, double range, int64_t t0, int64_t nt) {
  // (2k - 2^53) c == fma(k, 2c, -range) exactly (2^53 c == range: c is a power-of-two scaling of
  // range, exact unless range is tiny), so one DFMA of the unsigned top 53 bits gives the same
  // single rounding as the DMUL of the signed 2k - 2^53 -- with fewer 64-bit integer ops
  const double c2 = range * 0x1p-52;
  const bool vec = (reinterpret_cast<uintptr_t>(o) & 15) == 0 && fabs(range) >= 0x1p-900;
  const int64_t ng = vec ? vocab / 8 : 0;
  for (int64_t g = t0; g < ng; g += nt) {
    const int64_t v0 = 8 * g;
    uint64_t x = st + (uint64_t)(v0 + 1) * kGolden;
    const uint64_t pk = peak - (uint64_t)v0;
    const uint32_t pj = pk < 8 ? (uint32_t)pk : 8u;  // the peak's place in this group (8: none)
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t u = avalanche64(x);
      x += kGolden;
      f[j] = (float)__fma_rn((double)(u >> 11), c2, -range);
      if (pj == (uint32_t)j) f[j] = __fadd_rn(f[j], boost);
    }
    if constexpr (sizeof(OutT) == 4) {
      float4* q = reinterpret_cast<float4*>(o + v0);
      q[0] = make_float4(f[0], f[1], f[2], f[3]);
      q[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else {
      // round-to-nearest-even pairs in one instruction (F2FP.BF16.F32.PACK_AB): the values are
      // finite, where this equals f32_to_bf16_bits
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[j]) : "f"(f[2 * j + 1]), "f"(f[2 * j]));
      *reinterpret_cast<uint4*>(o + v0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  for (int64_t v = 8 * ng + t0; v < vocab; v += nt) o[v] = producer_value<OutT>(st, v, peak, boost, range);
}

// Monotone map float -> uint32 (larger float -> larger key; -0 < +0 handled as
// equal magnitude ordering is irrelevant because -0 == +0 never both matter).
__device__ __forceinline__ uint32_t f32_order_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_min_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ex2.approx.ftz.f32 -- the MUFU exponential (SFU pipe).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2): two independent IEEE round-to-nearest operations
// per instruction, bit-identical to two fmaf / adds.
__device__ __forceinline__ float2 ffma2_rn(float2 a, float b, float c) {  // (a.x b + c, a.y b + c)
  float2 r;
  asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %4};\n mov.b64 c, {%5, %5};\n"
      " fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float2 fadd2_rn(float2 a, float2 b) {  // (a.x + b.x, a.y + b.y)
  float2 r;
  asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n add.rn.f32x2 d, a, b;\n"
      " mov.b64 {%0, %1}, d;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// general packed pair forms (every operand a pair; a broadcast is make_float2(x, x))
#define LCB_F2OP(name, op)                                                                             \
  __device__ __forceinline__ float2 name(float2 a, float2 b) {                                         \
    float2 r;                                                                                          \
    asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n " op                \
        " d, a, b;\n mov.b64 {%0, %1}, d;\n}"                                                         \
        : "=f"(r.x), "=f"(r.y)                                                                         \
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                                     \
    return r;                                                                                          \
  }
LCB_F2OP(f2add, "add.rn.f32x2")
LCB_F2OP(f2sub, "sub.rn.f32x2")
LCB_F2OP(f2mul, "mul.rn.f32x2")
#undef LCB_F2OP
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {  // a * b + c, one rounding per lane
  float2 r;
  asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n mov.b64 c, {%6, %7};\n"
      " fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace lcb

#define LCB_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) {                                 \
      lcb_set_last_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
      return LC_E_CUDA;                                      \
    }                                                        \
  } while (0)

void lcb_set_last_error(const char* msg, const char* file, int line);
