// Block-level pieces shared by the probability kernels (lc_probs.cu) and the
// resample entry's entropy epilogue (lc_resample.cu): element loads, block
// reductions, and the per-row entropy / max probability of softmax(z / T)
// (sampling.py:112-126).
#pragma once
#include <math.h>

#include "lc_common.cuh"

namespace lcb {

constexpr int PB_THREADS = 256;

template <int DT>
__device__ __forceinline__ float ld(const char* row, int64_t i) {
  if (DT == LC_BF16) return bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(row)[i]);
  return reinterpret_cast<const float*>(row)[i];
}

static __device__ __forceinline__ float block_max(float v, float* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = -INFINITY;
  for (int w = 0; w < PB_THREADS / 32; ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

static __device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < PB_THREADS / 32; ++w) r += red[w];
  __syncthreads();
  return r;
}

// H = -sum p ln p = ln S - sum(e*s)/S with s <= 0 the shifted scaled logits;
// pmax = max p = 1/S (sampling.py:112-126).
// one block per row: H = log S - sum(e s) / S and max p = 1 / S of softmax(z / T), fp64
template <int DT>
__device__ __forceinline__ void entropy_row(const char* row, int64_t V, double T, double* H, double* pmax) {
  __shared__ float fred[PB_THREADS / 32];
  __shared__ double dred[PB_THREADS / 32];
  float m = -INFINITY;
  for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) m = fmaxf(m, ld<DT>(row, i));
  m = block_max(m, fred);
  if (T == 0.0) {
    if (threadIdx.x == 0) {
      *H = 0.0;
      *pmax = 1.0;
    }
    return;
  }
  const double mT = __ddiv_rn((double)m, T);
  double se = 0.0, ses = 0.0;
  for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) {
    double s = __dsub_rn(__ddiv_rn((double)ld<DT>(row, i), T), mT);
    double e = exp(s);
    se += e;
    if (e > 0.0) ses += e * s;
  }
  se = block_sum(se, dred);
  ses = block_sum(ses, dred);
  if (threadIdx.x == 0) {
    *H = log(se) - ses / se;
    *pmax = 1.0 / se;
  }
}

}  // namespace lcb
