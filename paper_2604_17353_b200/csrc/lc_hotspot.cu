// Hotspot scoring and selection on the device (reference
// sampling.py:112-160, logits_cache.py:153-183, engine.py:312).
//
// Scores live beside the rows: every slab row carries b = H * (1 - pmax) of
// softmax(z / T) (sampling.py:112-130 without the decay), a bound on |b - b_ref|
// (b_ref: the reference's numpy evaluation of the same row) and the temperature T
// it was computed at.  A row write (insert copy, producer fill, engine decode)
// invalidates it; the replayed prefix a write-back keeps in place keeps its scores.
//
//   score_rows     one block per cached row, fp64: s_i = fl(fl(z_i / T) - fl(m / T))
//                  exactly as numpy (sampling.py:65-66), e_i = exp(s_i), S = sum e,
//                  H = log S - (sum e_i s_i) / S (= -sum p log p), pmax = 1 / S;
//   select         one block per entry: s_t = b_t / (1 + decay t) (sampling.py:130),
//                  min-max normalisation, `norm > threshold`, the (-norm, t) cap
//                  (sampling.py:133-145), every decision certified against the score
//                  bounds -- an undecidable one flags the entry -- and the replay's
//                  draw-index layout: draw number of hotspot t = hotspots before t.
#include <math.h>

#include "lc_b200.h"
#include "lc_cache.cuh"
#include "lc_common.cuh"

namespace lcb {

const CacheDev* cache_dev(const lc_cache* c);

constexpr int HS_THREADS = 256;
constexpr double kU = 0x1p-53;

__device__ __forceinline__ double hs_block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int w = 0; w < HS_THREADS / 32; ++w) r += red[w];
  __syncthreads();
  return r;
}

__device__ __forceinline__ float hs_block_max(float v, float* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = -INFINITY;
#pragma unroll
  for (int w = 0; w < HS_THREADS / 32; ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

template <typename DT>
__device__ __forceinline__ float hs_ld(const DT* row, int64_t i) {
  if constexpr (sizeof(DT) == 2) return bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(row)[i]);
  else return reinterpret_cast<const float*>(row)[i];
}

// b and its bound for one row (block-wide; the result is valid in thread 0).
// Bound (DESIGN.md f2): the reference sums pairwise (gamma = (log2 V + 2) u), we sum
// ~V/256 terms per thread then a tree (gamma_o = (V/256 + 16) u); exp/log differ by
// <= 2 ulp; H = log S - X/S and -sum p log p agree to
//   |dH| <= (8u + 2 gamma)(H + 1) + (gamma_o + u)(1 + 2 (H + |log S|)),
// pmax = 1/S to pmax (gamma + gamma_o + 2u); b = H (1 - pmax) adds H |dpmax| + u b.
// An exactly one-hot row (S == 1, X == 0: every other e underflows) is exact: b = 0.
template <typename DT>
__device__ void score_row(const DT* row, int64_t V, double T, double* b_out, double* err_out, double* red,
                          float* fred) {
  float m = -INFINITY;
  bool nan = false;
  for (int64_t i = threadIdx.x; i < V; i += HS_THREADS) {
    const float z = hs_ld(row, i);
    nan |= z != z;
    m = fmaxf(m, z);
  }
  m = hs_block_max(m, fred);
  const double anynan = hs_block_sum(nan ? 1.0 : 0.0, red);
  if (T == 0.0 || anynan > 0.0 || !(m > -INFINITY) || !(m < INFINITY)) {
    // T == 0: softmax is a one-hot (sampling.py:61-64): H = 0, pmax = 1, b = 0 exactly;
    // a NaN / infinite row has no trustworthy score (NaN: the selection flags it)
    if (threadIdx.x == 0) {
      *b_out = T == 0.0 && anynan == 0.0 ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
      *err_out = 0.0;
    }
    return;
  }
  const double mT = __ddiv_rn((double)m, T);
  double se = 0.0, sx = 0.0;
  for (int64_t i = threadIdx.x; i < V; i += HS_THREADS) {
    const double s = __dsub_rn(__ddiv_rn((double)hs_ld(row, i), T), mT);
    const double e = exp(s);
    se += e;
    if (e > 0.0) sx += e * s;
  }
  se = hs_block_sum(se, red);
  sx = hs_block_sum(sx, red);
  if (threadIdx.x == 0) {
    const double lS = log(se);
    const double H = lS - sx / se;
    const double pm = 1.0 / se;
    const double b = H * (1.0 - pm);
    double err = 0.0;
    if (!(se == 1.0 && sx == 0.0)) {
      const double g = (log2((double)V) + 2.0) * kU;
      const double go = ((double)V / HS_THREADS + 16.0) * kU;
      const double Ha = fabs(H);
      const double dH = (8.0 * kU + 2.0 * g) * (Ha + 1.0) + (go + kU) * (1.0 + 2.0 * (Ha + fabs(lS)));
      err = (dH + Ha * pm * (g + go + 2.0 * kU) + kU * fabs(b)) * 1.25;  // 25% slack for the bound's own roundings
    }
    *b_out = b;
    *err_out = err;
  }
}

template <typename DT>
__global__ void __launch_bounds__(HS_THREADS)
score_rows_kernel(CacheDev c, const int32_t* __restrict__ slot, const uint32_t* __restrict__ gen,
                  const int32_t* __restrict__ pos, int64_t n, double T, int only_stale) {
  __shared__ double red[HS_THREADS / 32];
  __shared__ float fred[HS_THREADS / 32];
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const int s = slot[i], t = pos[i];
  if (!row_live(c, s, t, gen, i)) return;
  const int64_t sr = slab_row_of(c, s, t);
  if (only_stale && c.score_T[sr] == T) return;  // (NaN = never scored: always stale)
  double b = 0.0, e = 0.0;
  score_row<DT>(reinterpret_cast<const DT*>(c.slab) + sr * (int64_t)c.V, c.vocab[s], T, &b, &e, red, fred);
  if (threadIdx.x == 0) {
    c.score[sr] = b;
    c.score_err[sr] = e;
    c.score_T[sr] = T;
  }
}

// one block per entry
__global__ void __launch_bounds__(HS_THREADS)
hotspot_select_kernel(CacheDev c, const int32_t* __restrict__ slot, const uint32_t* __restrict__ gen,
                      int64_t n_ent, int max_pos, double T, double decay, double theta, int max_hot,
                      int32_t* __restrict__ draw_index, int32_t* __restrict__ n_hot, uint8_t* __restrict__ flags) {
  extern __shared__ double hs_sm[];
  __shared__ double red[HS_THREADS / 32];
  __shared__ int ired[HS_THREADS / 32 + 1];
  __shared__ int s_flag;
  const int64_t r = blockIdx.x;
  if (r >= n_ent) return;
  const int s = slot[r];
  const bool live = s >= 0 && s < c.E && c.alive[s] && c.gen[s] == gen[r];
  const int n = live ? c.nrows[s] : 0;
  int32_t* di = draw_index ? draw_index + r * (int64_t)max_pos : nullptr;
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  double* sv = hs_sm;       // s_t
  double* se = hs_sm + n;   // its bound
  int* sel = reinterpret_cast<int*>(hs_sm + 2 * n);
  int* drop = sel + n;  // cap decisions, kept apart from sel while other threads still read it
  double lmn = INFINITY, lmx = -INFINITY, lem = 0.0;
  for (int t = threadIdx.x; t < n; t += HS_THREADS) {
    const int64_t sr = slab_row_of(c, s, t);
    const double bt = c.score[sr];
    const double den = 1.0 + decay * (double)t;  // sampling.py:130 (same operation order)
    double v = bt / den;
    double e = c.score_err[sr] / den + 2.0 * kU * fabs(v);
    if (!(c.score_T[sr] == T)) atomicOr(&s_flag, 2);  // not scored at T
    if (v != v) {
      atomicOr(&s_flag, 1);
      v = 0.0;
    }
    sv[t] = v;
    se[t] = e;
    lmn = fmin(lmn, v);
    lmx = fmax(lmx, v);
    lem = fmax(lem, e);
  }
  // block min / max / max error (through the sum helper's scratch: three passes)
  {
    double x = warp_max(-lmn);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double y = -INFINITY;
    for (int w = 0; w < HS_THREADS / 32; ++w) y = fmax(y, red[w]);
    __syncthreads();
    lmn = -y;
    x = warp_max(lmx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    y = -INFINITY;
    for (int w = 0; w < HS_THREADS / 32; ++w) y = fmax(y, red[w]);
    __syncthreads();
    lmx = y;
    x = warp_max(lem);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    y = 0.0;
    for (int w = 0; w < HS_THREADS / 32; ++w) y = fmax(y, red[w]);
    __syncthreads();
    lem = y;
  }
  const double mn = lmn, mx = lmx, emax = lem;
  const double span = mx - mn;
  // span == 0: no hotspots (sampling.py:139-140); certain only if no score could differ
  const bool none = n == 0 || span == 0.0;
  if (n > 0 && span <= 4.0 * emax && emax > 0.0) atomicOr(&s_flag, 1);
  int cnt = 0;
  for (int t = threadIdx.x; t < n; t += HS_THREADS) {
    int k = 0;
    if (!none) {
      const double e = se[t] + emax;
      const double d = sv[t] - mn;
      const double lo = (d - e) * (1.0 - 4.0 * kU), hi = (d + e) * (1.0 + 4.0 * kU);
      const double slo = span - 2.0 * emax, shi = span + 2.0 * emax;
      // reference: norm = (s - min) / span (rounded), keep norm > theta
      const bool above = lo > theta * shi * (1.0 + 4.0 * kU) && lo > 0.0;
      const bool below = hi < theta * (slo > 0.0 ? slo : 0.0) * (1.0 - 4.0 * kU) || (d == 0.0 && se[t] == 0.0 &&
                                                                                     emax == 0.0);
      k = d / span > theta ? 1 : 0;
      if (!above && !below) atomicOr(&s_flag, 1);
    }
    sel[t] = k;
    cnt += k;
  }
  // selected count
  {
    int x = cnt;
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) ired[threadIdx.x >> 5] = x;
    __syncthreads();
    cnt = 0;
    for (int w = 0; w < HS_THREADS / 32; ++w) cnt += ired[w];
    __syncthreads();
  }
  if (max_hot >= 0 && cnt > max_hot) {
    // cap: keep the max_hot best by (-norm, t) (sampling.py:142-144); rank of t among the
    // selected = #{u selected: s_u > s_t or (s_u == s_t and u < t)}
    for (int t = threadIdx.x; t < n; t += HS_THREADS) {
      if (!sel[t]) continue;
      int rank = 0;
      bool close = false;
      for (int u = 0; u < n; ++u) {
        if (!sel[u] || u == t) continue;
        if (sv[u] > sv[t] || (sv[u] == sv[t] && u < t)) ++rank;
        if (fabs(sv[u] - sv[t]) <= se[u] + se[t] && (se[u] + se[t]) > 0.0) close = true;
      }
      drop[t] = rank >= max_hot;  // (sel stays as read by the other threads' ranks)
      // an undecidable order only matters across the cap boundary
      if (close && (rank == max_hot - 1 || rank == max_hot)) atomicOr(&s_flag, 1);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += HS_THREADS)
      if (sel[t] && drop[t]) sel[t] = 0;
    __syncthreads();
    cnt = max_hot;
  }
  __syncthreads();
  // draw numbers: hotspots before t (ascending t), for the replay's positions t < max_pos
  if (di) {
    int carry = 0;
    for (int t0 = 0; t0 < max_pos; t0 += HS_THREADS) {
      const int t = t0 + threadIdx.x;
      const int k = (t < n) ? (sel[t] != 0) : 0;
      int incl = k;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((threadIdx.x & 31) >= o) incl += y;
      }
      if ((threadIdx.x & 31) == 31) ired[threadIdx.x >> 5] = incl;
      __syncthreads();
      int wpre = 0, tot = 0;
      for (int w = 0; w < HS_THREADS / 32; ++w) {
        if (w < (int)(threadIdx.x >> 5)) wpre += ired[w];
        tot += ired[w];
      }
      if (t < max_pos) di[t] = k ? carry + wpre + incl - 1 : -1;
      carry += tot;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    if (n_hot) n_hot[r] = none ? 0 : cnt;
    if (flags) flags[r] = (uint8_t)(s_flag | (live ? 0 : 4));
  }
}

}  // namespace lcb

using namespace lcb;

extern "C" int lc_cache_score_rows(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, const int32_t* d_pos,
                                   int64_t n, double temperature, int32_t only_stale, void* stream) {
  const CacheDev* cd = cache_dev(cache);
  if (!cd || n < 0 || !(temperature >= 0.0) || (n > 0 && (!d_slot || !d_gen || !d_pos))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t i0 = 0; i0 < n; i0 += (1ll << 30)) {
    const int64_t m = n - i0 < (1ll << 30) ? n - i0 : (1ll << 30);
    if (cd->dtype == LC_F32)
      score_rows_kernel<float><<<(unsigned)m, HS_THREADS, 0, st>>>(*cd, d_slot + i0, d_gen + i0, d_pos + i0, m,
                                                                   temperature, only_stale);
    else
      score_rows_kernel<uint16_t><<<(unsigned)m, HS_THREADS, 0, st>>>(*cd, d_slot + i0, d_gen + i0, d_pos + i0, m,
                                                                      temperature, only_stale);
    LCB_CUDA_TRY(cudaGetLastError());
  }
  return LC_OK;
}

extern "C" int lc_cache_hotspots(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, int64_t n_entries,
                                 int32_t max_pos, double temperature, double decay, double threshold,
                                 int32_t max_hotspots, int32_t* d_draw_index, int32_t* d_n_hot, uint8_t* d_flags,
                                 void* stream) {
  const CacheDev* cd = cache_dev(cache);
  if (!cd || n_entries < 0 || max_pos < 0 || !(temperature >= 0.0) || !(decay >= 0.0) ||
      !(threshold >= 0.0 && threshold <= 1.0) || (n_entries > 0 && (!d_slot || !d_gen)))
    return LC_E_ARG;
  if (n_entries == 0) return LC_OK;
  const int max_rows = cd->maxp * cd->page_rows;
  const size_t smem = (size_t)max_rows * (2 * sizeof(double) + 2 * sizeof(int));
  if (smem > 200 * 1024) return LC_E_CONFIG;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(hotspot_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  hotspot_select_kernel<<<(unsigned)n_entries, HS_THREADS, smem, (cudaStream_t)stream>>>(
      *cd, d_slot, d_gen, n_entries, max_pos, temperature, decay, threshold, max_hotspots, d_draw_index, d_n_hot,
      d_flags);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}
