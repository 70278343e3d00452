// Probability-level entry points of the reference sampler API
// (sampling.py:57-126): softmax into fp64 probabilities, the inverse-CDF draw
// on an explicit probability vector, and the per-row entropy / max-prob used by
// hotspot scoring.  These serve the drop-in Python functions
// (paper_2604_17353_b200.sampling); the hot path is the fused lc_resample.
#include <math.h>

#include "lc_common.cuh"
#include "lc_numpy.cuh"
#include "lc_probs.cuh"

namespace lcb {

constexpr int PB_LEAVES = 2048;  // numpy pairwise-tree leaves summed in parallel (V <~ 130K; beyond: sequential)

struct PbShared {
  int2 lv[PB_LEAVES];
  double ls[PB_LEAVES];
  double bcast;
  int nleaf;
};

// first index i with row[i] == m (block-wide min)
template <int DT>
__device__ int64_t block_first_eq(const char* row, int64_t V, float m, int64_t* red) {
  int64_t a = INT64_MAX;
  for (int64_t i = threadIdx.x; i < V && a == INT64_MAX; i += PB_THREADS)
    if (ld<DT>(row, i) == m) a = i;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t y = __shfl_xor_sync(0xffffffffu, a, o);
    a = y < a ? y : a;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  int64_t r = INT64_MAX;
  for (int w = 0; w < PB_THREADS / 32; ++w) r = red[w] < r ? red[w] : r;
  __syncthreads();
  return r;
}

// softmax: s = f64(z)/T - max (sampling.py:65-66), e = exp(s), p = e / pairwise_sum(e)
template <int DT>
__global__ void __launch_bounds__(PB_THREADS)
softmax_kernel(const char* rows, int64_t row_bytes, int64_t V, const double* temps, double* out) {
  __shared__ float fred[PB_THREADS / 32];
  __shared__ int64_t ired[PB_THREADS / 32];
  __shared__ PbShared pb;
  const char* row = rows + blockIdx.x * row_bytes;
  double* o = out + blockIdx.x * V;
  const double T = temps[blockIdx.x];
  float m = -INFINITY;
  for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) m = fmaxf(m, ld<DT>(row, i));
  m = block_max(m, fred);
  if (T == 0.0) {  // one-hot at the first argmax (sampling.py:61-64)
    const int64_t arg = block_first_eq<DT>(row, V, m, ired);
    for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) o[i] = (i == arg) ? 1.0 : 0.0;
    return;
  }
  const double mT = __ddiv_rn((double)m, T);
  for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) o[i] = exp(__dsub_rn(__ddiv_rn((double)ld<DT>(row, i), T), mT));
  __syncthreads();
  // e.sum() in numpy's pairwise tree: leaves in parallel, the tree combined in order
  const double S = pairwise_block(o, V, pb.lv, pb.ls, PB_LEAVES, &pb.bcast, &pb.nleaf);
  for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) o[i] = __ddiv_rn(o[i], S);
}

// sample(): total = pairwise_sum(q); cdf = sequential cumsum; first index with
// cdf > u*total; clamp to V-1; back off over zeros (sampling.py:97-109).
// One block per row: the total in numpy's pairwise tree (block-parallel); the
// sequential cumsum's crossing is located from per-thread chunk sums (an
// exclusive block scan), then walked inside the owning chunk; the decision is
// certified against the rounding gap between that walk and numpy's sequential
// cumsum (both within (i + 1) 2^-53 * total of the exact prefix), else the
// sequential scan runs on one thread.
__global__ void __launch_bounds__(PB_THREADS)
draw_probs_kernel(const double* probs, int64_t V, int64_t stride, const double* u, int32_t* tok, uint8_t* flags) {
  __shared__ PbShared pb;
  __shared__ double dred[PB_THREADS / 32];
  __shared__ int64_t s_idx;
  __shared__ int s_unc;
  const double* q = probs + blockIdx.x * stride;
  const double total = pairwise_block(q, V, pb.lv, pb.ls, PB_LEAVES, &pb.bcast, &pb.nleaf);
  if (!(total > 0.0)) {
    if (threadIdx.x == 0) {
      tok[blockIdx.x] = -1;
      if (flags) flags[blockIdx.x] = LC_DRAW_BAD_ROW;
    }
    return;
  }
  const double t = u[blockIdx.x] * total;
  const int64_t ch = (V + PB_THREADS - 1) / PB_THREADS;
  const int64_t i0 = min((int64_t)threadIdx.x * ch, V), i1 = min(i0 + ch, V);
  double cs = 0.0;
  for (int64_t i = i0; i < i1; ++i) cs += q[i];
  // exclusive block scan of the chunk sums
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double incl = cs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) dred[w] = incl;
  if (threadIdx.x == 0) {
    s_idx = V;  // "never crossed": the reference clamps to V - 1
    s_unc = 0;
  }
  __syncthreads();
  double pre = incl - cs;
  for (int k = 0; k < w; ++k) pre += dred[k];
  const double eps = 4.0 * (double)(V + 2) * 0x1p-53 * total;  // both cumsums' gap to the exact prefix
  // the chunk whose (approximate) range holds t walks it; chunks near t on either side flag
  if (pre - eps <= t && t < pre + cs + eps && i1 > i0) {
    double c = pre;
    int64_t i = i0;
    for (; i < i1; ++i) {
      c += q[i];
      if (c > t) break;
    }
    if (i < i1) {
      const double cprev = c - q[i];
      if (!(c - t > eps) || !(t - cprev >= eps)) s_unc = 1;
      else atomicMin(reinterpret_cast<unsigned long long*>(&s_idx), (unsigned long long)i);
    } else if (!(t - c >= eps)) {
      s_unc = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t i = s_idx;
    if (s_unc) {  // undecided within the rounding gap: numpy's sequential cumsum
      double c = 0.0;
      for (i = 0; i < V; ++i) {
        c += q[i];
        if (c > t) break;
      }
    }
    if (i >= V) i = V - 1;
    while (i > 0 && q[i] == 0.0) --i;
    tok[blockIdx.x] = (int32_t)i;
    if (flags) flags[blockIdx.x] = 0;
  }
}

// Entropy and max of explicit probability rows (sampling.py:112-126):
// H = -sum_{p > 0} p ln p, pmax = max p (one block per row).
__global__ void __launch_bounds__(PB_THREADS)
prob_stats_kernel(const double* probs, int64_t V, int64_t stride, double* H, double* pmax) {
  __shared__ double dred[PB_THREADS / 32];
  const double* q = probs + blockIdx.x * stride;
  double h = 0.0, mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) {
    const double p = q[i];
    if (p > 0.0) h -= p * log(p);
    mx = fmax(mx, p);
  }
  h = warp_sum(h);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) dred[threadIdx.x >> 5] = h;
  __syncthreads();
  double hs = 0.0;
  for (int k = 0; k < PB_THREADS / 32; ++k) hs += dred[k];
  __syncthreads();
  if ((threadIdx.x & 31) == 0) dred[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = -INFINITY;
    for (int k = 0; k < PB_THREADS / 32; ++k) m = fmax(m, dred[k]);
    H[blockIdx.x] = hs + 0.0;  // (-0 -> +0: a one-hot row has entropy 0.0)
    pmax[blockIdx.x] = m;
  }
}

template <int DT>
__global__ void __launch_bounds__(PB_THREADS)
entropy_kernel(const char* rows, int64_t row_bytes, int64_t V, double T, double* H, double* pmax) {
  entropy_row<DT>(rows + blockIdx.x * row_bytes, V, T, H + blockIdx.x, pmax + blockIdx.x);
}

// rows given by address (slab rows of cached entries, lc_cache_row_entropy); a null
// address (missing row) yields H = 0, max p = 1
template <int DT>
__global__ void __launch_bounds__(PB_THREADS)
entropy_ptr_kernel(const char* const* rows, const int32_t* vocab, double T, double* H, double* pmax) {
  const char* row = rows[blockIdx.x];
  if (!row) {
    if (threadIdx.x == 0) {
      H[blockIdx.x] = 0.0;
      pmax[blockIdx.x] = 1.0;
    }
    return;
  }
  entropy_row<DT>(row, vocab[blockIdx.x], T, H + blockIdx.x, pmax + blockIdx.x);
}

int launch_entropy_ptrs(const char* const* d_rows, const int32_t* d_vocab, int dtype, int64_t n, double T, double* H,
                        double* pmax, cudaStream_t st) {
  if (n <= 0) return LC_OK;
  if (dtype == LC_F32) entropy_ptr_kernel<LC_F32><<<(unsigned)n, PB_THREADS, 0, st>>>(d_rows, d_vocab, T, H, pmax);
  else entropy_ptr_kernel<LC_BF16><<<(unsigned)n, PB_THREADS, 0, st>>>(d_rows, d_vocab, T, H, pmax);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

}  // namespace lcb

using namespace lcb;

extern "C" int lc_softmax(const void* d_rows, int dtype, int64_t vocab, int64_t row_stride, int64_t n_rows,
                          const double* d_temperature, double* d_out, void* stream) {
  if (n_rows < 0 || vocab < 1 || (n_rows > 0 && (!d_rows || !d_temperature || !d_out))) return LC_E_ARG;
  if (n_rows == 0) return LC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == LC_F32)
    softmax_kernel<LC_F32><<<(unsigned)n_rows, PB_THREADS, 0, st>>>((const char*)d_rows, row_stride * 4, vocab,
                                                                    d_temperature, d_out);
  else if (dtype == LC_BF16)
    softmax_kernel<LC_BF16><<<(unsigned)n_rows, PB_THREADS, 0, st>>>((const char*)d_rows, row_stride * 2, vocab,
                                                                     d_temperature, d_out);
  else
    return LC_E_ARG;
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_draw_probs(const double* d_probs, int64_t vocab, int64_t n_rows, int64_t row_stride,
                             const double* d_u, int32_t* d_token, uint8_t* d_flags, void* stream) {
  if (n_rows < 0 || vocab < 1 || (n_rows > 0 && (!d_probs || !d_u || !d_token))) return LC_E_ARG;
  if (n_rows == 0) return LC_OK;
  draw_probs_kernel<<<(unsigned)n_rows, PB_THREADS, 0, (cudaStream_t)stream>>>(d_probs, vocab, row_stride, d_u,
                                                                               d_token, d_flags);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_prob_stats(const double* d_probs, int64_t vocab, int64_t n_rows, int64_t row_stride,
                             double* d_entropy, double* d_pmax, void* stream) {
  if (n_rows < 0 || vocab < 1 || (n_rows > 0 && (!d_probs || !d_entropy || !d_pmax))) return LC_E_ARG;
  if (n_rows == 0) return LC_OK;
  prob_stats_kernel<<<(unsigned)n_rows, PB_THREADS, 0, (cudaStream_t)stream>>>(d_probs, vocab, row_stride,
                                                                               d_entropy, d_pmax);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_row_entropy(const void* d_rows, int dtype, int64_t vocab, int64_t row_stride, int64_t n_rows,
                              double temperature, double* d_entropy, double* d_pmax, void* stream) {
  if (n_rows < 0 || vocab < 1 || (n_rows > 0 && (!d_rows || !d_entropy || !d_pmax))) return LC_E_ARG;
  if (n_rows == 0) return LC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == LC_F32)
    entropy_kernel<LC_F32><<<(unsigned)n_rows, PB_THREADS, 0, st>>>((const char*)d_rows, row_stride * 4, vocab,
                                                                    temperature, d_entropy, d_pmax);
  else if (dtype == LC_BF16)
    entropy_kernel<LC_BF16><<<(unsigned)n_rows, PB_THREADS, 0, st>>>((const char*)d_rows, row_stride * 2, vocab,
                                                                     temperature, d_entropy, d_pmax);
  else
    return LC_E_ARG;
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

// truncate() on explicit probabilities (sampling.py:71-94), slow reference-shaped path: kept prefix of the
// (p desc, id asc) order by block-wide argmax steps, sequential csum against
// top_p ('left' cut, inclusive), renormalised by numpy's pairwise sum of the
// kept values in sorted order.  O(V * kept) -- an API-parity path, not the hot
// path (the fused lc_resample never materialises truncated probabilities).
namespace lcb {
// fallback (rows the fast path below cannot take): kept prefix by block-wide argmax steps
__device__ void truncate_row_slow(const double* p, int64_t V, int topk, double topp, double* o, int32_t* ord,
                                  double* val, double* s_bp, int64_t* s_bi) {
  const int64_t lim = (topk > 0 && topk < V) ? topk : V;
  double last_p = INFINITY;
  int64_t last_id = -1, n = 0;
  double c = 0.0;
  while (n < lim) {
    double bp = -INFINITY;
    int64_t bi = INT64_MAX;
    for (int64_t i = threadIdx.x; i < V; i += PB_THREADS) {
      double pi = p[i];
      bool after = (pi < last_p) || (pi == last_p && i > last_id);
      if (after && (pi > bp || (pi == bp && i < bi))) {
        bp = pi;
        bi = i;
      }
    }
    s_bp[threadIdx.x] = bp;
    s_bi[threadIdx.x] = bi;
    __syncthreads();
    for (int s = PB_THREADS / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        double op = s_bp[threadIdx.x + s];
        int64_t oi = s_bi[threadIdx.x + s];
        if (op > s_bp[threadIdx.x] || (op == s_bp[threadIdx.x] && oi < s_bi[threadIdx.x])) {
          s_bp[threadIdx.x] = op;
          s_bi[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    bp = s_bp[0];
    bi = s_bi[0];
    __syncthreads();
    if (bi == INT64_MAX) break;
    if (threadIdx.x == 0) {
      ord[n] = (int32_t)bi;
      val[n] = bp;
    }
    ++n;
    last_p = bp;
    last_id = bi;
    if (topp < 1.0) {
      c += bp;
      if (c >= topp) break;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ks = pairwise_seq(val, n);
    for (int64_t i = 0; i < V; ++i) o[i] = 0.0;
    for (int64_t i = 0; i < n; ++i) o[ord[i]] = __ddiv_rn(val[i], ks);
  }
}
}  // namespace lcb

namespace lcb {
// Fast path of truncate(): a radix select over the order keys of p (8-bit digits from the top,
// per-bin counts and masses) finds a key bound L such that C = {key >= L} -- a prefix of the
// (p desc, id asc) order -- holds the kept set (|C| >= top_k, or mass(C) >= top_p with a margin
// covering the summation-order gap to numpy's sequential cumsum) with |C| <= TR_CAP.  C is
// gathered, sorted (bitonic on (p desc, id asc)), one thread runs numpy's sequential cumsum
// over it (a prefix's csum values depend only on that prefix) and the pairwise-sum normaliser
// over the kept values in sorted order, and the block scatters kept / ks.  Rows it cannot take
// (> TR_CAP values at the boundary, NaN, a mass target above the row's total) take the slow path.
constexpr int TR_CAP = 4096;

struct TrSmem {
  unsigned long long ck[TR_CAP];  // candidate order keys (after the sort: their p values)
  int ci[TR_CAP];                 // candidate ids
  unsigned int hc[256];
  double hm[256];
  double s_bp[PB_THREADS];
  int64_t s_bi[PB_THREADS];
  unsigned long long prefix, lbound;
  long long acnt;
  double amass, ks;
  int pbits, mode, ncand, K;  // mode: 0 refining, 1 bound found, 2 slow path
};

__device__ __forceinline__ unsigned long long tr_key(double p) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(p == 0.0 ? 0.0 : p);  // -0 == +0
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double tr_val(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

__global__ void __launch_bounds__(PB_THREADS)
truncate_probs_kernel(const double* probs, int64_t V, int64_t stride, int topk, double topp, double* out,
                      int32_t* ord_scr, double* val_scr) {
  extern __shared__ __align__(16) unsigned char tr_raw[];
  TrSmem& sm = *reinterpret_cast<TrSmem*>(tr_raw);
  const double* p = probs + blockIdx.x * stride;
  double* o = out + blockIdx.x * stride;
  const int tid = threadIdx.x;
  const long long Ktk = (topk > 0 && topk < V) ? topk : V;
  const bool by_k = Ktk < V, by_p = topp < 1.0;
  const double target = topp * (1.0 + 4.0 * (double)(V + 8) * 0x1p-53);
  if (tid == 0) {
    sm.prefix = 0ull;
    sm.pbits = 0;
    sm.acnt = 0;
    sm.amass = 0.0;
    sm.mode = 0;
    sm.ncand = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 8 && sm.mode == 0; ++pass) {
    const int shift = 56 - 8 * pass;
    const int pbits = sm.pbits;
    const unsigned long long prefix = sm.prefix;
    for (int b = tid; b < 256; b += PB_THREADS) {
      sm.hc[b] = 0u;
      sm.hm[b] = 0.0;
    }
    __syncthreads();
    bool nan = false;
    for (int64_t i = tid; i < V; i += PB_THREADS) {
      const double pi = p[i];
      nan |= pi != pi;
      const unsigned long long k = tr_key(pi);
      if (pbits == 0 || (k >> (64 - pbits)) == prefix) {
        const int b = (int)((k >> shift) & 255ull);
        atomicAdd(&sm.hc[b], 1u);
        atomicAdd(&sm.hm[b], pi);
      }
    }
    nan = __syncthreads_or(nan);
    if (tid == 0) {
      if (nan) {
        sm.mode = 2;
      } else {
        long long c = sm.acnt;
        double m = sm.amass;
        int bs = -1;
        for (int b = 255; b >= 0; --b) {
          c += sm.hc[b];
          m += sm.hm[b];
          if ((by_k && c >= Ktk) || (by_p && m >= target)) {
            bs = b;
            break;
          }
        }
        if (bs < 0) {
          // never reached inside this range: only possible at the top level (target above the
          // row's mass, or no truncation asked): every element is a candidate
          if (pbits == 0 && c <= TR_CAP) {
            sm.mode = 1;
            sm.lbound = 0ull;
          } else {
            sm.mode = 2;
          }
        } else if (c <= TR_CAP) {
          sm.mode = 1;
          sm.lbound = ((prefix << 8) | (unsigned long long)bs) << shift;
          if (pbits > 0) sm.lbound |= 0ull;  // (prefix bits already in place above the digit)
        } else if (pass == 7) {
          sm.mode = 2;  // one value holds more than TR_CAP elements
        } else {
          for (int b = 255; b > bs; --b) {
            sm.acnt += sm.hc[b];
            sm.amass += sm.hm[b];
          }
          sm.prefix = (prefix << 8) | (unsigned long long)bs;
          sm.pbits = pbits + 8;
        }
      }
    }
    __syncthreads();
  }
  if (sm.mode != 1) {
    truncate_row_slow(p, V, topk, topp, o, ord_scr + blockIdx.x * V, val_scr + blockIdx.x * V, sm.s_bp, sm.s_bi);
    return;
  }
  // gather C = {key >= lbound}
  const unsigned long long L = sm.lbound;
  for (int64_t i = tid; i < V; i += PB_THREADS) {
    const unsigned long long k = tr_key(p[i]);
    if (k >= L) {
      const int slot = atomicAdd(&sm.ncand, 1);
      if (slot < TR_CAP) {
        sm.ck[slot] = k;
        sm.ci[slot] = (int)i;
      }
    }
  }
  __syncthreads();
  const int nc = sm.ncand;
  if (nc > TR_CAP) {  // (cannot happen: the count above is exact) -- defensive
    truncate_row_slow(p, V, topk, topp, o, ord_scr + blockIdx.x * V, val_scr + blockIdx.x * V, sm.s_bp, sm.s_bi);
    return;
  }
  int np2 = 1;
  while (np2 < nc) np2 <<= 1;
  for (int i = nc + tid; i < np2; i += PB_THREADS) {  // padding sorts last
    sm.ck[i] = 0ull;
    sm.ci[i] = 0x7fffffff;
  }
  __syncthreads();
  // bitonic sort, "before" = (key desc, id asc) first
  for (int k = 2; k <= np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < np2; i += PB_THREADS) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long ka = sm.ck[i], kb = sm.ck[l];
          const int ia = sm.ci[i], ib = sm.ci[l];
          const bool a_first = ka > kb || (ka == kb && ia < ib);
          const bool asc = (i & k) == 0;  // this block of the network puts "before" first
          if (asc != a_first) {
            sm.ck[i] = kb;
            sm.ck[l] = ka;
            sm.ci[i] = ib;
            sm.ci[l] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  // values in sorted order (in place), then numpy's cumsum cut and pairwise normaliser
  for (int i = tid; i < nc; i += PB_THREADS) sm.ck[i] = (unsigned long long)__double_as_longlong(tr_val(sm.ck[i]));
  __syncthreads();
  if (tid == 0) {
    const double* v = reinterpret_cast<const double*>(sm.ck);
    long long K = Ktk < nc ? Ktk : nc;
    bool ok = Ktk <= nc;
    if (by_p) {
      double c = 0.0;
      long long i = 0;
      for (; i < K; ++i) {
        c += v[i];
        if (c >= topp) break;
      }
      if (i < K) {
        K = i + 1;
        ok = true;
      }  // else: no index reached top_p within the first min(top_k, nc): all top_k kept (ok iff nc >= Ktk)
    }
    sm.K = ok ? (int)K : -1;
    if (ok) sm.ks = pairwise_seq(v, K);
  }
  __syncthreads();
  const int K = sm.K;
  if (K < 0) {
    truncate_row_slow(p, V, topk, topp, o, ord_scr + blockIdx.x * V, val_scr + blockIdx.x * V, sm.s_bp, sm.s_bi);
    return;
  }
  for (int64_t i = tid; i < V; i += PB_THREADS) o[i] = 0.0;
  __syncthreads();
  const double ks = sm.ks;
  const double* v = reinterpret_cast<const double*>(sm.ck);
  for (int i = tid; i < K; i += PB_THREADS) o[sm.ci[i]] = __ddiv_rn(v[i], ks);
}
}  // namespace lcb

extern "C" int lc_truncate_probs(const double* d_probs, int64_t vocab, int64_t n_rows, int64_t row_stride,
                                 int32_t top_k, double top_p, double* d_out, void* d_scratch, void* stream) {
  if (n_rows < 0 || vocab < 1 || (n_rows > 0 && (!d_probs || !d_out || !d_scratch))) return LC_E_ARG;
  if (!(top_p > 0.0 && top_p <= 1.0)) return LC_E_CONFIG;
  if (n_rows == 0) return LC_OK;
  int32_t* ord = (int32_t*)d_scratch;
  double* val = (double*)((char*)d_scratch + ((n_rows * vocab * 4 + 255) & ~255ll));
  static bool attr = false;
  if (!attr) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(lcb::truncate_probs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(lcb::TrSmem)));
    attr = true;
  }
  lcb::truncate_probs_kernel<<<(unsigned)n_rows, lcb::PB_THREADS, sizeof(lcb::TrSmem), (cudaStream_t)stream>>>(
      d_probs, vocab, row_stride, top_k, top_p, d_out, ord, val);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}
