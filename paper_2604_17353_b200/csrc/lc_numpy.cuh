// numpy reduction-order emulation shared by the EXACT tier and the
// probability-level API (softmax / draw on explicit probabilities).
#pragma once
#include "lc_common.cuh"

namespace lcb {

// numpy pairwise_sum emulation: follows numpy's loops_utils.h: n < 8 ->
// sequential from 0.0; n <= 128 -> 8 strided accumulators combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail; else split at
// n/2 - (n/2)%8.  Verified against np.sum in tests/test_oracle.py.

static __device__ __noinline__ double pairwise_seq(const double* a, int64_t n) {
  struct Fr {
    int64_t lo, n;
    int state;
    double left;
  };
  Fr st[48];
  int sp = 0;
  double ret = 0.0;
  st[sp++] = {0, n, 0, 0.0};
  while (sp > 0) {
    Fr& f = st[sp - 1];
    if (f.n < 8) {
      double r = 0.0;
      for (int64_t i = 0; i < f.n; ++i) r += a[f.lo + i];
      ret = r;
      --sp;
      continue;
    }
    if (f.n <= 128) {
      double r[8];
      for (int j = 0; j < 8; ++j) r[j] = a[f.lo + j];
      int64_t i = 8;
      for (; i < f.n - (f.n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += a[f.lo + i + j];
      double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < f.n; ++i) res += a[f.lo + i];
      ret = res;
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp++] = {f.lo, n2, 0, 0.0};
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp++] = {f.lo + n2, f.n - n2, 0, 0.0};
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}


// One pairwise leaf (n <= 128): numpy's unrolled block, or the short sequential sum.
static __device__ __forceinline__ double pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

// Walk numpy's pairwise tree over [0, n).  LIST: write the first cap leaves
// (lo, n) in order to lv and their total count to *nleaves; else combine the
// leaf sums ls[] in the tree's order and return the total.
template <bool LIST>
static __device__ __noinline__ double pairwise_walk(int64_t n, int2* lv, const double* ls, int cap, int* nleaves) {
  struct Fr {
    int64_t lo, n;
    int state;
    double left;
  };
  Fr st[48];
  int sp = 0, k = 0;
  double ret = 0.0;
  st[sp++] = {0, n, 0, 0.0};
  while (sp > 0) {
    Fr& f = st[sp - 1];
    if (f.n <= 128) {
      if (LIST) {
        if (k < cap) lv[k] = make_int2((int)f.lo, (int)f.n);
      } else {
        ret = ls[k];
      }
      ++k;
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp++] = {f.lo, n2, 0, 0.0};
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp++] = {f.lo + n2, f.n - n2, 0, 0.0};
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  if (LIST) *nleaves = k;
  return ret;
}

// Block-cooperative pairwise_seq (same tree, same roundings): thread 0 lists the
// leaves, the block sums them in parallel, thread 0 combines them in order.
// Every thread of the block must call it; all get the result.  lv/ls hold cap
// leaves (shared memory); beyond that, thread 0 runs pairwise_seq.
static __device__ double pairwise_block(const double* a, int64_t n, int2* lv, double* ls, int cap, double* bcast,
                                        int* icnt) {
  if (threadIdx.x == 0) pairwise_walk<true>(n, lv, nullptr, cap, icnt);
  __syncthreads();
  const int nl = *icnt;
  double r = 0.0;
  if (nl <= cap) {
    for (int i = threadIdx.x; i < nl; i += blockDim.x) ls[i] = pairwise_leaf(a + lv[i].x, lv[i].y);
    __syncthreads();
    if (threadIdx.x == 0) *bcast = pairwise_walk<false>(n, nullptr, ls, cap, nullptr);
  } else if (threadIdx.x == 0) {
    *bcast = pairwise_seq(a, n);
  }
  __syncthreads();
  r = *bcast;
  __syncthreads();
  return r;
}

}  // namespace lcb
