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


}  // namespace lcb
