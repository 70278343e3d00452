// Device-side layout of a logits-cache handle (lc_cache.cu), shared with the kernels
// that address cached rows directly (lc_engine.cu).
#pragma once
#include <stdint.h>

#include "lc_common.cuh"

namespace lcb {

struct Ctl {
  long long total_bytes;
  long long budget;
  long long clock;
  long long lookups;
  long long hits;
  long long inserts;
  long long evictions;
  long long ring_head;  // positions grow monotonically; index = pos % R
  long long ring_tail;
  int alive;
  int free_slot_top;
  int free_page_top;
  int side_count;
  int error;  // first lc_status raised inside a kernel (sticky until read)
};

struct CacheDev {
  Ctl* ctl;
  uint64_t* hkeys;
  int32_t* hvals;  // slot, -1 empty
  uint32_t hmask;
  uint64_t* digest;
  unsigned long long* last_hit;
  uint32_t* gen;
  int32_t* pins;
  int32_t* nrows;
  int32_t* vocab;
  uint8_t* alive;
  long long* nbytes;
  int32_t* pages;       // [E][maxp]
  int32_t* free_slots;  // stack
  int32_t* free_pages;  // stack
  int32_t* tokens;      // [P * page_rows]
  double* score;        // [P * page_rows] hotspot base score H (1 - pmax) of the row (lc_hotspot.cu)
  double* score_err;    // its bound vs the reference's evaluation
  double* score_T;      // the temperature it was computed at (NaN: none / row rewritten)
  char* slab;           // [P * page_rows * V] of dtype
  unsigned long long* ring_clock;
  int32_t* ring_slot;
  long long R;  // power of two
  long long rmask;
  unsigned long long* side_clock;
  int32_t* side_slot;
  int side_cap;
  int E, P, maxp, page_rows, V, dtype;
};

// slab row index of entry s, position t
__device__ __forceinline__ int64_t slab_row_of(const CacheDev& c, int s, int t) {
  return (int64_t)c.pages[(int64_t)s * c.maxp + t / c.page_rows] * c.page_rows + t % c.page_rows;
}

// (slot, pos[, gen]) names a live row: a handle whose entry was overwritten or evicted
// (generation moved on) reads nothing
__device__ __forceinline__ bool row_live(const CacheDev& c, int s, int t, const uint32_t* gen, int64_t i) {
  return s >= 0 && s < c.E && c.alive[s] && (!gen || c.gen[s] == gen[i]) && t >= 0 && t < c.nrows[s];
}

// a row write makes the row's hotspot score stale
__device__ __forceinline__ void invalidate_score(const CacheDev& c, int64_t sr) {
  c.score_T[sr] = __longlong_as_double(0x7ff8000000000000ll);
}

}  // namespace lcb
