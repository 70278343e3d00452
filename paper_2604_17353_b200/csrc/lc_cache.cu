// K3 (digest -> slot index) + K4 (HBM slab) + the reference's eviction policy.
//
// Reference: pkg/src/agentserve/logits_cache.py
//   lookup            :87-94   lookups += 1; hit -> clock += 1, last_hit = clock, hits += 1
//   update            :96-126  overwrite subtracts old bytes, NEW entry (pins reset),
//                              clock += 1, last_hit = clock, bytes += n*V*4 + 8n
//   _evict_over_budget:128-140 while total > budget and len > 1: evict the unpinned
//                              entry with min (last_hit, digest); stop if all pinned
//   pin / unpin       :145-149
//
// Design:
//   * index: open addressing, linear probing, 2x over-provisioned, probed by
//     tiles of 8 lanes reading 8 consecutive buckets per round; deletion by
//     backward shift (no tombstones);
//   * last_hit values are unique clock ticks, so min (last_hit, digest) is the
//     entry with the oldest tick.  Every tick appends (clock, slot) to an event
//     ring; the ring tail is the LRU end.  An event is live iff the slot is
//     alive and its last_hit still equals the event's clock (lazy deletion).
//     Pinned events met at the tail move to a side list (they are older than
//     everything left in the ring and are re-checked first);
//   * a batch of inserts is applied in index order by one sequential "policy"
//     thread (the semantics are sequential); row copies into the slab run in
//     parallel afterwards, only for entries still alive at the end of the batch;
//   * slots and pages come from LIFO free stacks -- the discipline restated in
//     oracle/cache_ref.py, so slot and page indices are bit-exact vs the oracle.
#include <cub/cub.cuh>
#include <cstdio>
#include <new>
#include <vector>

#include "lc_cache.cuh"
#include "lc_common.cuh"
#include "lc_resample.cuh"
#include "lc_stage.cuh"

namespace lcb {

__device__ __forceinline__ uint32_t home_bucket(uint64_t d, uint32_t mask) {
  return (uint32_t)((d ^ (d >> 29) ^ (d >> 47)) & mask);
}

// ---- lookup ----------------------------------------------------------------------------------

// 8-lane tiles, one key per tile; each round a tile reads 8 consecutive buckets.
__global__ void lookup_probe_kernel(CacheDev c, const uint64_t* __restrict__ dig, int64_t n, int32_t* __restrict__ out) {
  const int64_t key = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  const int lane = threadIdx.x & 31;
  const unsigned tile_bits = 0xffu << (lane & 24);
  const bool active = key < n;
  const uint64_t d = active ? dig[key] : 0ull;
  const uint32_t start = home_bucket(d, c.hmask);
  int result = -1;
  bool done = !active;
  for (uint32_t round = 0; __any_sync(0xffffffffu, !done); ++round) {
    bool match = false, empty = false;
    if (!done) {
      uint32_t b = (start + round * 8u + sub) & c.hmask;
      int32_t v = c.hvals[b];
      match = v >= 0 && c.hkeys[b] == d;
      empty = v < 0;
      if (match) result = v;
      if (round * 8u > c.hmask) empty = true;  // table full safety
    }
    unsigned mm = __ballot_sync(0xffffffffu, match) & tile_bits;
    unsigned em = __ballot_sync(0xffffffffu, empty) & tile_bits;
    if (!done) {
      if (mm) {
        result = __shfl_sync(tile_bits, result, __ffs(mm) - 1, 32);
        done = true;
      } else if (em) {
        // linear probing: the key cannot lie past the first empty bucket --
        // unless a match sits before it inside this round (handled above)
        result = -1;
        done = true;
      }
    }
  }
  if (active && sub == 0) out[key] = result;
}

// In-order commit of a lookup batch: hit ranks -> clock ticks, last_hit, ring events.
__global__ void __launch_bounds__(1024) lookup_commit_kernel(CacheDev c, const int32_t* __restrict__ slot, int64_t n,
                                                             uint32_t* gen_out, int32_t* len_out, int32_t* vocab_out,
                                                             int32_t* slot_out) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long s_clock, s_head;
  if (threadIdx.x == 0) {
    s_clock = c.ctl->clock;
    s_head = c.ctl->ring_head;
  }
  __syncthreads();
  for (int64_t b0 = 0; b0 < n; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int s = i < n ? slot[i] : -1;
    const int hit = s >= 0;
    int rank, total;
    Scan(tmp).ExclusiveSum(hit, rank, total);
    if (hit) {
      const unsigned long long ck = (unsigned long long)(s_clock + rank + 1);
      atomicMax(&c.last_hit[s], ck);
      const long long pos = (s_head + rank) & c.rmask;
      c.ring_clock[pos] = ck;
      c.ring_slot[pos] = s;
    }
    if (i < n) {
      if (slot_out) slot_out[i] = s;
      if (gen_out) gen_out[i] = hit ? c.gen[s] : 0u;
      if (len_out) len_out[i] = hit ? c.nrows[s] : 0;
      if (vocab_out) vocab_out[i] = hit ? c.vocab[s] : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_clock += total;
      s_head += total;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    c.ctl->lookups += n;
    c.ctl->hits += s_clock - c.ctl->clock;
    c.ctl->clock = s_clock;
    c.ctl->ring_head = s_head;
  }
}

// ---- sequential policy thread helpers ------------------------------------------------------

__device__ int table_find(const CacheDev& c, uint64_t d) {
  uint32_t b = home_bucket(d, c.hmask);
  for (uint32_t k = 0; k <= c.hmask; ++k, b = (b + 1) & c.hmask) {
    int v = c.hvals[b];
    if (v < 0) return -1;
    if (c.hkeys[b] == d) return v;
  }
  return -1;
}

__device__ void table_insert(const CacheDev& c, uint64_t d, int s) {
  uint32_t b = home_bucket(d, c.hmask);
  while (c.hvals[b] >= 0) b = (b + 1) & c.hmask;
  c.hkeys[b] = d;
  c.hvals[b] = s;
}

__device__ void table_delete(const CacheDev& c, uint64_t d) {
  uint32_t i = home_bucket(d, c.hmask);
  for (;;) {
    int v = c.hvals[i];
    if (v < 0) return;
    if (c.hkeys[i] == d) break;
    i = (i + 1) & c.hmask;
  }
  uint32_t j = i;
  for (;;) {
    j = (j + 1) & c.hmask;
    if (c.hvals[j] < 0) break;
    uint32_t k = home_bucket(c.hkeys[j], c.hmask);
    bool stays = (i <= j) ? (i < k && k <= j) : (i < k || k <= j);
    if (stays) continue;
    c.hkeys[i] = c.hkeys[j];
    c.hvals[i] = c.hvals[j];
    i = j;
  }
  c.hvals[i] = -1;
}

__device__ __forceinline__ bool event_live(const CacheDev& c, int s, unsigned long long ck) {
  return c.alive[s] && c.last_hit[s] == ck;
}

// Oldest live unpinned entry, consuming it from the side list or the ring tail.
__device__ int next_victim(const CacheDev& c) {
  Ctl* ctl = c.ctl;
  // side list (already in clock order): drop stale entries, take the first unpinned
  int w = 0, found = -1;
  for (int j = 0; j < ctl->side_count; ++j) {
    int s = c.side_slot[j];
    unsigned long long ck = c.side_clock[j];
    if (!event_live(c, s, ck)) continue;
    if (found < 0 && c.pins[s] == 0) {
      found = s;
      continue;
    }
    c.side_slot[w] = s;
    c.side_clock[w] = ck;
    ++w;
  }
  ctl->side_count = w;
  if (found >= 0) return found;
  while (ctl->ring_tail < ctl->ring_head) {
    long long pos = ctl->ring_tail & c.rmask;
    int s = c.ring_slot[pos];
    unsigned long long ck = c.ring_clock[pos];
    ctl->ring_tail++;
    if (!event_live(c, s, ck)) continue;
    if (c.pins[s] > 0) {
      if (ctl->side_count < c.side_cap) {
        c.side_slot[ctl->side_count] = s;
        c.side_clock[ctl->side_count] = ck;
        ctl->side_count++;
      } else {
        ctl->error = LC_E_CAPACITY;  // too many pinned entries to track
      }
      continue;
    }
    return s;
  }
  return -1;
}

__device__ void push_pages(const CacheDev& c, int s) {
  Ctl* ctl = c.ctl;
  for (int k = 0; k < c.maxp; ++k) {
    int pg = c.pages[(int64_t)s * c.maxp + k];
    if (pg < 0) break;
    c.free_pages[ctl->free_page_top++] = pg;
    c.pages[(int64_t)s * c.maxp + k] = -1;
  }
}

// Overwrite: the old entry's pages are pushed in REVERSE page order, so the new entry's
// pops (page 0 first) get them back in place -- page k of the new entry is page k of the
// old one.  A write-back (engine.py:349-361) whose first `keep` rows are the replayed
// prefix of the old entry therefore finds them where they are: no copy (DESIGN.md f3).
__device__ void push_pages_rev(const CacheDev& c, int s) {
  Ctl* ctl = c.ctl;
  int np = 0;
  while (np < c.maxp && c.pages[(int64_t)s * c.maxp + np] >= 0) ++np;
  for (int k = np - 1; k >= 0; --k) {
    c.free_pages[ctl->free_page_top++] = c.pages[(int64_t)s * c.maxp + k];
    c.pages[(int64_t)s * c.maxp + k] = -1;
  }
}

// keep[i] > 0 (write-back): the insert must overwrite the key's live entry whose generation
// is keep_gen[i], with at least keep[i] rows of the same vocab; its first keep[i] rows stay
// in place.  Anything else latches LC_E_STATE (the rows were not copied).
__device__ __forceinline__ bool keep_ok(const CacheDev& c, bool overwrite, int s, uint32_t old_gen, int keep,
                                        uint32_t want_gen, int nr, int vv) {
  return overwrite && old_gen == want_gen && keep <= nr && c.nrows[s] >= keep && c.vocab[s] == vv;
}

__device__ void evict_entry(const CacheDev& c, int s) {
  Ctl* ctl = c.ctl;
  table_delete(c, c.digest[s]);
  ctl->total_bytes -= c.nbytes[s];
  push_pages(c, s);
  c.free_slots[ctl->free_slot_top++] = s;
  c.gen[s] += 1u;
  c.alive[s] = 0;
  ctl->alive -= 1;
  ctl->evictions += 1;
}

// One thread applies the batch in index order (logits_cache.py:96-140).  Kept as the
// reference-shaped A/B path (LCB_SCALAR_POLICY=1) and as the body of the warp kernel's
// rare fallbacks (pinned entries at the LRU end, long probe chains).
__global__ void insert_policy_scalar_kernel(CacheDev c, const uint64_t* __restrict__ dig, const int32_t* __restrict__ lens,
                                     const int32_t* __restrict__ vocabs, int64_t n, int32_t* out_slot,
                                     uint32_t* out_gen, const int32_t* __restrict__ keep,
                                     const uint32_t* __restrict__ keep_gen) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Ctl* ctl = c.ctl;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t d = dig[i];
    const int nr = lens[i];
    const int vv = vocabs[i];
    const int np = (nr + c.page_rows - 1) / c.page_rows;
    out_slot[i] = -1;
    out_gen[i] = 0;
    if (nr < 0 || vv < 1 || vv > c.V || np > c.maxp) {
      if (!ctl->error) ctl->error = LC_E_CONFIG;
      continue;
    }
    const long long bytes = (long long)nr * vv * 4 + 8ll * nr;  // logits_cache.py:54-56
    int s = table_find(c, d);
    if (keep && keep[i] > 0 && !keep_ok(c, s >= 0, s, s >= 0 ? c.gen[s] : 0u, keep[i], keep_gen[i], nr, vv)) {
      if (!ctl->error) ctl->error = LC_E_STATE;
    }
    if (s >= 0) {  // overwrite: the key keeps its slot, the entry is new
      ctl->total_bytes -= c.nbytes[s];
      push_pages_rev(c, s);
      c.gen[s] += 1u;
    } else {
      if (ctl->free_slot_top == 0) {
        if (!ctl->error) ctl->error = LC_E_CAPACITY;
        continue;
      }
      s = c.free_slots[--ctl->free_slot_top];
      table_insert(c, d, s);
      c.alive[s] = 1;
      ctl->alive += 1;
    }
    if (ctl->free_page_top < np) {
      // out of slab pages (possible when entries narrower than the slab make the accounted
      // budget admit more rows than the slab holds): roll the insert back -- the key leaves
      // the index (an overwritten entry is already gone, as in the reference), its slot goes
      // back on the free stack -- and latch the error (oracle/cache_ref.py does the same)
      if (!ctl->error) ctl->error = LC_E_CAPACITY;
      table_delete(c, d);
      c.free_slots[ctl->free_slot_top++] = s;
      c.alive[s] = 0;
      c.nrows[s] = 0;
      c.nbytes[s] = 0;
      ctl->alive -= 1;
      continue;
    }
    for (int k = 0; k < np; ++k) c.pages[(int64_t)s * c.maxp + k] = c.free_pages[--ctl->free_page_top];
    ctl->clock += 1;
    c.last_hit[s] = (unsigned long long)ctl->clock;
    c.pins[s] = 0;
    c.nrows[s] = nr;
    c.vocab[s] = vv;
    c.nbytes[s] = bytes;
    c.digest[s] = d;
    {
      long long pos = ctl->ring_head & c.rmask;
      c.ring_clock[pos] = (unsigned long long)ctl->clock;
      c.ring_slot[pos] = s;
      ctl->ring_head++;
    }
    ctl->total_bytes += bytes;
    ctl->inserts += 1;
    out_slot[i] = s;
    out_gen[i] = c.gen[s];
    while (ctl->total_bytes > ctl->budget && ctl->alive > 1) {
      int v = next_victim(c);
      if (v < 0) break;
      evict_entry(c, v);
    }
  }
}

// ---- warp policy ------------------------------------------------------------------------
//
// The same sequential semantics as insert_policy_scalar_kernel, run by one warp whose 32
// lanes hold identical copies of the control block in registers.  Each step's loads are
// spread over lanes (one round trip instead of a dependent chain), hash probes read a
// 32-bucket window at once, and the lines the next inserts and the next LRU victims will
// touch are prefetched into L1 ahead of use:
//   * input chunk c+2 is loaded, the home windows of chunk c+1 are prefetched;
//   * the event ring is consumed through 32-position windows; the next window's events
//     are loaded one window ahead and their slots' metadata and hash windows prefetched;
//     events found dead stay dead (liveness is monotone: ticks are unique);
//   * the free stacks keep their recently pushed top in a lane-distributed register window,
//     so the pop that follows an eviction's push needs no memory round trip.
// Only this warp touches the cache during the kernel, so L1-resident lines stay coherent.

__constant__ int g_pf_mode = 1;  // 0 none, 1 L1, 2 L2 (LCB_POLICY_PF; A/B of the prefetch level)
__device__ __forceinline__ void pf1(const void* p) {
  const int m = g_pf_mode;
  if (m == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  else if (m == 2) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

__device__ __forceinline__ void pf_window(const CacheDev& c, uint64_t d) {
  const uint32_t b = home_bucket(d, c.hmask);
  pf1(c.hvals + b);
  pf1(c.hvals + ((b + 31) & c.hmask));
  pf1(c.hkeys + b);
  pf1(c.hkeys + ((b + 15) & c.hmask));
  pf1(c.hkeys + ((b + 31) & c.hmask));
}

// Register mirror of stack entries [base, base + 32): lane l holds entry base + l when bit l is set.
struct RegStack {
  long long base;
  unsigned valid;
  int val;
};

// Push v_k (held by lane k, k < m) at indices idx0 + k; lanes k < m store to memory.
__device__ __forceinline__ void rs_push_many(RegStack& r, int32_t* arr, long long idx0, int m, int vk, int lane) {
  if (lane < m) arr[idx0 + lane] = vk;
  if (idx0 < r.base || idx0 + m > r.base + 32) {
    r.base = idx0;
    r.valid = 0;
  }
  const int off = (int)(idx0 - r.base);
  const int src = lane - off;
  const int v = __shfl_sync(0xffffffffu, vk, src & 31);
  if (src >= 0 && src < m) r.val = v;
  r.valid |= (m >= 32 ? 0xffffffffu : ((1u << m) - 1u)) << off;
}

// Lane k (k < m) returns entry idx_hi - k (a pop of m entries, top first).
__device__ __forceinline__ int rs_get_many(const RegStack& r, const int32_t* arr, long long idx_hi, int m, int lane) {
  const long long idx = idx_hi - lane;
  const long long off = idx - r.base;
  const bool hit = off >= 0 && off < 32 && ((r.valid >> (int)(off & 31)) & 1u);
  const int v = __shfl_sync(0xffffffffu, r.val, (int)(off & 31));
  if (lane >= m) return -1;
  return hit ? v : arr[idx];
}

// Single-entry push / pop (the common case: one slot, single-page entries).
__device__ __forceinline__ void rs_push1(RegStack& r, int32_t* arr, long long idx, int v, int lane) {
  if (lane == 0) arr[idx] = v;
  if (idx < r.base || idx >= r.base + 32) {
    r.base = idx;
    r.valid = 0;
  }
  const int off = (int)(idx - r.base);
  if (lane == off) r.val = v;
  r.valid |= 1u << off;
}
__device__ __forceinline__ int rs_get1(const RegStack& r, const int32_t* arr, long long idx) {
  const long long off = idx - r.base;
  const bool hit = off >= 0 && off < 32 && ((r.valid >> (int)(off & 31)) & 1u);
  const int v = __shfl_sync(0xffffffffu, r.val, (int)(off & 31));
  return hit ? v : arr[idx];
}

// 32-bucket window probe at d's home bucket.  found: slot or -1; *empty_pos: first empty
// bucket index (absolute) or -1 when the window holds none; *chain_open: the probe chain
// runs past the window without a verdict.
__device__ __forceinline__ int window_find(const CacheDev& c, uint64_t d, int lane, uint32_t* empty_b, bool* open) {
  const uint32_t b0 = home_bucket(d, c.hmask);
  const uint32_t bl = (b0 + lane) & c.hmask;
  const int hv = c.hvals[bl];
  const uint64_t hk = c.hkeys[bl];
  const unsigned em = __ballot_sync(0xffffffffu, hv < 0);
  const unsigned mm = __ballot_sync(0xffffffffu, hv >= 0 && hk == d);
  const int fe = em ? __ffs(em) - 1 : 32;
  const unsigned before = fe >= 32 ? 0xffffffffu : ((1u << fe) - 1u);
  const unsigned hit = mm & before;
  *empty_b = fe < 32 ? ((b0 + fe) & c.hmask) : 0xffffffffu;
  *open = !hit && fe >= 32;
  if (!hit) return -1;
  return __shfl_sync(0xffffffffu, hv, __ffs(hit) - 1);
}

// Backward-shift deletion of d when its chain closes inside the 32-bucket window;
// otherwise lane 0 runs the scalar table_delete.
__device__ __forceinline__ void window_delete(const CacheDev& c, uint64_t d, int lane, uint32_t sh_b,
                                              unsigned& st_home, uint32_t w_hb, unsigned& w_bstale) {
  auto mark = [&](uint32_t b) {
    st_home |= __ballot_sync(0xffffffffu, sh_b == b);
    w_bstale |= __ballot_sync(0xffffffffu, w_hb == b || ((w_hb + 1) & c.hmask) == b);
  };
  const uint32_t b0 = home_bucket(d, c.hmask);
  const uint32_t bl = (b0 + lane) & c.hmask;
  const int hv = c.hvals[bl];
  const uint64_t hk = c.hkeys[bl];
  const unsigned em = __ballot_sync(0xffffffffu, hv < 0);
  const unsigned mm = __ballot_sync(0xffffffffu, hv >= 0 && hk == d);
  const int fe = em ? __ffs(em) - 1 : 32;
  const unsigned hit = mm & (fe >= 32 ? 0xffffffffu : ((1u << fe) - 1u));
  if (!hit) {
    if (fe >= 32) {  // chain leaves the window
      if (lane == 0) table_delete(c, d);
      __syncwarp();
      st_home = 0xffffffffu;
      w_bstale = 0xffffffffu;
    }
    return;  // absent
  }
  int i = __ffs(hit) - 1;
  if (i + 1 >= 32 || (em >> (i + 1)) == 0u) {  // shift may run past the window
    if (lane == 0) table_delete(c, d);
    __syncwarp();
    st_home = 0xffffffffu;
    w_bstale = 0xffffffffu;
    return;
  }
  const uint32_t home_l = home_bucket(hk, c.hmask);
  for (int j = i + 1;; ++j) {
    const int vj = __shfl_sync(0xffffffffu, hv, j);
    if (vj < 0) break;
    const uint32_t k = __shfl_sync(0xffffffffu, home_l, j);
    const uint32_t ai = (b0 + i) & c.hmask, aj = (b0 + j) & c.hmask;
    const bool stays = (ai <= aj) ? (ai < k && k <= aj) : (ai < k || k <= aj);
    if (stays) continue;
    const uint64_t kj = __shfl_sync(0xffffffffu, hk, j);
    if (lane == 0) {
      c.hkeys[ai] = kj;
      c.hvals[ai] = vj;
    }
    mark(ai);
    i = j;
  }
  if (lane == 0) c.hvals[(b0 + i) & c.hmask] = -1;
  mark((b0 + i) & c.hmask);
  __syncwarp();
}

struct RingWin {
  long long base;      // first position of the current window, -1 = none
  unsigned loaded;     // positions that existed (< head) when loaded
  unsigned dead;       // events known dead
  int slot;            // lane l: event base + l
  unsigned long long clock;
  unsigned stale;      // records whose slot was written since the window was entered
  unsigned bstale;     // records whose home bucket (or the one after it) was written since
  uint32_t hb;         // lane l's digest home bucket
  bool quick;          // its key sits at hb with hb + 1 empty: deletion = clearing hb
  int pins, pg;        // lane l's entry when live: pins, first page (maxp == 1), bytes, digest, gen
  long long nb;
  uint64_t dg;
  uint32_t gen;
  long long nbase;     // next window, loaded ahead
  unsigned nloaded;
  int nslot;
  unsigned long long nclock;
};

__device__ __forceinline__ void ring_load_next(const CacheDev& c, RingWin& w, long long nb, long long head, int lane) {
  w.nbase = nb;
  const long long p = nb + lane;
  const bool ok = p < head;
  w.nloaded = __ballot_sync(0xffffffffu, ok);
  w.nslot = ok ? c.ring_slot[p & c.rmask] : -1;
  w.nclock = ok ? c.ring_clock[p & c.rmask] : 0ull;
}

__device__ __forceinline__ void ring_prefetch_next(const CacheDev& c, const RingWin& w) {
  const int s = w.nslot;
  if (s >= 0) {
    pf1(c.alive + s);
    pf1(c.last_hit + s);
    pf1(c.pins + s);
    pf1(c.nbytes + s);
    pf1(c.digest + s);
    pf1(c.gen + s);
    pf1(c.pages + (int64_t)s * c.maxp);
  }
}

// Enter the window starting at position t: take the preloaded one when it matches.
__device__ __forceinline__ void ring_enter(const CacheDev& c, RingWin& w, long long t, long long head, int lane) {
  if (w.nbase != t) ring_load_next(c, w, t, head, lane);
  w.base = w.nbase;
  w.loaded = w.nloaded;
  w.slot = w.nslot;
  w.clock = w.nclock;
  // liveness prefilter, the live events' entry records (valid until their slot is written:
  // w.stale) and the hash windows of their digests
  const int s = w.slot;
  bool live = false;
  w.pins = 0;
  w.pg = -2;
  w.nb = 0;
  w.dg = 0;
  w.gen = 0;
  if (s >= 0) {
    live = c.alive[s] && c.last_hit[s] == w.clock;
    if (live) {
      w.dg = c.digest[s];
      w.pins = c.pins[s];
      w.nb = c.nbytes[s];
      w.gen = c.gen[s];
      if (c.maxp == 1) w.pg = c.pages[s];
    }
  }
  w.hb = home_bucket(w.dg, c.hmask);
  w.quick = false;
  if (live) w.quick = c.hvals[w.hb] == s && c.hkeys[w.hb] == w.dg && c.hvals[(w.hb + 1) & c.hmask] < 0;
  w.dead = __ballot_sync(0xffffffffu, !live) & w.loaded;
  w.stale = 0u;
  w.bstale = 0u;
  // next window: events now, metadata lines prefetched; the window after: ring lines
  pf1(c.ring_slot + ((t + 64 + lane) & c.rmask));
  pf1(c.ring_clock + ((t + 64 + lane) & c.rmask));
  ring_load_next(c, w, t + 32, head, lane);
  ring_prefetch_next(c, w);
}

struct Victim {
  int s;
  long long nbytes;
  uint64_t digest;
  uint32_t gen;
  int pg;       // first page when known (maxp == 1), else -2
  bool scalar;  // chosen by the scalar fallback (control block reloaded)
  bool quick;   // deletion = clearing bucket hb (record still valid)
  uint32_t hb;
};

__device__ __forceinline__ void ctl_flush(const CacheDev& c, const Ctl& L, int lane) {
  if (lane == 0) *c.ctl = L;
  __syncwarp();
}

// Oldest live unpinned entry (next_victim), or s = -1.
__device__ __forceinline__ Victim warp_next_victim(const CacheDev& c, Ctl& L, RingWin& w, int lane) {
  Victim v{-1, 0, 0, 0, -2, false, false, 0u};
  for (;;) {
    if (L.side_count > 0) break;  // pinned entries pending: scalar path
    if (L.ring_tail >= L.ring_head) return v;
    if (w.base < 0 || L.ring_tail < w.base || L.ring_tail >= w.base + 32) ring_enter(c, w, L.ring_tail, L.ring_head, lane);
    const int off = (int)(L.ring_tail - w.base);
    if (!((w.loaded >> off) & 1u)) {  // appended after the window was read
      w.base = -1;
      w.nbase = -1;
      continue;
    }
    const unsigned cand = ~w.dead & w.loaded & (0xffffffffu << off);
    if (!cand) {
      const unsigned rest = w.loaded & (0xffffffffu << off);
      L.ring_tail = w.base + (32 - __clz(rest));  // every loaded event from off on is dead
      continue;
    }
    const int o = __ffs(cand) - 1;
    L.ring_tail = w.base + o;
    const int s = __shfl_sync(0xffffffffu, w.slot, o);
    const unsigned long long ck = __shfl_sync(0xffffffffu, w.clock, o);
    if (!((w.stale >> o) & 1u)) {  // the record taken at window entry still holds: live
      const int pins = __shfl_sync(0xffffffffu, w.pins, o);
      if (pins > 0) break;  // scalar path moves it to the side list
      L.ring_tail++;
      v.s = s;
      v.nbytes = __shfl_sync(0xffffffffu, w.nb, o);
      v.digest = __shfl_sync(0xffffffffu, w.dg, o);
      v.gen = __shfl_sync(0xffffffffu, w.gen, o);
      v.pg = __shfl_sync(0xffffffffu, w.pg, o);
      v.quick = __shfl_sync(0xffffffffu, (int)w.quick, o) && !((w.bstale >> o) & 1u);
      v.hb = __shfl_sync(0xffffffffu, w.hb, o);
      return v;
    }
    const bool alive = c.alive[s];
    const unsigned long long lh = c.last_hit[s];
    const int pins = c.pins[s];
    const long long nb = c.nbytes[s];
    const uint64_t dg = c.digest[s];
    const uint32_t g = c.gen[s];
    if (!(alive && lh == ck)) {
      w.dead |= 1u << o;
      L.ring_tail++;
      continue;
    }
    if (pins > 0) break;  // scalar path moves it to the side list
    L.ring_tail++;
    v.s = s;
    v.nbytes = nb;
    v.digest = dg;
    v.gen = g;
    return v;
  }
  // scalar fallback: the reference-shaped next_victim over the control block in memory
  ctl_flush(c, L, lane);
  int s = -1;
  if (lane == 0) s = next_victim(c);
  __syncwarp();
  s = __shfl_sync(0xffffffffu, s, 0);
  L = *c.ctl;
  w.base = -1;
  w.nbase = -1;
  v.s = s;
  v.scalar = true;
  if (s >= 0) {
    v.nbytes = c.nbytes[s];
    v.digest = c.digest[s];
    v.gen = c.gen[s];
  }
  return v;
}

// push_pages for the warp policy: the entry's pages go on the free stack in page order
__device__ __forceinline__ void warp_push_pages(const CacheDev& c, Ctl& L, RegStack& fp, int s, int lane,
                                                int known_pg = -2) {
  if (c.maxp == 1) {
    const int pg = known_pg != -2 ? known_pg : c.pages[s];
    if (pg >= 0) {
      if (lane == 0) c.pages[s] = -1;
      rs_push1(fp, c.free_pages, L.free_page_top, pg, lane);
      L.free_page_top += 1;
    }
    return;
  }
  for (int k0 = 0; k0 < c.maxp; k0 += 32) {
    const int k = k0 + lane;
    const int pg = k < c.maxp ? c.pages[(int64_t)s * c.maxp + k] : -1;
    const unsigned have = __ballot_sync(0xffffffffu, pg >= 0);
    const int m = __ffs(~have) - 1 < 0 ? 32 : __ffs(~have) - 1;
    if (lane < m) c.pages[(int64_t)s * c.maxp + k] = -1;
    rs_push_many(fp, c.free_pages, L.free_page_top, m, pg, lane);
    L.free_page_top += m;
    if (m < 32) break;
  }
}

// Overwrite push (see push_pages_rev): pages np-1 .. 0 of entry s, so the pops that follow
// return page 0 first.
__device__ __forceinline__ void warp_push_pages_rev(const CacheDev& c, Ctl& L, RegStack& fp, int s, int lane,
                                                    int known_pg = -2) {
  if (c.maxp == 1) {
    warp_push_pages(c, L, fp, s, lane, known_pg);
    return;
  }
  const int nr = c.nrows[s];
  const int np = min(c.maxp, (nr + c.page_rows - 1) / c.page_rows);
  for (int k0 = 0; k0 < np; k0 += 32) {
    const int m = min(32, np - k0);
    const int k = np - 1 - (k0 + lane);
    const int pg = lane < m ? c.pages[(int64_t)s * c.maxp + k] : -1;
    if (lane < m) c.pages[(int64_t)s * c.maxp + k] = -1;
    rs_push_many(fp, c.free_pages, L.free_page_top, m, pg, lane);
    L.free_page_top += m;
  }
}

// resume (optional, written by commit_kernel): [0] = first insert still to apply, [1] = 1 when
// the insert before it still owes its evictions; the warp applies inserts [resume[0], n).
__global__ void __launch_bounds__(32) insert_policy_kernel(CacheDev c, const uint64_t* __restrict__ dig,
                                                           const int32_t* __restrict__ lens,
                                                           const int32_t* __restrict__ vocabs, int64_t n,
                                                           int32_t* out_slot, uint32_t* out_gen,
                                                           const int32_t* __restrict__ keep,
                                                           const uint32_t* __restrict__ keep_gen,
                                                           const int* __restrict__ resume) {
  const int lane = threadIdx.x;
  bool pend = false;
  if (resume) {
    const int64_t start = resume[0];
    pend = resume[1] != 0;
    if (start >= n && !pend) return;
    dig += start;
    lens += start;
    vocabs += start;
    out_slot += start;
    out_gen += start;
    if (keep) {
      keep += start;
      keep_gen += start;
    }
    n -= start;
  }
  Ctl L = *c.ctl;
  RegStack fs{-1ll << 40, 0u, 0}, fp{-1ll << 40, 0u, 0};
  RingWin w;
  w.base = -1;
  w.nbase = -1;
  w.slot = -1;
  w.stale = 0u;
  w.bstale = 0u;
  w.hb = 0u;
  w.quick = false;
  int last_ev_slot = -1;
  uint32_t last_ev_gen = 0;
  // chunk pipeline: cur (c), nx1 (c+1), nx2 (c+2)
  auto ld = [&](int64_t i, uint64_t& d, int& nr, int& vv) {
    if (i < n) {
      d = dig[i];
      nr = lens[i];
      vv = vocabs[i];
    } else {
      d = 0;
      nr = -1;
      vv = 0;
    }
  };
  // the LRU eviction loop after an insert (logits_cache.py:134-140); sh_b / sp_s / st_home /
  // st_slot are the current chunk's speculative records, marked by every write
  auto evict_loop = [&](uint32_t sh_b, int sp_s, unsigned& st_home, unsigned& st_slot) {
    auto mark_slot = [&](int x) {
      st_slot |= __ballot_sync(0xffffffffu, sp_s == x);
      w.stale |= __ballot_sync(0xffffffffu, w.slot == x);
    };
    while (L.total_bytes > L.budget && L.alive > 1) {
      Victim v = warp_next_victim(c, L, w, lane);
      if (v.s < 0) break;
      // evict_entry
      mark_slot(v.s);
      if (v.quick) {  // key at its home bucket, next bucket empty: no shift
        if (lane == 0) c.hvals[v.hb] = -1;
        st_home |= __ballot_sync(0xffffffffu, sh_b == v.hb);
        w.bstale |= __ballot_sync(0xffffffffu, w.hb == v.hb || ((w.hb + 1) & c.hmask) == v.hb);
      } else {
        window_delete(c, v.digest, lane, sh_b, st_home, w.hb, w.bstale);
      }
      L.total_bytes -= v.nbytes;
      warp_push_pages(c, L, fp, v.s, lane, v.pg);
      rs_push1(fs, c.free_slots, L.free_slot_top, v.s, lane);
      L.free_slot_top += 1;
      if (lane == 0) {
        c.gen[v.s] = v.gen + 1u;
        c.alive[v.s] = 0;
      }
      last_ev_slot = v.s;
      last_ev_gen = v.gen + 1u;
      L.alive -= 1;
      L.evictions += 1;
      __syncwarp();
    }
  };
  if (pend) {  // the fast commit stopped inside an insert's eviction loop
    unsigned h0 = 0u, s0 = 0u;
    evict_loop(0xffffffffu, -1, h0, s0);
  }
  uint64_t d0, d1, d2;
  int n0, n1, n2, v0, v1, v2;
  ld(lane, d0, n0, v0);
  ld(32 + lane, d1, n1, v1);
  if (lane < n) pf_window(c, d0);
  for (int64_t i0 = 0; i0 < n; i0 += 32) {
    ld(i0 + 64 + lane, d2, n2, v2);
    if (i0 + 32 + lane < n) pf_window(c, d1);
    // speculative records of this chunk's keys (lane l = element l): the home bucket and,
    // when it holds the key, the entry's bytes / generation / first page.  A record is used
    // only while nothing it depends on was written since (st_home: its home bucket;
    // st_slot: its entry); every table or entry write below marks the records it touches.
    const uint32_t sh_b = home_bucket(d0, c.hmask);
    int sh_v = -1, sp_s = -1, sp_pg = -2;
    uint64_t sh_k = 0;
    long long sp_nb = 0;
    uint32_t sp_gen = 0;
    if (i0 + lane < n) {
      sh_v = c.hvals[sh_b];
      sh_k = c.hkeys[sh_b];
      if (sh_v >= 0 && sh_k == d0) {
        sp_s = sh_v;
        sp_nb = c.nbytes[sp_s];
        sp_gen = c.gen[sp_s];
        if (c.maxp == 1) sp_pg = c.pages[sp_s];
      }
    }
    unsigned st_home = 0u, st_slot = 0u;
    auto mark_slot = [&](int x) {
      st_slot |= __ballot_sync(0xffffffffu, sp_s == x);
      w.stale |= __ballot_sync(0xffffffffu, w.slot == x);
    };
    int my_slot = -1;
    uint32_t my_gen = 0;
    const int cnt = (int)min((int64_t)32, n - i0);
    for (int j = 0; j < cnt; ++j) {
      const uint64_t d = __shfl_sync(0xffffffffu, d0, j);
      const int nr = __shfl_sync(0xffffffffu, n0, j);
      const int vv = __shfl_sync(0xffffffffu, v0, j);
      const int np = c.page_rows == 1 ? nr : (nr + c.page_rows - 1) / c.page_rows;
      if (nr < 0 || vv < 1 || vv > c.V || np > c.maxp) {
        if (!L.error) L.error = LC_E_CONFIG;
        continue;
      }
      const long long bytes = (long long)nr * vv * 4 + 8ll * nr;  // logits_cache.py:54-56
      uint32_t eb;
      bool open = false;
      int s;
      const bool rec = !((st_home >> j) & 1u);
      const int hv0 = __shfl_sync(0xffffffffu, sh_v, j);
      const uint64_t hk0 = __shfl_sync(0xffffffffu, sh_k, j);
      bool from_rec = false;
      if (rec && hv0 >= 0 && hk0 == d) {  // found at its home bucket
        s = hv0;
        from_rec = !((st_slot >> j) & 1u);
      } else if (rec && hv0 < 0) {  // empty home bucket: absent, and the insert goes there
        s = -1;
        eb = __shfl_sync(0xffffffffu, sh_b, j);
      } else {
        s = window_find(c, d, lane, &eb, &open);
        if (open) {
          if (lane == 0) s = table_find(c, d);
          s = __shfl_sync(0xffffffffu, s, 0);
        }
      }
      uint32_t g;
      if (s >= 0) {  // overwrite: the key keeps its slot, the entry is new
        long long onb;
        int opg = -2;
        if (from_rec) {
          onb = __shfl_sync(0xffffffffu, sp_nb, j);
          g = __shfl_sync(0xffffffffu, sp_gen, j) + 1u;
          opg = __shfl_sync(0xffffffffu, sp_pg, j);
        } else {
          onb = c.nbytes[s];
          g = c.gen[s] + 1u;
        }
        mark_slot(s);
        if (keep) {
          const int i = (int)(i0 + j);
          if (keep[i] > 0 && !keep_ok(c, true, s, g - 1u, keep[i], keep_gen[i], nr, vv) && !L.error)
            L.error = LC_E_STATE;
        }
        L.total_bytes -= onb;
        warp_push_pages_rev(c, L, fp, s, lane, opg);
        if (lane == 0) c.gen[s] = g;
      } else {
        if (keep && keep[i0 + j] > 0 && !L.error) L.error = LC_E_STATE;  // write-back of a gone entry
        if (L.free_slot_top == 0) {
          if (!L.error) L.error = LC_E_CAPACITY;
          continue;
        }
        s = rs_get1(fs, c.free_slots, L.free_slot_top - 1);
        L.free_slot_top--;
        mark_slot(s);
        if (eb == 0xffffffffu || open) {  // no empty bucket in the window
          if (lane == 0) table_insert(c, d, s);
          st_home = 0xffffffffu;
          w.bstale = 0xffffffffu;
        } else {
          if (lane == 0) {
            c.hkeys[eb] = d;
            c.hvals[eb] = s;
          }
          st_home |= __ballot_sync(0xffffffffu, sh_b == eb);
          w.bstale |= __ballot_sync(0xffffffffu, w.hb == eb || ((w.hb + 1) & c.hmask) == eb);
        }
        if (lane == 0) c.alive[s] = 1;
        L.alive += 1;
        g = (s == last_ev_slot) ? last_ev_gen : c.gen[s];
      }
      if (L.free_page_top < np) {
        // out of slab pages: roll back as insert_policy_scalar_kernel does (key out of the
        // index, slot back on the free stack, error latched)
        if (!L.error) L.error = LC_E_CAPACITY;
        mark_slot(s);
        window_delete(c, d, lane, sh_b, st_home, w.hb, w.bstale);
        rs_push1(fs, c.free_slots, L.free_slot_top, s, lane);
        L.free_slot_top += 1;
        if (lane == 0) {
          c.alive[s] = 0;
          c.nrows[s] = 0;
          c.nbytes[s] = 0;
        }
        last_ev_slot = s;
        last_ev_gen = g;
        L.alive -= 1;
        __syncwarp();
        continue;
      }
      if (np == 1) {  // (single-page entries: one broadcast value, no lane scatter)
        const int pg = rs_get1(fp, c.free_pages, L.free_page_top - 1);
        if (lane == 0) c.pages[(int64_t)s * c.maxp] = pg;
        L.free_page_top -= 1;
      } else {
        for (int k0 = 0; k0 < np; k0 += 32) {
          const int m = min(32, np - k0);
          const int pg = rs_get_many(fp, c.free_pages, L.free_page_top - 1, m, lane);
          if (lane < m) c.pages[(int64_t)s * c.maxp + k0 + lane] = pg;
          L.free_page_top -= m;
        }
      }
      L.clock += 1;
      if (lane == 0) {
        c.last_hit[s] = (unsigned long long)L.clock;
        c.pins[s] = 0;
        c.nrows[s] = nr;
        c.vocab[s] = vv;
        c.nbytes[s] = bytes;
        c.digest[s] = d;
        const long long pos = L.ring_head & c.rmask;
        c.ring_clock[pos] = (unsigned long long)L.clock;
        c.ring_slot[pos] = s;
      }
      L.ring_head++;
      L.total_bytes += bytes;
      L.inserts += 1;
      if (lane == j) {
        my_slot = s;
        my_gen = g;
      }
      __syncwarp();
      evict_loop(sh_b, sp_s, st_home, st_slot);
    }
    if (lane < cnt) {
      out_slot[i0 + lane] = my_slot;
      out_gen[i0 + lane] = my_gen;
    }
    d0 = d1; n0 = n1; v0 = v1;
    d1 = d2; n1 = n2; v1 = v2;
  }
  __syncwarp();
  if (lane == 0) *c.ctl = L;
}

// ---- batched fast commit (single-page entries: BASELINE config 4) ---------------------------
//
// The warp policy spends ~400 dependent warp instructions per insert on probes, LRU window
// bookkeeping and hash-table edits (profiles/r1_ncu_policy_v3.txt).  For caches of
// single-page entries (maxp == 1) a batch is split three ways instead:
//   * prep_keys_kernel / prep_prev_kernel (parallel): each insert's start-of-batch view -- the
//     slot holding its key and that entry's generation / bytes / page -- and the previous
//     insert of the same key in the batch;
//   * prep_cand_kernel (parallel): the LRU end of the event ring at batch start, compacted per
//     256-position tile to the live events with their entries' records;
//   * commit_kernel: ONE thread applies the batch in index order from those records (streamed
//     into shared memory by bulk copies), with the free-stack tops mirrored in shared memory
//     and a bitmap of the start-of-batch entries gone (overwritten or evicted) during the
//     batch -- the only thing that can invalidate a record, since entries created in the
//     batch are younger than every start-of-batch candidate and so never its victims.
//     Hash-table edits decide nothing (slots and pages come from the stacks), so the commit
//     thread only logs them and a second warp applies the log in order, overlapped.
// Anything outside that model (a side list of pinned entries at batch start, a config or
// capacity error, the scanned candidates used up) stops the commit at that insert with the
// control block flushed, and insert_policy_kernel resumes from there.  Slots, generations,
// victims and accounting are those of insert_policy_scalar_kernel (logits_cache.py:96-140).

struct alignas(16) InsRec {  // 48 B
  uint64_t d;
  long long nb0;   // bytes of the entry holding d at batch start
  long long nb;    // the insert's bytes (logits_cache.py:54-56)
  int32_t s0;      // its slot, -1 absent
  uint32_t gen0;   // its generation
  int32_t pg0;     // its page, -1 none
  int32_t nr;      // the insert's rows (-1: invalid -- the warp policy latches the error)
  int32_t vv;      // its vocab
  int32_t prev;    // largest j < i with d_j == d_i, -1 none
  int32_t pad;
};
struct alignas(16) CandRec {  // 48 B: one live event at batch start
  uint64_t dg;
  long long nb;
  unsigned long long ck;
  int32_t s;
  uint32_t gen;
  int32_t pg;
  int32_t off;  // ring position - tail0
  int32_t pins;
  int32_t pad;
};
struct HashOp {  // s >= 0: insert d -> s; s < 0: delete d
  uint64_t d;
  int32_t s;
  int32_t pad;
};
static_assert(sizeof(InsRec) % 16 == 0 && sizeof(CandRec) % 16 == 0, "bulk-copied records");
constexpr int kFcTile = 256;    // records per bulk-copied tile
constexpr int kFcMirror = 2048;  // free-stack entries mirrored in shared memory

__global__ void prep_keys_kernel(CacheDev c, const uint64_t* __restrict__ dig, const int32_t* __restrict__ lens,
                                 const int32_t* __restrict__ vocabs, int64_t n, InsRec* __restrict__ rec) {
  const int64_t key = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  const int lane = threadIdx.x & 31;
  const unsigned tile_bits = 0xffu << (lane & 24);
  const bool active = key < n;
  const uint64_t d = active ? dig[key] : 0ull;
  const uint32_t start = home_bucket(d, c.hmask);
  int result = -1;
  bool done = !active;
  for (uint32_t round = 0; __any_sync(0xffffffffu, !done); ++round) {
    bool match = false, empty = false;
    if (!done) {
      const uint32_t b = (start + round * 8u + sub) & c.hmask;
      const int32_t v = c.hvals[b];
      match = v >= 0 && c.hkeys[b] == d;
      empty = v < 0;
      if (match) result = v;
      if (round * 8u > c.hmask) empty = true;
    }
    const unsigned mm = __ballot_sync(0xffffffffu, match) & tile_bits;
    const unsigned em = __ballot_sync(0xffffffffu, empty) & tile_bits;
    if (!done) {
      if (mm) {
        result = __shfl_sync(tile_bits, result, __ffs(mm) - 1, 32);
        done = true;
      } else if (em) {
        result = -1;
        done = true;
      }
    }
  }
  if (active && sub == 0) {
    InsRec r;
    r.d = d;
    r.s0 = result;
    r.nr = lens[key];
    r.vv = vocabs[key];
    if (r.nr < 0 || r.vv < 1 || r.vv > c.V || r.nr > c.page_rows * c.maxp) r.nr = -1;
    r.nb = r.nr >= 0 ? (long long)r.nr * r.vv * 4 + 8ll * r.nr : 0;  // logits_cache.py:54-56
    r.prev = -1;
    r.gen0 = result >= 0 ? c.gen[result] : 0u;
    r.nb0 = result >= 0 ? c.nbytes[result] : 0;
    r.pg0 = result >= 0 ? c.pages[(int64_t)result * c.maxp] : -1;
    rec[key] = r;
  }
}

// prev[i] = the largest j < i with d_j == d_i: block b scans the key tiles b, b-1, ... 0 from
// shared memory until every key of the block found one (duplicates are rare: usually all tiles)
__global__ void __launch_bounds__(256) prep_prev_kernel(const uint64_t* __restrict__ dig, int64_t n,
                                                        InsRec* __restrict__ rec) {
  __shared__ uint64_t t[256];
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const uint64_t d = i < n ? dig[i] : 0ull;
  int prev = -1;
  for (int tb = blockIdx.x; tb >= 0; --tb) {
    const int64_t j0 = (int64_t)tb * 256;
    __syncthreads();
    t[threadIdx.x] = j0 + threadIdx.x < n ? dig[j0 + threadIdx.x] : 0ull;
    __syncthreads();
    if (prev < 0 && i < n) {
      const int jm = (int)min((int64_t)256, i - j0);
      for (int k0 = jm - 1; k0 >= 0 && prev < 0; k0 -= 16) {
        int f = -1;
#pragma unroll
        for (int u = 15; u >= 0; --u) {  // the highest matching k of the 16 wins
          const int k = k0 - u;
          if (k >= 0 && t[k] == d) f = k;
        }
        if (f >= 0) prev = (int)(j0 + f);
      }
    }
    if (__syncthreads_and(prev >= 0 || i >= n)) break;
  }
  if (i < n && prev >= 0) rec[i].prev = prev;
}

// Tile b: ring positions tail0 + 256 b + [0, 256) below min(head0, tail0 + mcap); the live
// events (alive, last_hit == event clock) in position order with their entries' records.
__global__ void __launch_bounds__(256) prep_cand_kernel(CacheDev c, long long mcap, CandRec* __restrict__ cand,
                                                        int* __restrict__ cnt) {
  __shared__ int wcnt[8];
  const long long tail0 = c.ctl->ring_tail, head0 = c.ctl->ring_head;
  const long long lim = min(head0, tail0 + mcap);
  const long long p = tail0 + (long long)blockIdx.x * 256 + threadIdx.x;
  bool live = false;
  int s = -1;
  unsigned long long ck = 0;
  if (p < lim) {
    s = c.ring_slot[p & c.rmask];
    ck = c.ring_clock[p & c.rmask];
    live = c.alive[s] && c.last_hit[s] == ck;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, live);
  if (lane == 0) wcnt[wid] = __popc(b);
  __syncthreads();
  int off = __popc(b & ((1u << lane) - 1u)), tot = 0;
  for (int k = 0; k < 8; ++k) {
    if (k < wid) off += wcnt[k];
    tot += wcnt[k];
  }
  if (live) {
    CandRec r;
    r.dg = c.digest[s];
    r.nb = c.nbytes[s];
    r.ck = ck;
    r.s = s;
    r.gen = c.gen[s];
    r.pg = c.pages[(int64_t)s * c.maxp];
    r.off = (int)(p - tail0);
    r.pins = c.pins[s];
    r.pad = 0;
    cand[(int64_t)blockIdx.x * 256 + off] = r;
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Entry-metadata writes of one committed insert (i >= 0) or eviction (i < 0), queued by the
// commit thread for the writer warp.
struct alignas(16) WRec {  // 32 B
  uint64_t d;
  int32_t s;
  uint32_t g;   // the entry's generation (insert) / the slot's next generation (eviction)
  int32_t pg;   // insert: its page (-1 none); eviction: 1 when pages[s] must be cleared
  int32_t i;    // insert index, -1 eviction
  int32_t nr, vv;
};
constexpr int kFcWRing = 1024;  // writer records in flight
constexpr int kFcWin = 33;      // staged window row stride (conflict-free transposed access)

// grid (1), block 128.  Warp 0 lane 0 commits; warp 1 applies the hash-edit log; warp 2 writes
// the entries' metadata, ring events and outputs from the commit records; all four warps fill
// the shared-memory mirrors first.  Dynamic shared memory: fc_smem_bytes.
__global__ void __launch_bounds__(128) commit_kernel(CacheDev c, const InsRec* __restrict__ rec, int64_t n,
                                                     const CandRec* __restrict__ cand, const int* __restrict__ cnt,
                                                     int ntiles, long long mcap, HashOp* __restrict__ hlog,
                                                     int32_t* __restrict__ out_slot, uint32_t* __restrict__ out_gen,
                                                     int* __restrict__ resume) {
  extern __shared__ __align__(16) unsigned char fc_smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(fc_smem);  // rec 0/1, cand 0/1
  // [0] log count, [1] finished, [2] writer records queued, [3] writer records done
  volatile int* s_flag = reinterpret_cast<volatile int*>(fc_smem + 32);
  InsRec* rbuf = reinterpret_cast<InsRec*>(fc_smem + 64);
  CandRec* cbuf = reinterpret_cast<CandRec*>(rbuf + 2 * kFcTile);
  WRec* wring = reinterpret_cast<WRec*>(cbuf + 2 * kFcTile);
  unsigned long long* wk = reinterpret_cast<unsigned long long*>(wring + kFcWRing);  // staged windows
  int* wv = reinterpret_cast<int*>(wk + 32 * kFcWin);
  int* ms_val = wv + 32 * kFcWin;
  uint32_t* ms_gen = reinterpret_cast<uint32_t*>(ms_val + kFcMirror);
  int* mp_val = reinterpret_cast<int*>(ms_gen + kFcMirror);
  int* cnt_s = mp_val + kFcMirror;
  uint32_t* gone = reinterpret_cast<uint32_t*>(cnt_s + ntiles);
  const int tid = threadIdx.x, lane = tid & 31;
  Ctl L = *c.ctl;
  const int bs = max(0, L.free_slot_top - kFcMirror / 2);
  const int bp = max(0, L.free_page_top - kFcMirror / 2);
  for (int k = tid; k < (c.E + 31) / 32; k += blockDim.x) gone[k] = 0u;
  for (int k = tid; k < kFcMirror; k += blockDim.x) {
    if (bs + k < L.free_slot_top) {
      const int v = c.free_slots[bs + k];
      ms_val[k] = v;
      ms_gen[k] = c.gen[v];
    }
    if (bp + k < L.free_page_top) mp_val[k] = c.free_pages[bp + k];
  }
  for (int k = tid; k < ntiles; k += blockDim.x) cnt_s[k] = cnt[k];
  if (tid == 0) {
    for (int k = 0; k < 4; ++k) mbar_init(&bars[k], 1);
    mbar_fence_init();
    for (int k = 0; k < 4; ++k) s_flag[k] = 0;
  }
  __syncthreads();

  if (tid >= 32 && tid < 64) {  // ---- log warp: apply the hash edits in log order ----
    int k = 0;
    for (;;) {
      const int fin = s_flag[1];
      __threadfence_block();
      const int avail = s_flag[0];
      if (k >= avail) {
        if (fin) break;
        __nanosleep(64);
        continue;
      }
      __threadfence_block();
      const int m = min(32, avail - k);
      HashOp op{0ull, -1, 0};
      if (lane < m) op = hlog[k + lane];
      const uint32_t hb = home_bucket(op.d, c.hmask);
      // stage the m windows, all loads in flight together (from L2, where this warp's edits
      // land); bucket hb_j + t of edit j at [t][j]
      for (int j0 = 0; j0 < m; j0 += 16) {
        int v[16];
        unsigned long long kk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t b = (__shfl_sync(0xffffffffu, hb, (j0 + u) & 31) + lane) & c.hmask;
          if (j0 + u < m) {
            v[u] = __ldcg(c.hvals + b);
            kk[u] = __ldcg(reinterpret_cast<const unsigned long long*>(c.hkeys) + b);
          }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (j0 + u < m) {
            wv[lane * kFcWin + j0 + u] = v[u];
            wk[lane * kFcWin + j0 + u] = kk[u];
          }
      }
      __syncwarp();
      // lane j: edit j's footprint [hb, hb + fe] (its cluster from the home bucket up to the
      // first empty bucket) from its own window column; lng: the chain leaves the window
      int fe = 32, at = -1;
      if (lane < m) {
        for (int t = 0; t < 32; ++t) {
          const int hv = wv[t * kFcWin + lane];
          if (hv < 0) {
            fe = t;
            break;
          }
          if (op.s < 0 && at < 0 && wk[t * kFcWin + lane] == op.d) at = t;
        }
      }
      const bool lng = lane < m && fe >= 32;
      // edits whose footprint meets (or touches) an earlier edit's, and every edit after a long
      // one, are applied one by one after the others; the rest commute and run lane-parallel
      bool seq = false;
      const unsigned long_before = __ballot_sync(0xffffffffu, lng) & ((1u << lane) - 1u);
      if (long_before || lng) seq = true;
      for (int q = 0; q < m - 1; ++q) {
        const uint32_t hq = __shfl_sync(0xffffffffu, hb, q);
        const int fq = __shfl_sync(0xffffffffu, fe, q);
        if (q < lane && (((hb - hq) & c.hmask) <= (uint32_t)fq + 1u || ((hq - hb) & c.hmask) <= (uint32_t)fe + 1u))
          seq = true;
      }
      if (lane < m && !seq) {
        if (op.s >= 0) {
          const uint32_t b = (hb + fe) & c.hmask;
          c.hkeys[b] = op.d;
          c.hvals[b] = op.s;
        } else if (at >= 0) {  // backward shift inside the cluster [at, fe)
          int i = at;
          for (int t = at + 1; t < fe; ++t) {
            const uint64_t kt = wk[t * kFcWin + lane];
            const uint32_t kh = home_bucket(kt, c.hmask);
            const uint32_t ai = (hb + i) & c.hmask, aj = (hb + t) & c.hmask;
            const bool stays = (ai <= aj) ? (ai < kh && kh <= aj) : (ai < kh || kh <= aj);
            if (stays) continue;
            c.hkeys[ai] = kt;
            c.hvals[ai] = wv[t * kFcWin + lane];
            i = t;
          }
          c.hvals[(hb + i) & c.hmask] = -1;
        }
      }
      __syncwarp();
      unsigned todo = __ballot_sync(0xffffffffu, lane < m && seq);
      while (todo) {  // the rest in log order, warp-cooperative over fresh windows
        const int j = __ffs(todo) - 1;
        todo &= todo - 1u;
        const uint64_t d = __shfl_sync(0xffffffffu, op.d, j);
        const int s = __shfl_sync(0xffffffffu, op.s, j);
        if (s >= 0) {
          uint32_t eb;
          bool open = false;
          window_find(c, d, lane, &eb, &open);
          if (lane == 0) {
            if (eb != 0xffffffffu && !open) {
              c.hkeys[eb] = d;
              c.hvals[eb] = s;
            } else {
              table_insert(c, d, s);
            }
          }
          __syncwarp();
        } else {
          unsigned h0 = 0u, b0 = 0u;
          window_delete(c, d, lane, 0xffffffffu, h0, 0xffffffffu, b0);
        }
      }
      k += m;
    }
    if (lane == 0) reinterpret_cast<unsigned long long*>(resume)[3] = globaltimer_ns();
    return;
  }

  if (tid >= 64 && tid < 96) {  // ---- writer warp: entry metadata, ring events, outputs ----
    int k = 0, ins = 0;
    for (;;) {
      const int fin = s_flag[1];
      __threadfence_block();
      const int avail = s_flag[2];
      if (k >= avail) {
        if (fin) break;
        __nanosleep(64);
        continue;
      }
      __threadfence_block();
      while (k < avail) {  // 32 records per round, one per lane
        const int m = min(32, avail - k);
        WRec w{0ull, -1 - lane, 0u, -1, -2, 0, 0};
        if (lane < m) w = wring[(k + lane) & (kFcWRing - 1)];
        const int s = w.s;
        const bool is_ins = w.i >= 0;
        // a slot recurs in a round only as (eviction, then the insert that popped it): the
        // round's last record of a slot writes its fields
        const unsigned peers = __match_any_sync(0xffffffffu, s);
        const bool last = (peers >> lane) == 1u;
        const unsigned insm = __ballot_sync(0xffffffffu, is_ins);
        const int rank = ins + __popc(insm & ((1u << lane) - 1u));
        if (is_ins) {
          const unsigned long long ck = (unsigned long long)(L.clock + rank + 1);
          const long long pos = (L.ring_head + rank) & c.rmask;
          c.ring_clock[pos] = ck;
          c.ring_slot[pos] = s;
          out_slot[w.i] = s;
          out_gen[w.i] = w.g;
          if (last) {
            c.last_hit[s] = ck;
            c.nbytes[s] = (long long)w.nr * w.vv * 4 + 8ll * w.nr;  // logits_cache.py:54-56
            c.digest[s] = w.d;
            c.pins[s] = 0;
            c.nrows[s] = w.nr;
            c.vocab[s] = w.vv;
            c.gen[s] = w.g;
            c.pages[s] = w.pg;
            c.alive[s] = 1;
          }
        } else if (lane < m && last) {
          c.gen[s] = w.g;
          if (w.pg) c.pages[s] = -1;
          c.alive[s] = 0;
        }
        ins += __popc(insm);
        k += m;
        __syncwarp();
      }
      if (lane == 0) s_flag[3] = k;
    }
    return;
  }
  if (tid != 0) return;

  // ---- commit thread ----
  reinterpret_cast<unsigned long long*>(resume)[1] = globaltimer_ns();
  const long long tail0 = L.ring_tail, head0 = L.ring_head;
  const long long lim = min(head0, tail0 + mcap);
  const int nct = (int)((lim - tail0 + kFcTile - 1) / kFcTile);  // candidate tiles to walk
  const int nrt = (int)((n + kFcTile - 1) / kFcTile);
  constexpr uint32_t kRecTile = kFcTile * sizeof(InsRec), kCandTile = kFcTile * sizeof(CandRec);
  for (int t = 0; t < 2; ++t) {
    if (t < nrt) {
      mbar_expect_tx(&bars[t], kRecTile);
      bulk_load(rbuf + t * kFcTile, rec + (int64_t)t * kFcTile, kRecTile, &bars[t]);
    }
    if (t < nct) {
      mbar_expect_tx(&bars[2 + t], kCandTile);
      bulk_load(cbuf + t * kFcTile, cand + (int64_t)t * kFcTile, kCandTile, &bars[2 + t]);
    }
  }
  int rt_issued = min(nrt, 2) - 1, rt_waited = -1, ct_issued = min(nct, 2) - 1;
  int ct = 0, ci = 0, ccnt = 0;
  if (nct > 0) {
    mbar_wait(&bars[2], 0);
    ccnt = cnt_s[0];
  }
  int wq = 0, wdone = 0;  // writer records queued / known done
  long long cy_wput = 0, cy_drain = 0, cy_tile = 0, n_drain = 0;  // LCB_FC_PROF diagnostics
  auto wput = [&](const WRec& w) {
    if (wq - wdone >= kFcWRing) {
      const long long c0 = clock64();
      do {
        wdone = s_flag[3];
      } while (wq - wdone >= kFcWRing);
      cy_wput += clock64() - c0;
    }
    wring[wq & (kFcWRing - 1)] = w;
    ++wq;
  };
  auto wpublish = [&]() {
    __threadfence_block();
    s_flag[2] = wq;
  };
  auto wdrain = [&]() {  // the global entry state is current once the writer caught up
    const long long c0 = clock64();
    ++n_drain;
    wpublish();
    while (s_flag[3] < wq) {
    }
    __threadfence_block();
    wdone = wq;
    cy_drain += clock64() - c0;
  };
  auto is_gone = [&](int s) { return (gone[s >> 5] >> (s & 31)) & 1u; };
  auto set_gone = [&](int s) { gone[s >> 5] |= 1u << (s & 31); };
  int lo_s = 1 << 30, lo_p = 1 << 30;  // lowest mirrored stack index pushed (flushed at the end)
  auto spush = [&](int v, uint32_t g) {
    const int x = L.free_slot_top++;
    const unsigned m = (unsigned)(x - bs);
    if (m < (unsigned)kFcMirror) {
      ms_val[m] = v;
      ms_gen[m] = g;
      lo_s = min(lo_s, x);
    } else {
      c.free_slots[x] = v;
    }
  };
  auto ppush = [&](int v) {
    const int x = L.free_page_top++;
    const unsigned m = (unsigned)(x - bp);
    if (m < (unsigned)kFcMirror) {
      mp_val[m] = v;
      lo_p = min(lo_p, x);
    } else {
      c.free_pages[x] = v;
    }
  };
  int log_n = 0;
  int stop = (int)n;
  int pend = 0;
  // the hot control fields in registers, counters relative to the batch start
  long long tot = L.total_bytes;
  const long long budget = L.budget;
  int alive = L.alive, ni = 0, ne = 0;
  if (L.side_count > 0) stop = 0;  // pinned entries wait at the LRU end: the warp policy handles them
  const InsRec* rt_base = rbuf;
  int k = kFcTile - 1, t = -1;
  for (int i = 0; i < stop; ++i) {
    if (++k == kFcTile) {  // next record tile
      k = 0;
      ++t;
      const long long c0 = clock64();
      mbar_wait(&bars[t & 1], (t >> 1) & 1);
      cy_tile += clock64() - c0;
      rt_waited = t;
      rt_base = rbuf + (t & 1) * kFcTile;
    }
    const InsRec r = rt_base[k];
    if (k == kFcTile - 1 && t + 2 < nrt) {  // tile consumed: fetch tile t + 2 into its buffer
      rt_issued = t + 2;
      fence_proxy_async();
      mbar_expect_tx(&bars[t & 1], kRecTile);
      bulk_load(rbuf + (t & 1) * kFcTile, rec + (int64_t)(t + 2) * kFcTile, kRecTile, &bars[t & 1]);
    }
    if (r.nr < 0) {  // config error: the warp latches it
      stop = i;
      break;
    }
    const int np = r.nr > 0 ? 1 : 0;
    int s = -1, pg_old = -1;
    uint32_t g_old = 0;
    long long nb_old = 0;
    bool ow = false;
    if (r.prev >= 0) {  // the key's entry was made earlier in this batch: read it once written
      wdrain();
      s = out_slot[r.prev];
      g_old = out_gen[r.prev];
      nb_old = c.nbytes[s];
      pg_old = c.pages[s];
      ow = true;
    } else if (r.s0 >= 0 && !is_gone(r.s0)) {
      s = r.s0;
      g_old = r.gen0;
      nb_old = r.nb0;
      pg_old = r.pg0;
      ow = true;
    }
    if ((!ow && L.free_slot_top == 0) || L.free_page_top + (ow && pg_old >= 0 ? 1 : 0) < np) {
      stop = i;  // capacity: the warp latches the error / rolls back as the reference shape does
      break;
    }
    uint32_t g;
    if (ow) {  // overwrite: the key keeps its slot, the entry is new
      tot -= nb_old;
      if (pg_old >= 0) ppush(pg_old);
      g = g_old + 1u;
      if (r.prev < 0) set_gone(s);
    } else {
      const int x = --L.free_slot_top;
      const unsigned m = (unsigned)(x - bs);
      if (m < (unsigned)kFcMirror) {
        s = ms_val[m];
        g = ms_gen[m];
      } else {  // below the mirror: global, current once the writer caught up
        wdrain();
        s = c.free_slots[x];
        g = c.gen[s];
      }
      hlog[log_n++] = HashOp{r.d, s, 0};
      ++alive;
    }
    int pg = -1;
    if (np) {
      const int x = --L.free_page_top;
      const unsigned m = (unsigned)(x - bp);
      pg = m < (unsigned)kFcMirror ? mp_val[m] : c.free_pages[x];
    }
    wput(WRec{r.d, s, g, pg, i, r.nr, r.vv});
    ++ni;
    tot += r.nb;
    while (tot > budget && alive > 1) {
      // next_victim over the start-of-batch candidates
      bool found = false;
      CandRec v;
      for (;;) {
        if (ci >= ccnt) {
          if (ct + 1 >= nct) break;  // scanned window used up
          if (ct + 2 < nct) {
            ct_issued = ct + 2;
            fence_proxy_async();
            mbar_expect_tx(&bars[2 + (ct & 1)], kCandTile);
            bulk_load(cbuf + (ct & 1) * kFcTile, cand + (int64_t)(ct + 2) * kFcTile, kCandTile, &bars[2 + (ct & 1)]);
          }
          ++ct;
          ci = 0;
          const long long c0 = clock64();
          mbar_wait(&bars[2 + (ct & 1)], (ct >> 1) & 1);
          cy_tile += clock64() - c0;
          ccnt = cnt_s[ct];
          continue;
        }
        v = cbuf[(ct & 1) * kFcTile + ci++];
        if (is_gone(v.s)) continue;  // overwritten during the batch: its event died
        if (v.pins > 0) {            // pinned: to the side list (next_victim)
          if (L.side_count < c.side_cap) {
            c.side_slot[L.side_count] = v.s;
            c.side_clock[L.side_count] = v.ck;
            L.side_count++;
          } else if (!L.error) {
            L.error = LC_E_CAPACITY;
          }
          continue;
        }
        found = true;
        break;
      }
      if (!found) {  // every scanned event consumed: the warp continues from the ring tail
        pend = 1;
        break;
      }
      // evict_entry
      set_gone(v.s);
      hlog[log_n++] = HashOp{v.dg, -1, 0};
      tot -= v.nb;
      if (v.pg >= 0) ppush(v.pg);
      spush(v.s, v.gen + 1u);
      wput(WRec{0ull, v.s, v.gen + 1u, v.pg >= 0 ? 1 : 0, -1, 0, 0});
      --alive;
      ++ne;
    }
    if ((i & 31) == 31) {  // publish every 32 inserts (the fence waits for this thread's stores)
      __threadfence_block();
      s_flag[0] = log_n;
      s_flag[2] = wq;
    }
    if (pend) {
      stop = i + 1;
      break;
    }
  }
  // the ring tail: past the last candidate taken (every scanned event when they ran out)
  if (pend) {
    L.ring_tail = lim;
  } else if (nct > 0 && ci > 0) {
    L.ring_tail = tail0 + cbuf[(ct & 1) * kFcTile + ci - 1].off + 1;
  } else if (nct > 0 && ct > 0) {  // (a tile boundary: the last record of the previous tile)
    L.ring_tail = tail0 + (long long)ct * kFcTile;
  }
  L.total_bytes = tot;
  L.alive = alive;
  L.clock += ni;
  L.ring_head += ni;
  L.inserts += ni;
  L.evictions += ne;
  // drain the tile loads still in flight (a CTA must not exit with bulk copies pending)
  for (int t = rt_waited + 1; t <= rt_issued; ++t) mbar_wait(&bars[t & 1], (t >> 1) & 1);
  for (int t = (nct > 0 ? ct : -1) + 1; t <= ct_issued; ++t) mbar_wait(&bars[2 + (t & 1)], (t >> 1) & 1);
  // the mirrored stack ranges back to memory
  for (int x = lo_s; x < min(bs + kFcMirror, L.free_slot_top); ++x) c.free_slots[x] = ms_val[x - bs];
  for (int x = lo_p; x < min(bp + kFcMirror, L.free_page_top); ++x) c.free_pages[x] = mp_val[x - bp];
  *c.ctl = L;
  resume[0] = (int)stop;
  resume[1] = pend;
  reinterpret_cast<unsigned long long*>(resume)[2] = globaltimer_ns();
  reinterpret_cast<long long*>(resume)[4] = cy_wput;
  reinterpret_cast<long long*>(resume)[5] = cy_drain;
  reinterpret_cast<long long*>(resume)[6] = cy_tile;
  reinterpret_cast<long long*>(resume)[7] = n_drain;
  __threadfence_block();
  s_flag[0] = log_n;
  s_flag[2] = wq;
  s_flag[1] = 1;
}

__host__ __device__ constexpr size_t fc_smem_bytes(int ntiles, int E) {
  return 64 + 2 * kFcTile * (sizeof(InsRec) + sizeof(CandRec)) + kFcWRing * sizeof(WRec) + 32 * kFcWin * 12 +
         (size_t)kFcMirror * 12 + (size_t)ntiles * 4 + (size_t)((E + 31) / 32) * 4;
}

// Copy the rows/tokens of inserts whose entry is still alive at the end of the batch.
template <typename SrcT, typename DstT>
__global__ void insert_copy_kernel(CacheDev c, const int32_t* __restrict__ lens, const int32_t* __restrict__ vocabs,
                                   const char* __restrict__ src, int64_t src_stride, const int64_t* __restrict__ offs,
                                   const int32_t* __restrict__ toks, const int32_t* __restrict__ out_slot,
                                   const uint32_t* __restrict__ out_gen, int64_t i0,
                                   const int32_t* __restrict__ keep) {
  const int64_t i = i0 + blockIdx.y;
  const int s = out_slot[i];
  if (s < 0 || !c.alive[s] || c.gen[s] != out_gen[i]) return;
  const int nr = lens[i], vv = vocabs[i];
  const int kp = keep ? keep[i] : 0;
  for (int t = blockIdx.x; t < nr; t += gridDim.x) {
    const int pg = c.pages[(int64_t)s * c.maxp + t / c.page_rows];
    const int64_t slab_row = (int64_t)pg * c.page_rows + t % c.page_rows;
    if (threadIdx.x == 0 && (toks || t >= kp)) c.tokens[slab_row] = toks ? toks[offs[i] + t] : 0;
    if (t < kp || !src) continue;
    if (threadIdx.x == 0) invalidate_score(c, slab_row);  // replayed prefix in place / rows written later by the producer
    const SrcT* srow = reinterpret_cast<const SrcT*>(src) + (offs[i] + t) * src_stride;
    DstT* drow = reinterpret_cast<DstT*>(c.slab) + slab_row * (int64_t)c.V;
    const bool same = sizeof(SrcT) == sizeof(DstT);
    const bool al = ((reinterpret_cast<uintptr_t>(srow) | reinterpret_cast<uintptr_t>(drow)) & 15) == 0;
    if (same && al) {
      const int per = 16 / sizeof(DstT);
      const int nv = vv / per;
      // streaming (evict-first) loads and stores: rows pass through L2 once and must not
      // evict the index / event ring / entry metadata the policy warp works on
      for (int k = threadIdx.x; k < nv; k += blockDim.x)
        __stcs(reinterpret_cast<uint4*>(drow) + k, __ldcs(reinterpret_cast<const uint4*>(srow) + k));
      for (int k = nv * per + threadIdx.x; k < vv; k += blockDim.x) drow[k] = reinterpret_cast<const DstT*>(srow)[k];
    } else {
      for (int k = threadIdx.x; k < vv; k += blockDim.x) {
        float f;
        if (sizeof(SrcT) == 4) f = reinterpret_cast<const float*>(srow)[k];
        else f = bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(srow)[k]);
        if (sizeof(DstT) == 4) reinterpret_cast<float*>(drow)[k] = f;
        else reinterpret_cast<uint16_t*>(drow)[k] = f32_to_bf16_bits(f);
      }
    }
  }
}

__global__ void pin_kernel(CacheDev c, const int32_t* __restrict__ slot, const uint32_t* __restrict__ gen, int64_t n,
                           int delta) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = slot[i];
  if (s < 0 || s >= c.E) return;
  if (c.alive[s] && c.gen[s] == gen[i]) atomicAdd(&c.pins[s], delta);
}

template <typename DstT>
__global__ void gather_kernel(CacheDev c, const int32_t* __restrict__ slot, const int32_t* __restrict__ pos,
                              const uint32_t* __restrict__ gen, int64_t n, DstT* out, int64_t out_stride) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const int s = slot[i], t = pos[i];
  DstT* o = out + i * out_stride;
  bool ok = row_live(c, s, t, gen, i);
  const int vv = ok ? c.vocab[s] : 0;
  const int64_t slab_row =
      ok ? (int64_t)c.pages[(int64_t)s * c.maxp + t / c.page_rows] * c.page_rows + t % c.page_rows : 0;
  for (int k = threadIdx.x; k < out_stride; k += blockDim.x) {
    float f = 0.0f;
    if (ok && k < vv) {
      if (c.dtype == LC_F32) f = reinterpret_cast<const float*>(c.slab)[slab_row * c.V + k];
      else f = bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(c.slab)[slab_row * c.V + k]);
    }
    if (sizeof(DstT) == 4) reinterpret_cast<float*>(o)[k] = f;
    else reinterpret_cast<uint16_t*>(o)[k] = f32_to_bf16_bits(f);
  }
}

// slab address of cached row (slot, pos) -- null when the entry or position is gone
__global__ void row_ptr_kernel(CacheDev c, const int32_t* __restrict__ slot, const int32_t* __restrict__ pos,
                               const uint32_t* __restrict__ gen, int64_t n, const char** out, int32_t* vocab_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = slot[i], t = pos[i];
  const bool ok = row_live(c, s, t, gen, i);
  const size_t esz = c.dtype == LC_F32 ? 4 : 2;
  out[i] = ok ? c.slab + ((int64_t)c.pages[(int64_t)s * c.maxp + t / c.page_rows] * c.page_rows + t % c.page_rows) *
                             (int64_t)c.V * esz
              : nullptr;
  vocab_out[i] = ok ? c.vocab[s] : 1;
}

__global__ void tokens_kernel(CacheDev c, const int32_t* __restrict__ slot, const int32_t* __restrict__ pos,
                              const uint32_t* __restrict__ gen, int64_t n, int32_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = slot[i], t = pos[i];
  if (!row_live(c, s, t, gen, i)) {
    out[i] = -1;
    return;
  }
  int64_t slab_row = (int64_t)c.pages[(int64_t)s * c.maxp + t / c.page_rows] * c.page_rows + t % c.page_rows;
  out[i] = c.tokens[slab_row];
}

// Ring compaction: rebuild the ring from live entries sorted by last_hit.
__global__ void compact_keys_kernel(CacheDev c, unsigned long long* keys, int32_t* vals) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.E) return;
  keys[i] = c.alive[i] ? c.last_hit[i] : ~0ull;
  vals[i] = i;
}

__global__ void compact_write_kernel(CacheDev c, const unsigned long long* keys, const int32_t* vals) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int alive = c.ctl->alive;
  if (i < alive) {
    c.ring_clock[i] = keys[i];
    c.ring_slot[i] = vals[i];
  }
  if (i == 0) {
    c.ctl->ring_tail = 0;
    c.ctl->ring_head = alive;
    c.ctl->side_count = 0;
  }
}

__global__ void init_kernel(CacheDev c) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = i; k <= (int64_t)c.hmask; k += stride) c.hvals[k] = -1;
  for (int64_t k = i; k < c.E; k += stride) {
    c.free_slots[k] = c.E - 1 - (int)k;  // pop order 0, 1, 2, ... (oracle/cache_ref.py)
    c.alive[k] = 0;
    c.gen[k] = 0;
    c.pins[k] = 0;
    c.nrows[k] = 0;
    c.last_hit[k] = 0;
  }
  for (int64_t k = i; k < (int64_t)c.E * c.maxp; k += stride) c.pages[k] = -1;
  for (int64_t k = i; k < c.P; k += stride) c.free_pages[k] = c.P - 1 - (int)k;
  for (int64_t k = i; k < (int64_t)c.P * c.page_rows; k += stride) invalidate_score(c, k);
}

}  // namespace lcb

using namespace lcb;

struct lc_cache {
  lc_cache_config cfg;
  CacheDev dev;
  Ctl* d_ctl;
  void* sort_tmp;
  size_t sort_tmp_bytes;
  unsigned long long* sort_keys[2];
  int32_t* sort_vals[2];
  int32_t* d_probe;  // lookup probe results
  int64_t probe_cap;
  long long ring_bound;  // host upper bound of ring occupancy
  std::vector<void*> allocs;
  void* fc_buf;  // fast-commit scratch (records, candidates, hash log), grown on demand
  size_t fc_cap;
};

namespace lcb {
// device view of a handle, for kernels in other translation units (lc_engine.cu)
const CacheDev* cache_dev(const lc_cache* c) { return c ? &c->dev : nullptr; }
}  // namespace lcb

static int cache_alloc(lc_cache* c, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    lcb_set_last_error(cudaGetErrorString(e), __FILE__, __LINE__);
    return LC_E_CUDA;
  }
  c->allocs.push_back(*p);
  return LC_OK;
}

extern "C" int lc_cache_destroy(lc_cache* c) {
  if (!c) return LC_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  for (void* p : c->allocs) cudaFree(p);
  if (c->fc_buf) cudaFree(c->fc_buf);
  cudaSetDevice(dev);
  delete c;
  return LC_OK;
}

extern "C" int lc_cache_create(const lc_cache_config* cfg, lc_cache** out) {
  if (!cfg || !out) return LC_E_ARG;
  *out = nullptr;
  if (cfg->vocab < 1 || cfg->vocab > (1 << 28) || (cfg->dtype != LC_F32 && cfg->dtype != LC_BF16) ||
      cfg->page_rows < 1 || cfg->key_capacity < 1 || cfg->key_capacity > (1 << 30) || cfg->page_capacity < 1 ||
      cfg->page_capacity > (1ll << 31) - 1 || cfg->max_pages < 1 || cfg->budget_bytes < 0)
    return LC_E_CONFIG;
  LCB_CUDA_TRY(cudaSetDevice(cfg->device));
  if (const char* e = getenv("LCB_POLICY_PF")) {
    const int m = atoi(e);
    LCB_CUDA_TRY(cudaMemcpyToSymbol(g_pf_mode, &m, sizeof(int)));
  }
  lc_cache* c = new (std::nothrow) lc_cache();
  if (!c) return LC_E_CAPACITY;
  c->cfg = *cfg;
  CacheDev& d = c->dev;
  d.E = (int)cfg->key_capacity;
  d.P = (int)cfg->page_capacity;
  d.maxp = cfg->max_pages;
  d.page_rows = cfg->page_rows;
  d.V = (int)cfg->vocab;
  d.dtype = cfg->dtype;
  uint32_t H = 16;
  while (H < 2u * (uint32_t)d.E) H <<= 1;
  d.hmask = H - 1;
  d.R = 4096;
  while (d.R < 4ll * d.E + 4096) d.R <<= 1;
  d.rmask = d.R - 1;
  d.side_cap = d.E < 65536 ? d.E : 65536;
  const size_t esz = cfg->dtype == LC_F32 ? 4 : 2;
  int rc = 0;
#define ALLOC(ptr, n)                                                     \
  do {                                                                    \
    rc = cache_alloc(c, (void**)&(ptr), (size_t)(n) * sizeof(*(ptr)));    \
    if (rc) {                                                             \
      lc_cache_destroy(c);                                                \
      return rc;                                                          \
    }                                                                     \
  } while (0)
  ALLOC(c->d_ctl, 1);
  d.ctl = c->d_ctl;
  ALLOC(d.hkeys, H);
  ALLOC(d.hvals, H);
  ALLOC(d.digest, d.E);
  ALLOC(d.last_hit, d.E);
  ALLOC(d.gen, d.E);
  ALLOC(d.pins, d.E);
  ALLOC(d.nrows, d.E);
  ALLOC(d.vocab, d.E);
  ALLOC(d.alive, d.E);
  ALLOC(d.nbytes, d.E);
  ALLOC(d.pages, (int64_t)d.E * d.maxp);
  ALLOC(d.free_slots, d.E);
  ALLOC(d.free_pages, d.P);
  ALLOC(d.tokens, (int64_t)d.P * d.page_rows);
  ALLOC(d.score, (int64_t)d.P * d.page_rows);
  ALLOC(d.score_err, (int64_t)d.P * d.page_rows);
  ALLOC(d.score_T, (int64_t)d.P * d.page_rows);
  rc = cache_alloc(c, (void**)&d.slab, (size_t)d.P * d.page_rows * d.V * esz);
  if (rc) {
    lc_cache_destroy(c);
    return LC_E_CAPACITY;
  }
  ALLOC(d.ring_clock, d.R);
  ALLOC(d.ring_slot, d.R);
  ALLOC(d.side_clock, d.side_cap);
  ALLOC(d.side_slot, d.side_cap);
  for (int k = 0; k < 2; ++k) {
    ALLOC(c->sort_keys[k], d.E);
    ALLOC(c->sort_vals[k], d.E);
  }
  c->sort_tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, c->sort_tmp_bytes, c->sort_keys[0], c->sort_keys[1], c->sort_vals[0],
                                  c->sort_vals[1], d.E);
  rc = cache_alloc(c, &c->sort_tmp, c->sort_tmp_bytes);
  if (rc) {
    lc_cache_destroy(c);
    return rc;
  }
  c->probe_cap = 0;
  c->d_probe = nullptr;
#undef ALLOC
  Ctl h{};
  h.budget = cfg->budget_bytes;
  h.free_slot_top = d.E;
  h.free_page_top = d.P;
  LCB_CUDA_TRY(cudaMemcpy(c->d_ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice));
  init_kernel<<<1024, 256>>>(d);
  LCB_CUDA_TRY(cudaGetLastError());
  LCB_CUDA_TRY(cudaDeviceSynchronize());
  c->ring_bound = 0;
  *out = c;
  return LC_OK;
}

static int ensure_ring(lc_cache* c, int64_t incoming, cudaStream_t st) {
  if (c->ring_bound + incoming <= c->dev.R) return LC_OK;
  CacheDev& d = c->dev;
  compact_keys_kernel<<<ceil_div(d.E, 256), 256, 0, st>>>(d, c->sort_keys[0], c->sort_vals[0]);
  LCB_CUDA_TRY(cudaGetLastError());
  size_t tb = c->sort_tmp_bytes;
  LCB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->sort_tmp, tb, c->sort_keys[0], c->sort_keys[1], c->sort_vals[0],
                                               c->sort_vals[1], d.E, 0, 64, st));
  compact_write_kernel<<<ceil_div(d.E, 256), 256, 0, st>>>(d, c->sort_keys[1], c->sort_vals[1]);
  LCB_CUDA_TRY(cudaGetLastError());
  c->ring_bound = d.E;
  if (c->ring_bound + incoming > d.R) return LC_E_CAPACITY;  // batch larger than the ring
  return LC_OK;
}

extern "C" int lc_cache_lookup(lc_cache* c, const uint64_t* d_digests, int64_t n, int32_t* d_slot, uint32_t* d_gen,
                               int32_t* d_len, int32_t* d_vocab, void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_digests || !d_slot))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_ring(c, n, st);
  if (rc) return rc;
  const int threads = 256;
  lookup_probe_kernel<<<ceil_div(n * 8, threads), threads, 0, st>>>(c->dev, d_digests, n, d_slot);
  LCB_CUDA_TRY(cudaGetLastError());
  lookup_commit_kernel<<<1, 1024, 0, st>>>(c->dev, d_slot, n, d_gen, d_len, d_vocab, nullptr);
  LCB_CUDA_TRY(cudaGetLastError());
  c->ring_bound += n;
  return LC_OK;
}

static int insert_impl(lc_cache* c, const uint64_t* d_digests, const int32_t* d_lengths, const int32_t* d_vocabs,
                       int64_t n, const void* d_rows, int32_t rows_dtype, int64_t rows_stride,
                       const int64_t* d_row_offsets, const int32_t* d_tokens, int32_t max_len, int32_t* d_slot,
                       uint32_t* d_gen, const int32_t* d_keep, const uint32_t* d_keep_gen, cudaStream_t st) {
  int rc = ensure_ring(c, n, st);
  if (rc) return rc;
  const char* sp = getenv("LCB_SCALAR_POLICY");  // A/B hooks, read per call (tests switch them)
  const bool scalar = sp && atoi(sp) != 0;
  const char* fe = getenv("LCB_FAST_COMMIT");
  long long mcap = 8 * n + 4096;
  if (mcap > c->dev.R) mcap = c->dev.R;
  mcap = (mcap + kFcTile - 1) / kFcTile * kFcTile;
  const int ntiles = (int)(mcap / kFcTile);
  const size_t smem = fc_smem_bytes(ntiles, c->dev.E);
  const bool fast = !scalar && !d_keep && c->dev.maxp == 1 && n <= 65536 && smem <= 232448 &&
                    !(fe && atoi(fe) == 0);
  if (scalar) {
    insert_policy_scalar_kernel<<<1, 32, 0, st>>>(c->dev, d_digests, d_lengths, d_vocabs, n, d_slot, d_gen, d_keep,
                                                  d_keep_gen);
  } else if (fast) {
    const size_t nrec = (size_t)(n + kFcTile - 1) / kFcTile * kFcTile;
    const size_t o_cand = nrec * sizeof(InsRec);
    const size_t o_cnt = o_cand + (size_t)mcap * sizeof(CandRec);
    const size_t o_log = (o_cnt + (size_t)ntiles * 4 + 15) / 16 * 16;
    const size_t o_res = o_log + (size_t)(n + mcap) * sizeof(HashOp);
    const size_t need = o_res + 64;  // resume[0..1] + commit start / commit end / log end (ns)
    if (need > c->fc_cap) {
      if (c->fc_buf) LCB_CUDA_TRY(cudaFree(c->fc_buf));
      c->fc_buf = nullptr;
      c->fc_cap = 0;
      LCB_CUDA_TRY(cudaMalloc(&c->fc_buf, need));
      c->fc_cap = need;
    }
    char* b = (char*)c->fc_buf;
    InsRec* rec = (InsRec*)b;
    CandRec* cand = (CandRec*)(b + o_cand);
    int* cnt = (int*)(b + o_cnt);
    HashOp* hlog = (HashOp*)(b + o_log);
    int* resume = (int*)(b + o_res);
    static bool smem_set = false;
    if (!smem_set) {
      LCB_CUDA_TRY(cudaFuncSetAttribute(commit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
      smem_set = true;
    }
    prep_keys_kernel<<<ceil_div(n * 8, 256), 256, 0, st>>>(c->dev, d_digests, d_lengths, d_vocabs, n, rec);
    prep_prev_kernel<<<ceil_div(n, 256), 256, 0, st>>>(d_digests, n, rec);
    prep_cand_kernel<<<ntiles, 256, 0, st>>>(c->dev, mcap, cand, cnt);
    commit_kernel<<<1, 128, smem, st>>>(c->dev, rec, n, cand, cnt, ntiles, mcap, hlog, d_slot, d_gen, resume);
    insert_policy_kernel<<<1, 32, 0, st>>>(c->dev, d_digests, d_lengths, d_vocabs, n, d_slot, d_gen, d_keep,
                                           d_keep_gen, resume);
    if (getenv("LCB_FC_PROF")) {  // phase times of the fast commit (diagnostic, synchronises)
      unsigned long long h[8];
      LCB_CUDA_TRY(cudaMemcpyAsync(h, resume, sizeof(h), cudaMemcpyDeviceToHost, st));
      LCB_CUDA_TRY(cudaStreamSynchronize(st));
      fprintf(stderr,
              "fast_commit n=%lld stop=%d pend=%d commit_us=%.1f log_us=%.1f wput_kcy=%.1f drain_kcy=%.1f (%llu) "
              "tile_kcy=%.1f\n",
              (long long)n, (int)(h[0] & 0xffffffffu), (int)(h[0] >> 32), (h[2] - h[1]) * 1e-3, (h[3] - h[1]) * 1e-3,
              h[4] * 1e-3, h[5] * 1e-3, h[7], h[6] * 1e-3);
    }
  } else {
    insert_policy_kernel<<<1, 32, 0, st>>>(c->dev, d_digests, d_lengths, d_vocabs, n, d_slot, d_gen, d_keep,
                                           d_keep_gen, nullptr);
  }
  LCB_CUDA_TRY(cudaGetLastError());
  c->ring_bound += n;
  if (max_len > 0 && (d_rows || d_tokens)) {
    const int bx = max_len < 64 ? max_len : 64;
    for (int64_t i0 = 0; i0 < n; i0 += 65535) {
      const int ny = (int)((n - i0) < 65535 ? (n - i0) : 65535);
      dim3 grid(bx, ny);
      const char* src = (const char*)d_rows;
      if (rows_dtype == LC_F32 && c->cfg.dtype == LC_F32)
        insert_copy_kernel<float, float><<<grid, 256, 0, st>>>(c->dev, d_lengths, d_vocabs, src, rows_stride,
                                                               d_row_offsets, d_tokens, d_slot, d_gen, i0, d_keep);
      else if (rows_dtype == LC_F32)
        insert_copy_kernel<float, uint16_t><<<grid, 256, 0, st>>>(c->dev, d_lengths, d_vocabs, src, rows_stride,
                                                                  d_row_offsets, d_tokens, d_slot, d_gen, i0, d_keep);
      else if (c->cfg.dtype == LC_BF16)
        insert_copy_kernel<uint16_t, uint16_t><<<grid, 256, 0, st>>>(c->dev, d_lengths, d_vocabs, src, rows_stride,
                                                                     d_row_offsets, d_tokens, d_slot, d_gen, i0,
                                                                     d_keep);
      else
        insert_copy_kernel<uint16_t, float><<<grid, 256, 0, st>>>(c->dev, d_lengths, d_vocabs, src, rows_stride,
                                                                  d_row_offsets, d_tokens, d_slot, d_gen, i0, d_keep);
      LCB_CUDA_TRY(cudaGetLastError());
    }
  }
  return LC_OK;
}

extern "C" int lc_cache_insert(lc_cache* c, const uint64_t* d_digests, const int32_t* d_lengths,
                               const int32_t* d_vocabs, int64_t n, const void* d_rows, int32_t rows_dtype,
                               int64_t rows_stride, const int64_t* d_row_offsets, const int32_t* d_tokens,
                               int32_t max_len, int32_t* d_slot, uint32_t* d_gen, void* stream) {
  if (!c || n < 0) return LC_E_ARG;
  if (n == 0) return LC_OK;
  if (!d_digests || !d_lengths || !d_vocabs || !d_slot || !d_gen || !d_row_offsets) return LC_E_ARG;
  if (max_len > 0 && !d_rows) return LC_E_ARG;
  if (rows_dtype != LC_F32 && rows_dtype != LC_BF16) return LC_E_ARG;
  return insert_impl(c, d_digests, d_lengths, d_vocabs, n, d_rows, rows_dtype, rows_stride, d_row_offsets, d_tokens,
                     max_len, d_slot, d_gen, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int lc_cache_writeback(lc_cache* c, const uint64_t* d_digests, const int32_t* d_lengths,
                                  const int32_t* d_vocabs, const int32_t* d_keep, const uint32_t* d_keep_gen,
                                  int64_t n, const void* d_rows, int32_t rows_dtype, int64_t rows_stride,
                                  const int64_t* d_row_offsets, const int32_t* d_tokens, int32_t max_len,
                                  int32_t* d_slot, uint32_t* d_gen, void* stream) {
  if (!c || n < 0) return LC_E_ARG;
  if (n == 0) return LC_OK;
  if (!d_digests || !d_lengths || !d_vocabs || !d_keep || !d_keep_gen || !d_slot || !d_gen) return LC_E_ARG;
  if ((d_rows || d_tokens) && !d_row_offsets) return LC_E_ARG;
  if (rows_dtype != LC_F32 && rows_dtype != LC_BF16) return LC_E_ARG;
  return insert_impl(c, d_digests, d_lengths, d_vocabs, n, d_rows, rows_dtype, rows_stride, d_row_offsets, d_tokens,
                     max_len, d_slot, d_gen, d_keep, d_keep_gen, (cudaStream_t)stream);
}

// f1: the synthetic producer writing straight into cached rows (slot, pos) of live entries
// (model.py:67-83, kernels.py:47-60): no staging row, no insert copy.
template <typename OutT>
__global__ void fill_rows_kernel(CacheDev c, const int32_t* __restrict__ slot, const uint32_t* __restrict__ gen,
                                 const int32_t* __restrict__ pos, const uint64_t* __restrict__ states, int64_t n,
                                 double conc, double range) {
  const int64_t i = blockIdx.y;
  if (i >= n) return;
  const int s = slot[i], t = pos[i];
  if (!row_live(c, s, t, gen, i)) return;
  const int64_t vocab = c.vocab[s];
  const int64_t slab_row = (int64_t)c.pages[(int64_t)s * c.maxp + t / c.page_rows] * c.page_rows + t % c.page_rows;
  OutT* o = reinterpret_cast<OutT*>(c.slab) + slab_row * (int64_t)c.V;
  if (blockIdx.x == 0 && threadIdx.x == 0) invalidate_score(c, slab_row);
  const uint64_t st = states[i];
  const uint64_t peak = avalanche64(st ^ kPeakSalt) % (uint64_t)vocab;
  const float boost = (float)__dmul_rn(conc, range);
  produce_row<OutT>(o, vocab, st, peak, boost, range, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
}

__global__ void set_tokens_kernel(CacheDev c, const int32_t* __restrict__ slot, const uint32_t* __restrict__ gen,
                                  const int32_t* __restrict__ pos, const int32_t* __restrict__ tok, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = slot[i], t = pos[i];
  if (!row_live(c, s, t, gen, i)) return;
  c.tokens[(int64_t)c.pages[(int64_t)s * c.maxp + t / c.page_rows] * c.page_rows + t % c.page_rows] = tok[i];
}

__global__ void entry_len_kernel(CacheDev c, const int32_t* __restrict__ slot, const uint32_t* __restrict__ gen,
                                 int64_t n, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = slot[i];
  out[i] = (s >= 0 && s < c.E && c.alive[s] && c.gen[s] == gen[i]) ? c.nrows[s] : -1;
}

extern "C" int lc_cache_entry_len(lc_cache* c, const int32_t* d_slot, const uint32_t* d_gen, int64_t n,
                                  int32_t* d_len, void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_slot || !d_gen || !d_len))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  entry_len_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(c->dev, d_slot, d_gen, n, d_len);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_cache_fill_rows(lc_cache* c, const int32_t* d_slot, const uint32_t* d_gen, const int32_t* d_pos,
                                  const uint64_t* d_states, int64_t n, double concentration, double logit_range,
                                  void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_slot || !d_gen || !d_pos || !d_states))) return LC_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t i0 = 0; i0 < n; i0 += 65535) {
    const int ny = (int)((n - i0) < 65535 ? (n - i0) : 65535);
    const int bx = (int)(ceil_div(c->cfg.vocab, 256) < 32 ? ceil_div(c->cfg.vocab, 256) : 32);
    dim3 grid(bx, ny);
    if (c->cfg.dtype == LC_F32)
      fill_rows_kernel<float><<<grid, 256, 0, st>>>(c->dev, d_slot + i0, d_gen + i0, d_pos + i0, d_states + i0, ny,
                                                    concentration, logit_range);
    else
      fill_rows_kernel<uint16_t><<<grid, 256, 0, st>>>(c->dev, d_slot + i0, d_gen + i0, d_pos + i0, d_states + i0, ny,
                                                       concentration, logit_range);
    LCB_CUDA_TRY(cudaGetLastError());
  }
  return LC_OK;
}

extern "C" int lc_cache_set_tokens(lc_cache* c, const int32_t* d_slot, const uint32_t* d_gen, const int32_t* d_pos,
                                   const int32_t* d_tokens, int64_t n, void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_slot || !d_gen || !d_pos || !d_tokens))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  set_tokens_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(c->dev, d_slot, d_gen, d_pos, d_tokens, n);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_cache_pin(lc_cache* c, const int32_t* d_slot, const uint32_t* d_gen, int64_t n, int32_t delta,
                            void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_slot || !d_gen))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  pin_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(c->dev, d_slot, d_gen, n, delta);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_cache_gather(lc_cache* c, const int32_t* d_slot, const int32_t* d_pos, const uint32_t* d_gen,
                               int64_t n, void* d_out, int32_t out_dtype, int64_t out_stride, void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_slot || !d_pos || !d_out)) || out_stride < 1) return LC_E_ARG;
  if (n == 0) return LC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t i0 = 0; i0 < n; i0 += (1 << 30)) {
    int64_t nn = n - i0 < (1 << 30) ? n - i0 : (1 << 30);
    if (out_dtype == LC_F32)
      gather_kernel<float><<<(unsigned)nn, 256, 0, st>>>(c->dev, d_slot + i0, d_pos + i0, d_gen ? d_gen + i0 : nullptr, nn,
                                                         (float*)d_out + i0 * out_stride, out_stride);
    else
      gather_kernel<uint16_t><<<(unsigned)nn, 256, 0, st>>>(c->dev, d_slot + i0, d_pos + i0, d_gen ? d_gen + i0 : nullptr, nn,
                                                            (uint16_t*)d_out + i0 * out_stride, out_stride);
    LCB_CUDA_TRY(cudaGetLastError());
  }
  return LC_OK;
}

extern "C" int lc_cache_tokens(lc_cache* c, const int32_t* d_slot, const int32_t* d_pos, const uint32_t* d_gen,
                               int64_t n, int32_t* d_out, void* stream) {
  if (!c || n < 0 || (n > 0 && (!d_slot || !d_pos || !d_out))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  tokens_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(c->dev, d_slot, d_pos, d_gen, n, d_out);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

namespace lcb {
int launch_entropy_ptrs(const char* const* d_rows, const int32_t* d_vocab, int dtype, int64_t n, double T, double* H,
                        double* pmax, cudaStream_t st);
}

extern "C" int lc_cache_row_entropy(lc_cache* c, const int32_t* d_slot, const int32_t* d_pos, const uint32_t* d_gen,
                                    int64_t n, double temperature, double* d_entropy, double* d_pmax, void* stream) {
  if (!c || n < 0 || !(temperature >= 0.0) || (n > 0 && (!d_slot || !d_pos || !d_entropy || !d_pmax)))
    return LC_E_ARG;
  if (n == 0) return LC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  void* scratch = nullptr;  // row addresses + vocab sizes, stream-ordered
  LCB_CUDA_TRY(cudaMallocAsync(&scratch, (size_t)n * (sizeof(char*) + sizeof(int32_t)) + 16, st));
  const char** ptrs = reinterpret_cast<const char**>(scratch);
  int32_t* voc = reinterpret_cast<int32_t*>(ptrs + n);
  row_ptr_kernel<<<ceil_div(n, 256), 256, 0, st>>>(c->dev, d_slot, d_pos, d_gen, n, ptrs, voc);
  int rc = LC_OK;
  if (cudaGetLastError() != cudaSuccess) rc = LC_E_CUDA;
  if (rc == LC_OK) rc = lcb::launch_entropy_ptrs(ptrs, voc, c->dev.dtype, n, temperature, d_entropy, d_pmax, st);
  LCB_CUDA_TRY(cudaFreeAsync(scratch, st));
  return rc;
}

extern "C" int lc_cache_resample(lc_cache* c, const lc_task* d_tasks, int64_t n_tasks, lc_draws draws,
                                 void* d_workspace, int64_t workspace_bytes, int64_t* d_counters, void* stream) {
  if (!c) return LC_E_ARG;
  return lcb::resample_launch(c->dev.slab, c->dev.dtype, c->dev.V, c->dev.V, d_tasks, n_tasks, draws, c->dev.pages,
                              c->dev.maxp, c->dev.page_rows, d_workspace, workspace_bytes, d_counters,
                              (cudaStream_t)stream);
}

extern "C" int lc_cache_stats_get(lc_cache* c, lc_cache_stats* out, void* stream) {
  if (!c || !out) return LC_E_ARG;
  Ctl h;
  cudaStream_t st = (cudaStream_t)stream;
  LCB_CUDA_TRY(cudaMemcpyAsync(&h, c->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  LCB_CUDA_TRY(cudaStreamSynchronize(st));
  out->entries = h.alive;
  out->total_bytes = h.total_bytes;
  out->budget_bytes = h.budget;
  out->lookups = h.lookups;
  out->hits = h.hits;
  out->inserts = h.inserts;
  out->evictions = h.evictions;
  out->clock = h.clock;
  out->free_pages = h.free_page_top;
  out->free_slots = h.free_slot_top;
  out->error = h.error;
  if (h.error) {
    int zero = 0;
    LCB_CUDA_TRY(cudaMemcpyAsync(&c->d_ctl->error, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    LCB_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return LC_OK;
}

extern "C" int lc_cache_slab(lc_cache* c, void** d_base, int64_t* row_stride, int32_t* dtype) {
  if (!c) return LC_E_ARG;
  if (d_base) *d_base = c->dev.slab;
  if (row_stride) *row_stride = c->dev.V;
  if (dtype) *dtype = c->dev.dtype;
  return LC_OK;
}

extern "C" int lc_cache_page_table(lc_cache* c, const int32_t** d_pages, int32_t* max_pages, int32_t* page_rows) {
  if (!c) return LC_E_ARG;
  if (d_pages) *d_pages = c->dev.pages;
  if (max_pages) *max_pages = c->dev.maxp;
  if (page_rows) *page_rows = c->dev.page_rows;
  return LC_OK;
}

extern "C" int lc_cache_snapshot(lc_cache* c, uint64_t* d_digest, unsigned long long* d_last_hit, uint32_t* d_gen,
                                 int32_t* d_pins, int32_t* d_nrows, int32_t* d_vocab, uint8_t* d_alive,
                                 void* stream) {
  if (!c) return LC_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t E = (size_t)c->dev.E;
  if (d_digest) LCB_CUDA_TRY(cudaMemcpyAsync(d_digest, c->dev.digest, E * 8, cudaMemcpyDeviceToDevice, st));
  if (d_last_hit) LCB_CUDA_TRY(cudaMemcpyAsync(d_last_hit, c->dev.last_hit, E * 8, cudaMemcpyDeviceToDevice, st));
  if (d_gen) LCB_CUDA_TRY(cudaMemcpyAsync(d_gen, c->dev.gen, E * 4, cudaMemcpyDeviceToDevice, st));
  if (d_pins) LCB_CUDA_TRY(cudaMemcpyAsync(d_pins, c->dev.pins, E * 4, cudaMemcpyDeviceToDevice, st));
  if (d_nrows) LCB_CUDA_TRY(cudaMemcpyAsync(d_nrows, c->dev.nrows, E * 4, cudaMemcpyDeviceToDevice, st));
  if (d_vocab) LCB_CUDA_TRY(cudaMemcpyAsync(d_vocab, c->dev.vocab, E * 4, cudaMemcpyDeviceToDevice, st));
  if (d_alive) LCB_CUDA_TRY(cudaMemcpyAsync(d_alive, c->dev.alive, E, cudaMemcpyDeviceToDevice, st));
  return LC_OK;
}
