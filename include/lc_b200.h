/*
 * lc_b200.h -- C ABI of the B200-native Logits-Cache re-sampling path.
 *
 * This is the drop-in boundary for the reference's logits-cache interface
 * (reference: /root/reference/pkg/src/agentserve).  The
 * reference exposes that interface as in-process Python (no FFI); the entry
 * points below are what a binding of that interface needs, each one citing
 * the reference function it replaces.  INTEGRATION.md shows the ctypes
 * binding the reference side would add.
 *
 * Conventions
 *   - every function returns an int status (lc_status); nothing throws across
 *     the ABI; lc_last_error() describes the last failure on this thread;
 *   - pointers named d_* are DEVICE pointers on the handle's device; h_* are
 *     host pointers;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream); calls are asynchronous on that stream unless documented as
 *     synchronising;
 *   - a cache handle is single-threaded: the caller serialises calls (the
 *     reference serialises every cache access under InferenceEngine._lock,
 *     engine.py:113, 267-268).
 */
#ifndef LC_B200_H
#define LC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LC_ABI_VERSION 5

typedef enum lc_status {
  LC_OK = 0,
  LC_E_CONFIG = 1,    /* -> agentserve.errors.ConfigError (errors.py:6) */
  LC_E_ZERO_MASS = 2, /* -> RuntimeError (sampling.py:101-102) */
  LC_E_CAPACITY = 3,  /* slab pages or entry slots exhausted */
  LC_E_CUDA = 4,      /* CUDA runtime failure (lc_last_error has the text) */
  LC_E_ARG = 5,       /* bad argument (null pointer, negative size ...) */
  LC_E_STATE = 6      /* a write-back's replayed prefix is no longer the key's live entry */
} lc_status;

typedef enum lc_dtype { LC_F32 = 0, LC_BF16 = 1 } lc_dtype;

/* per-draw flags written by the resample entry points */
#define LC_DRAW_PRECISE 1u    /* decided by the fp64 precise pass (fast path uncertain) */
#define LC_DRAW_UNRESOLVED 2u /* even the precise pass could not certify the decision */
#define LC_DRAW_BAD_ROW 4u    /* non-finite maximum / NaN logits: token = -1 */

int lc_abi_version(void);
const char* lc_status_string(int status);
const char* lc_last_error(void);

/* ------------------------------------------------------------------ mixing
 * Bit-exact integer primitives (determinism.md:14-92).                    */

/* Rolling prefix hash, one digest per prompt: digest[i] = hash_tokens(
 * tokens[offsets[i] .. offsets[i+1]), start = parent ? parent[i] : EMPTY_HASH).
 * Replaces StateKey.of (logits_cache.py:31-32) -> hash_tokens (mixing.py:68-73)
 * and its O(1) prefix extension (fold_token, mixing.py:63-65).               */
int lc_hash_prefix(const int32_t* d_tokens, const int64_t* d_offsets, const uint64_t* d_parent,
                   int64_t n_prompts, uint64_t* d_out, void* stream);

/* u[i] = RngStream(seeds[i]).next_float() at draw index index[i]
 * (mixing.py:81-98).                                                          */
int lc_uniforms(const uint64_t* d_seeds, const int64_t* d_index, int64_t n, double* d_out, void* stream);

/* Synthetic logits producer (reference model.py:67-83 / kernels.py:47-71 /
 * _mixcore.pyx:27-40): row r = fill_logits(states[r], vocab, conc, range),
 * written as dtype (bf16 = RNE of the fp32 value) at d_out + r*row_stride.   */
int lc_fill_logits(const uint64_t* d_states, int64_t n_rows, int64_t vocab, double concentration,
                   double logit_range, int dtype, void* d_out, int64_t row_stride, void* stream);

/* ---------------------------------------------------------------- resample
 * One task = one logits row + sampling parameters + a range of draws that
 * share the row (Best-of-N siblings at the same position share it).  Token
 * decision per draw = sample(truncate(softmax(z, T), top_k, top_p), u)
 * (sampling.py:57-109), bit-exact given the same u.                          */
typedef struct lc_task {
  int64_t row;        /* row index into `rows` (row_stride elements apart); -1 = cache (slot,pos) */
  int32_t slot;       /* cache entry slot (lc_cache_resample only) */
  int32_t pos;        /* position inside the cached trajectory */
  double temperature; /* SamplingConfig.temperature (>= 0) */
  int32_t top_k;      /* <= 0: none (SamplingConfig.top_k None) */
  int32_t vocab;      /* <= 0: the row width passed to the call */
  double top_p;       /* (0, 1] */
  int64_t draw_begin; /* draws [draw_begin, draw_end) of this task */
  int64_t draw_end;
  int64_t seed_base;  /* seed mode: draw d uses d_seed[seed_base + d - draw_begin] */
  int64_t u_index;    /* seed mode: RngStream draw number (< 0: use pos, the step-wise index) */
} lc_task;

/* Draw source, one of:
 *   d_u != NULL                 u = d_u[draw]                       (FixedUniform)
 *   d_u == NULL, d_index != 0   u = RngStream(d_seed[draw]) draw number d_index[draw]
 *   d_u == NULL, d_index == 0   u = RngStream(d_seed[task.seed_base + draw - draw_begin])
 *                               draw number task.u_index (or task.pos)
 * RngStream values are computed on the device bit-exactly (mixing.py:91-98). */
typedef struct lc_draws {
  const double* d_u;
  const uint64_t* d_seed;
  const int64_t* d_index;
  int32_t* d_token; /* out */
  uint8_t* d_flags; /* out, LC_DRAW_* (may be NULL) */
  int32_t* d_kept;  /* out, per TASK (may be NULL): |kept| of truncate() (sampling.py:71-94) --
                     * the kept set is the first d_kept[t] ids of the row in (logit desc, id asc)
                     * order, i.e. the reference's lexsort((ids, -p)) prefix; V for an untruncated
                     * row, 1 for T == 0, -1 for a bad row (NaN / non-finite max)            */
  double* d_entropy; /* out, per TASK (may be NULL): H = -sum p ln p of softmax(z, T) over the
                      * task's row (the untruncated distribution, sampling.py:112-115); NaN for a
                      * task whose row cannot be resolved.  An epilogue launch over the same rows */
  double* d_pmax;    /* out, per TASK (may be NULL): max p of that softmax (sampling.py:118-119) */
} lc_draws;

/* Bytes of scratch the resample entry points need for n_tasks tasks. */
int64_t lc_resample_workspace_bytes(int64_t n_tasks, int64_t vocab);

/* Resample rows of a plain device array.  d_counters (may be NULL) receives
 * int64 {tasks sent to the precise pass, unresolved draws, bad rows}
 * accumulated (atomicAdd) on the device.                                      */
int lc_resample(const void* d_rows, int dtype, int64_t vocab, int64_t row_stride, const lc_task* d_tasks,
                int64_t n_tasks, lc_draws draws, void* d_workspace, int64_t workspace_bytes,
                int64_t* d_counters, void* stream);

/* Inverse-CDF draw over explicit fp64 probability rows (sampling.py:97-109):
 * token[r] for row r with uniform u[r]; zero mass -> token -1 and flag. */
int lc_draw_probs(const double* d_probs, int64_t vocab, int64_t n_rows, int64_t row_stride, const double* d_u,
                  int32_t* d_token, uint8_t* d_flags, void* stream);

/* truncate() on explicit fp64 probability rows (sampling.py:71-94): top-k
 * (k <= 0: none) then nucleus on the untruncated mass, renormalised, written
 * to d_out (zeros outside the kept set).  d_scratch: n_rows*vocab*12 + 256
 * bytes.  top_k <= 0 and top_p == 1 is the identity (the caller may skip). */
int lc_truncate_probs(const double* d_probs, int64_t vocab, int64_t n_rows, int64_t row_stride, int32_t top_k,
                      double top_p, double* d_out, void* d_scratch, void* stream);

/* softmax at temperature T (sampling.py:57-68) into fp64 probabilities, with
 * the reference's operation order (f64 divide, subtract max, exp, divide by
 * numpy's pairwise sum).                                                      */
int lc_softmax(const void* d_rows, int dtype, int64_t vocab, int64_t row_stride, int64_t n_rows,
               const double* d_temperature, double* d_out, void* stream);

/* Per-row entropy (nats) and max probability of softmax(z, T), the hotspot
 * scores' inputs (sampling.py:112-126).                                       */
/* Entropy -sum_{p>0} p ln p and max p of explicit probability rows
 * (sampling.py:112-119, `entropy` / `max_prob`), one block per row.         */
int lc_prob_stats(const double* d_probs, int64_t vocab, int64_t n_rows, int64_t row_stride, double* d_entropy,
                  double* d_pmax, void* stream);
int lc_row_entropy(const void* d_rows, int dtype, int64_t vocab, int64_t row_stride, int64_t n_rows,
                   double temperature, double* d_entropy, double* d_pmax, void* stream);

/* ------------------------------------------------------------------- cache
 * HBM-resident replacement of LogitsCache (logits_cache.py:73-183):
 * an open-addressing digest -> slot index, a slab of [pages x page_rows x
 * vocab] rows (fp32 or bf16), the reference's LRU-by-last-hit eviction over
 * accounted bytes n*V*4 + 8*n (logits_cache.py:54-56, 128-140) and pins.     */
typedef struct lc_cache lc_cache;

typedef struct lc_cache_config {
  int64_t vocab;          /* slab row width (entries may be narrower) */
  int32_t dtype;          /* lc_dtype of the slab */
  int32_t page_rows;      /* rows per page (>= 1) */
  int64_t key_capacity;   /* max live entries */
  int64_t page_capacity;  /* pages in the slab */
  int32_t max_pages;      /* max pages per entry (bounds trajectory length) */
  int32_t device;         /* CUDA device ordinal */
  int64_t budget_bytes;   /* accounted-byte budget (LogitsCache(budget_bytes)) */
} lc_cache_config;

typedef struct lc_cache_stats {
  int64_t entries;      /* len(cache) */
  int64_t total_bytes;  /* accounted, logits_cache.py:78 */
  int64_t budget_bytes;
  int64_t lookups;      /* logits_cache.py:82 */
  int64_t hits;
  int64_t inserts;
  int64_t evictions;
  int64_t clock;        /* _hit_clock, logits_cache.py:79 */
  int64_t free_pages;
  int64_t free_slots;
  int64_t error;        /* latched lc_status from inside insert batches (cleared on read) */
} lc_cache_stats;

int lc_cache_create(const lc_cache_config* cfg, lc_cache** out);
int lc_cache_destroy(lc_cache* cache);

/* LogitsCache.lookup for a batch (logits_cache.py:87-94) in index order:
 * out_slot = -1 on a miss; hits tick the clock in index order.  out_len,
 * out_vocab, out_gen describe the hit entry (may be NULL).                    */
int lc_cache_lookup(lc_cache* cache, const uint64_t* d_digests, int64_t n, int32_t* d_slot, uint32_t* d_gen,
                    int32_t* d_len, int32_t* d_vocab, void* stream);

/* LogitsCache.update for a batch (logits_cache.py:96-140), applied in index
 * order: entry i has d_lengths[i] rows, row t being d_rows[(d_row_offsets[i] +
 * t) * rows_stride ...] (rows_dtype, first d_vocabs[i] columns; converted to
 * the slab dtype with round-to-nearest-even) and token d_tokens[d_row_offsets[i]
 * + t].  Accounted bytes are n*V*4 + 8*n whatever the slab dtype
 * (logits_cache.py:54-56).  max_len (host) = max(d_lengths) sizes the copy grid.
 * d_slot/d_gen receive the (slot, generation) of the entry each insert created;
 * a later insert or an eviction in the same batch may already have replaced it.
 * Errors inside the batch (entry wider than the slab: LC_E_CONFIG, exhausted
 * slots/pages: LC_E_CAPACITY) are latched and reported by lc_cache_stats_get. */
int lc_cache_insert(lc_cache* cache, const uint64_t* d_digests, const int32_t* d_lengths, const int32_t* d_vocabs,
                    int64_t n, const void* d_rows, int32_t rows_dtype, int64_t rows_stride,
                    const int64_t* d_row_offsets, const int32_t* d_tokens, int32_t max_len, int32_t* d_slot,
                    uint32_t* d_gen, void* stream);

/* Write-back (engine.py:349-361: merged = Z[:replayed] ++ new_rows; cache.update(key,
 * merged, out)) without copying the replayed rows.  As lc_cache_insert,
 * plus per entry keep[i] = rows already in the slab: when keep[i] > 0 the insert must
 * overwrite the key's live entry of generation keep_gen[i] (the caller holds a pin on it,
 * lc_cache_pin), whose first keep[i] rows become rows 0 .. keep[i]-1 of the new entry in
 * place (an overwrite returns the old pages in page order, oracle/cache_ref.py); anything
 * else latches LC_E_STATE.  Rows keep[i] .. len-1 are copied from d_rows when given, else
 * left for lc_cache_fill_rows; tokens (all len of them) from d_tokens when given.
 * Accounted bytes follow the reference (n*V*4 + 8n) as for any update.              */
int lc_cache_writeback(lc_cache* cache, const uint64_t* d_digests, const int32_t* d_lengths, const int32_t* d_vocabs,
                       const int32_t* d_keep, const uint32_t* d_keep_gen, int64_t n, const void* d_rows,
                       int32_t rows_dtype, int64_t rows_stride, const int64_t* d_row_offsets, const int32_t* d_tokens,
                       int32_t max_len, int32_t* d_slot, uint32_t* d_gen, void* stream);

/* The synthetic producer (model.py:67-83 logits_from_state -> kernels.py:47-60
 * fill_logits) writing straight into cached rows (slot, pos) of live entries, over the
 * entry's vocab, as the slab dtype (the miss path's rows never pass
 * through a staging buffer or an insert copy).                                      */
int lc_cache_fill_rows(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, const int32_t* d_pos,
                       const uint64_t* d_states, int64_t n, double concentration, double logit_range, void* stream);

/* len(entry) of (slot, generation) handles, -1 when the entry was overwritten or
 * evicted (the reference's entry object is no longer in cache.entries).            */
int lc_cache_entry_len(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, int64_t n, int32_t* d_len,
                       void* stream);

/* entry.token_seq[pos] = tokens[i] for cached rows (slot, pos) of live entries. */
int lc_cache_set_tokens(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, const int32_t* d_pos,
                        const int32_t* d_tokens, int64_t n, void* stream);

/* pin/unpin (logits_cache.py:145-149) by (slot, generation) handles; a
 * handle whose entry was overwritten or evicted is ignored (the reference
 * pins the old entry object).  delta = +1 pin, -1 unpin.                     */
int lc_cache_pin(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, int64_t n, int32_t delta,
                 void* stream);

/* Copy cached rows (slot, pos) out as out_dtype (entry.logits_seq[pos]).  d_gen (may be
 * NULL) holds each row's (slot, generation) handle generation: a row whose entry was
 * overwritten or evicted since reads as zeros (tokens: -1), like a dead slot.      */
int lc_cache_gather(lc_cache* cache, const int32_t* d_slot, const int32_t* d_pos, const uint32_t* d_gen, int64_t n,
                    void* d_out, int32_t out_dtype, int64_t out_stride, void* stream);
/* Cached tokens (entry.token_seq[pos]); -1 for a dead / stale row. */
int lc_cache_tokens(lc_cache* cache, const int32_t* d_slot, const int32_t* d_pos, const uint32_t* d_gen, int64_t n,
                    int32_t* d_out, void* stream);

/* Hotspot scoring straight from the slab (sampling.py:112-125 on entry.logits_seq):
 * entropy H and max probability of softmax(z / T) for cached rows (slot, pos), fp64,
 * without gathering the rows; a missing row gives H = 0, max p = 1.             */
int lc_cache_row_entropy(lc_cache* cache, const int32_t* d_slot, const int32_t* d_pos, const uint32_t* d_gen, int64_t n,
                         double temperature, double* d_entropy, double* d_pmax, void* stream);

/* Hotspot scores kept beside the cached rows (sampling.py:112-130):
 * b = H * (1 - pmax) of softmax(z / T) for rows (slot, pos) of live entries, with a
 * bound on its distance to the reference's numpy evaluation; only_stale != 0 skips
 * rows already scored at this T (a row write makes its score stale).              */
int lc_cache_score_rows(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, const int32_t* d_pos, int64_t n,
                        double temperature, int32_t only_stale, void* stream);

/* Hotspot selection (select_hotspots over the entry's scores, sampling.py:133-160 /
 * hotspots_for, logits_cache.py:153-163) for n entries, on the device: rows must be
 * scored at `temperature` (lc_cache_score_rows).  Per entry r: d_draw_index[r*max_pos
 * + t] = number of hotspots before t when t is a hotspot, else -1 (the layout of
 * lc_replay_tasks_hotspot; may be NULL), d_n_hot[r] = hotspot count, d_flags[r]: 1 =
 * a decision within the score bounds of the threshold / cap (undecidable against the
 * reference), 2 = some row not scored at T, 4 = dead handle.  max_hotspots < 0: none. */
int lc_cache_hotspots(lc_cache* cache, const int32_t* d_slot, const uint32_t* d_gen, int64_t n_entries, int32_t max_pos,
                      double temperature, double decay, double threshold, int32_t max_hotspots, int32_t* d_draw_index,
                      int32_t* d_n_hot, uint8_t* d_flags, void* stream);

/* Resample cached rows: tasks use (slot, pos) with row = -1. */
int lc_cache_resample(lc_cache* cache, const lc_task* d_tasks, int64_t n_tasks, lc_draws draws, void* d_workspace,
                      int64_t workspace_bytes, int64_t* d_counters, void* stream);

/* Fused replay helpers (engine.py:296-331 for a batch of requests x branches).
 * lc_replay_tasks: request r (slot d_slot[r] from lc_cache_lookup, -1 = miss,
 * trajectory length d_len[r]) replays positions t < min(d_len[r], max_pos);
 * task r*max_pos + t resamples cached row (slot, t) for the request's n_branch
 * branches with draws [(r*max_pos + t)*n_branch, +n_branch), branch b using
 * seed d_seeds[r*n_branch + b] at draw number t (step-wise: one draw per
 * position, engine.py:301-310).  Positions past the limit get empty draw
 * ranges.  d_temperature/d_top_k/d_top_p are per request; d_vocab (may be NULL =
 * the slab width) is the entry's own row width from lc_cache_lookup, so an
 * entry narrower than the slab is resampled over its own columns only.        */
int lc_replay_tasks(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab, int64_t n_req,
                    int32_t max_pos, int32_t n_branch,
                    const double* d_temperature, const int32_t* d_top_k, const double* d_top_p, lc_task* d_tasks,
                    void* stream);
/* Step-wise acceptance: for request r, branch b, the replay keeps positions up
 * to and including the first sampled token that differs from the cached one
 * (engine.py:305-310).  d_tokens is the draw-indexed output of the resample;
 * d_cached[r*max_pos + t] the cached tokens (lc_cache_tokens).  Writes
 * replayed_len and diverged_at (-1 = none) per (r, b).                        */
int lc_replay_accept(const int32_t* d_tokens, const int32_t* d_cached, const int32_t* d_len, int64_t n_req,
                     int32_t max_pos, int32_t n_branch, int32_t* d_replayed, int32_t* d_diverged, void* stream);

/* Windowed step-wise replay: the acceptance of lc_replay_accept evaluated W
 * positions at a time, so rows are resampled only while a branch of the request
 * is still replaying (same replayed_len / diverged_at / accepted tokens as the
 * full replay; engine.py:296-331).  lc_replay_window_init sets replayed 0,
 * diverged -1, d_live[r] = n_branch for requests with a cached prefix (else 0)
 * and *d_n_live = their sum.  lc_replay_window_tasks writes n_req*window tasks
 * (task r*window + k = row (slot, w0 + k), the draws of lc_replay_tasks' task
 * r*max_pos + w0 + k; empty when the request has no live branch or past the
 * limit).  lc_replay_window_accept advances the live branches through the
 * window's draws and decrements d_live / *d_n_live for every branch that
 * diverges or reaches the limit; the caller stops when *d_n_live == 0.        */
int lc_replay_window_init(const int32_t* d_len, int64_t n_req, int32_t max_pos, int32_t n_branch,
                          int32_t* d_replayed, int32_t* d_diverged, int32_t* d_live, int32_t* d_n_live,
                          void* stream);
int lc_replay_window_tasks(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab,
                           const int32_t* d_live, int64_t n_req, int32_t max_pos, int32_t n_branch, int32_t w0,
                           int32_t window, const double* d_temperature, const int32_t* d_top_k,
                           const double* d_top_p, lc_task* d_tasks, void* stream);
int lc_replay_window_accept(const int32_t* d_tokens, const int32_t* d_cached, const int32_t* d_len, int64_t n_req,
                            int32_t max_pos, int32_t n_branch, int32_t w0, int32_t window, int32_t* d_replayed,
                            int32_t* d_diverged, int32_t* d_live, int32_t* d_n_live, void* stream);

/* Hotspot replay policy (engine.py:311-326, ReplayPolicy.HOTSPOT).
 * d_draw_index[r*max_pos + t] = number of hotspots of request r before t when
 * t is a hotspot (the RngStream draw number of that sample), else -1.
 * lc_replay_tasks_hotspot: as lc_replay_tasks, but only hotspot positions get
 * draws.  lc_replay_accept_hotspot: non-hotspot positions copy the cached
 * token (written into d_tokens, so d_tokens is the engine's `out` list); the
 * replay stops after the first hotspot whose sample differs from the cache.   */
int lc_replay_tasks_hotspot(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab,
                            const int32_t* d_draw_index, int64_t n_req,
                            int32_t max_pos, int32_t n_branch, const double* d_temperature, const int32_t* d_top_k,
                            const double* d_top_p, lc_task* d_tasks, void* stream);
/* The hotspot tasks for a compact list: d_hot_pos[j] = r * max_pos + t of the j-th
 * hotspot position, d_hot_draw[j] its draw number; writes n_hot tasks (draws at the
 * same indices as lc_replay_tasks_hotspot), so the resample skips non-hotspot rows.   */
int lc_replay_tasks_hotspot_list(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab,
                                 const int64_t* d_hot_pos,
                                 const int32_t* d_hot_draw, int64_t n_hot, int32_t max_pos, int32_t n_branch,
                                 const double* d_temperature, const int32_t* d_top_k, const double* d_top_p,
                                 lc_task* d_tasks, void* stream);
int lc_replay_accept_hotspot(int32_t* d_tokens, const int32_t* d_cached, const int32_t* d_len,
                             const int32_t* d_draw_index, int64_t n_req, int32_t max_pos, int32_t n_branch,
                             int32_t* d_replayed, int32_t* d_diverged, void* stream);

/* Test probe: the resample tiers' exponentials e(z) ~ exp((z - m)/T) for given
 * z (mode 0 FAST corrected, 1 FAST cheap, 2 PRECISE table fp64), so tests can
 * pin their error bounds against fp64 (not on the hot path).                  */
int lc_probe_exp(const float* d_z, int64_t n, float m, double temperature, int mode, double* d_out, void* stream);

/* Synchronising: copy the counters out. */
int lc_cache_stats_get(lc_cache* cache, lc_cache_stats* h_out, void* stream);

/* Slab geometry (for callers that resample slab rows through lc_resample). */
int lc_cache_slab(lc_cache* cache, void** d_base, int64_t* row_stride, int32_t* dtype);
/* Copy per-slot entry metadata out (any pointer may be NULL):
 * digest u64, last_hit u64, generation u32, pins i32, rows i32, vocab i32,
 * alive u8 -- arrays of key_capacity elements.  Used by tests (slot parity with
 * the oracle) and by CachedTrajectory's lazy fields.                          */
int lc_cache_snapshot(lc_cache* cache, uint64_t* d_digest, unsigned long long* d_last_hit, uint32_t* d_gen,
                      int32_t* d_pins, int32_t* d_nrows, int32_t* d_vocab, uint8_t* d_alive, void* stream);
/* Page table [key_capacity][max_pages] (-1 = unused), for fused consumers. */
int lc_cache_page_table(lc_cache* cache, const int32_t** d_pages, int32_t* max_pages, int32_t* page_rows);

/* ------------------------------------------------------------------ engine
 * The miss path of replay-aware generate (engine.py:336-347) for a WAVE of requests
 * (distinct prompt keys; the caller orders waves as the reference orders calls).    */

/* digest_out[r] = fold_token over tokens[r*stride .. r*stride + count[r]) starting at
 * digest_in[r]: StateKey digest of prompt + out[:replayed] (engine.py:337 prefill of
 * prompt + out; fold_token prefix extension, mixing.py:63-65).                       */
int lc_engine_fold(const uint64_t* d_digest_in, const int32_t* d_tokens, int64_t stride, const int32_t* d_count,
                   int64_t n, uint64_t* d_digest_out, void* stream);

/* One decode step `step` of every request r of the wave: position t = start[r] + step
 * (inactive once t >= max_tokens); for step > 0 the digest absorbs the previous token
 * out[r*max_tokens + t - 1] (engine.py:227); the row fill_logits(mix2(model_seed,
 * digest)) (model.py:62-83, engine.py:213/231) is written into the write-back entry's
 * slab row (slot[r], gen[r], t) when that row is live (f1: no staging, no copy) and into
 * staging row r when d_staging != NULL; task r (resample of that row, draw number
 * u_start[r] + step, token -> out[r*max_tokens + t]) goes to d_tasks[r]: resample it with
 * lc_cache_resample (no staging) or lc_resample over the staging rows.
 * Without a cache handle, d_staging is required.                                     */
typedef struct lc_decode_step {
  int64_t n;                  /* requests in the wave (<= 65535) */
  int32_t vocab;              /* model vocab (ModelConfig.vocab_size) */
  int32_t max_tokens;         /* SamplingConfig.max_tokens of the wave */
  int32_t step;               /* decode step index (0 = the prefill row) */
  int32_t staging_dtype;      /* lc_dtype of d_staging (must equal the slab dtype with a cache) */
  uint64_t model_seed;        /* ModelConfig.seed */
  double concentration;       /* ModelConfig.concentration */
  double logit_range;         /* ModelConfig.logit_range */
  const int32_t* d_start;     /* [n] first decoded position (= replayed_len) */
  const int64_t* d_u_start;   /* [n] RngStream draws consumed before the decode */
  const uint64_t* d_digest_in;/* [n] digest before this step's fold */
  uint64_t* d_digest_out;     /* [n] digest after it (ping-pong with d_digest_in) */
  const int32_t* d_out;       /* [n * max_tokens] generated tokens (previous step's token read) */
  const int32_t* d_slot;      /* [n] write-back entry (cache mode) */
  const uint32_t* d_gen;      /* [n] its generation */
  const double* d_temperature;/* [n] */
  const int32_t* d_top_k;     /* [n] (<= 0: none) */
  const double* d_top_p;      /* [n] */
  void* d_staging;            /* [n * staging_stride] rows or NULL */
  int64_t staging_stride;     /* elements */
  lc_task* d_tasks;           /* [n] out */
} lc_decode_step;

int lc_engine_decode_step(lc_cache* cache, const lc_decode_step* step, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LC_B200_H */
