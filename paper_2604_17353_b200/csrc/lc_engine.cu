// The miss path of replay-aware generate (reference engine.py:336-347 with
// _prefill_internal / _decode_internal, engine.py:184-231) for a wave of requests,
// on the device: every decode step folds the previous token into the request's
// prefix digest (fold_token, mixing.py:63-65), produces the next logits row with the
// synthetic model (logits_from_state(mix2(seed, digest)), model.py:67-83) straight
// into the request's write-back entry in the slab, and emits the
// resample task of that row (draw number = the request's RngStream position).
//
//   lc_engine_fold         digest after the replayed tokens (prompt + out[:replayed])
//   lc_engine_decode_step  one decode step for every request of the wave
#include "lc_b200.h"
#include "lc_cache.cuh"
#include "lc_common.cuh"

namespace lcb {

const CacheDev* cache_dev(const lc_cache* c);

__global__ void engine_fold_kernel(const uint64_t* __restrict__ din, const int32_t* __restrict__ tok, int64_t stride,
                                   const int32_t* __restrict__ count, int64_t n, uint64_t* __restrict__ dout) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint64_t h = din[r];
  const int32_t* t = tok + r * stride;
  const int k = count[r];
  for (int i = 0; i < k; ++i) h = fold_token(h, t[i]);
  dout[r] = h;
}

// grid (ceil(V / chunk), B): the x blocks of request r fill its row together; every
// block of a row recomputes the (one-fold) digest, block x == 0 publishes it and the task.
template <typename OutT>
__global__ void engine_decode_kernel(CacheDev c, bool cache_rows, lc_decode_step a, int64_t chunk) {
  const int64_t r = blockIdx.y;
  if (r >= a.n) return;
  const int t = a.d_start[r] + a.step;
  const bool active = t < a.max_tokens;
  uint64_t d = a.d_digest_in[r];
  if (active && a.step > 0) d = fold_token(d, a.d_out[r * a.max_tokens + t - 1]);  // engine.py:227
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  bool live = false;
  int64_t srow = -1;
  if (active && cache_rows) {
    const int s = a.d_slot[r];
    live = row_live(c, s, t, a.d_gen, r) && c.vocab[s] == a.vocab;
    if (live) srow = slab_row_of(c, s, t);
  }
  if (lead) {
    if (live) invalidate_score(c, srow);
    a.d_digest_out[r] = d;
    lc_task tk;
    tk.row = a.d_staging ? r : (live ? srow : 0);
    tk.slot = -1;
    tk.pos = t;
    tk.temperature = a.d_temperature[r];
    tk.top_k = a.d_top_k[r];
    tk.vocab = a.vocab;
    tk.top_p = a.d_top_p[r];
    tk.draw_begin = r * a.max_tokens + (active ? t : 0);
    // an inactive request (or a dead entry with no staging row: the host checks) draws nothing
    tk.draw_end = tk.draw_begin + ((active && (a.d_staging || live)) ? 1 : 0);
    tk.seed_base = r;
    tk.u_index = a.d_u_start[r] + a.step;
    a.d_tasks[r] = tk;
  }
  if (!active) return;
  const uint64_t st = mix2(a.model_seed, d);  // logits_state (model.py:62-64)
  const uint64_t peak = avalanche64(st ^ kPeakSalt) % (uint64_t)a.vocab;
  const float boost = (float)__dmul_rn(a.concentration, a.logit_range);
  OutT* so = a.d_staging ? reinterpret_cast<OutT*>(a.d_staging) + r * a.staging_stride : nullptr;
  OutT* co = live ? reinterpret_cast<OutT*>(c.slab) + srow * (int64_t)c.V : nullptr;
  // the row's blocks stride over it in groups of 8 ids (one 16-byte store per 8 bf16, the stream
  // counter advanced by adds: produce_row, bit-identical to producer_value)
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if (co) produce_row<OutT>(co, a.vocab, st, peak, boost, a.logit_range, t0, nt);
  if (so) produce_row<OutT>(so, a.vocab, st, peak, boost, a.logit_range, t0, nt);
}

}  // namespace lcb

using namespace lcb;

extern "C" int lc_engine_fold(const uint64_t* d_digest_in, const int32_t* d_tokens, int64_t stride,
                              const int32_t* d_count, int64_t n, uint64_t* d_digest_out, void* stream) {
  if (n < 0 || (n > 0 && (!d_digest_in || !d_tokens || !d_count || !d_digest_out)) || stride < 0) return LC_E_ARG;
  if (n == 0) return LC_OK;
  engine_fold_kernel<<<ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(d_digest_in, d_tokens, stride, d_count, n,
                                                                         d_digest_out);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_engine_decode_step(lc_cache* cache, const lc_decode_step* step, void* stream) {
  if (!step) return LC_E_ARG;
  const lc_decode_step& a = *step;
  if (a.n < 0 || a.vocab < 2 || a.max_tokens < 1 || a.step < 0) return LC_E_ARG;
  if (a.n == 0) return LC_OK;
  if (!a.d_start || !a.d_u_start || !a.d_digest_in || !a.d_digest_out || !a.d_out || !a.d_temperature ||
      !a.d_top_k || !a.d_top_p || !a.d_tasks)
    return LC_E_ARG;
  if (!cache && !a.d_staging) return LC_E_ARG;
  if (cache && (!a.d_slot || !a.d_gen)) return LC_E_ARG;
  if (a.d_staging && a.staging_stride < a.vocab) return LC_E_ARG;
  if (a.n > 65535) return LC_E_ARG;
  const CacheDev* cd = cache_dev(cache);
  CacheDev c{};
  int dtype = a.staging_dtype;
  if (cd) {
    c = *cd;
    if (a.vocab > c.V) return LC_E_CONFIG;
    dtype = c.dtype;
    if (a.d_staging && a.staging_dtype != c.dtype) return LC_E_ARG;
  }
  const int64_t chunk = 4096;
  dim3 grid((unsigned)ceil_div(a.vocab, chunk), (unsigned)a.n);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == LC_F32)
    engine_decode_kernel<float><<<grid, 256, 0, st>>>(c, cd != nullptr, a, chunk);
  else if (dtype == LC_BF16)
    engine_decode_kernel<uint16_t><<<grid, 256, 0, st>>>(c, cd != nullptr, a, chunk);
  else
    return LC_E_ARG;
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}
