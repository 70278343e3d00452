// Fused replay plumbing: device-side task construction from lookup results
// and step-wise acceptance (engine.py:296-331), so that lookup -> resample ->
// accept runs as one stream-ordered sequence with no host synchronisation.
#include "lc_common.cuh"

namespace lcb {

__global__ void replay_tasks_kernel(const int32_t* __restrict__ slot, const int32_t* __restrict__ len,
                                    const int32_t* __restrict__ vocab, int64_t n_req,
                                    int max_pos, int nb, const double* __restrict__ temp,
                                    const int32_t* __restrict__ topk, const double* __restrict__ topp,
                                    lc_task* __restrict__ tasks) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req * (int64_t)max_pos) return;
  const int64_t r = i / max_pos;
  const int t = (int)(i % max_pos);
  const int s = slot[r];
  const int lim = s >= 0 ? min(len[r], max_pos) : 0;
  lc_task tk;
  tk.row = -1;
  tk.slot = s;
  tk.pos = t;
  tk.temperature = temp[r];
  tk.top_k = topk[r];
  tk.vocab = (vocab && s >= 0) ? vocab[r] : 0;  // the entry's own width (may be < the slab's)
  tk.top_p = topp[r];
  tk.draw_begin = i * nb;
  tk.draw_end = t < lim ? i * nb + nb : i * nb;
  tk.seed_base = r * nb;
  tk.u_index = t;
  tasks[i] = tk;
}

// one thread per (request, branch): first position whose draw differs from the
// cached token ends the replay; that divergent token is kept (engine.py:305-310)
__global__ void replay_accept_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ cached,
                                     const int32_t* __restrict__ len, int64_t n_req, int max_pos, int nb,
                                     int32_t* __restrict__ replayed, int32_t* __restrict__ diverged) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req * (int64_t)nb) return;
  const int64_t r = i / nb;
  const int b = (int)(i % nb);
  const int lim = min(len[r], max_pos);
  int rep = 0, div = -1;
  for (int t = 0; t < lim; ++t) {
    const int y = tok[((r * max_pos) + t) * (int64_t)nb + b];
    rep = t + 1;
    if (y != cached[r * max_pos + t]) {
      div = t;
      break;
    }
  }
  replayed[i] = rep;
  if (diverged) diverged[i] = div;
}

// Hotspot policy (engine.py:311-326): only hotspot positions draw; the stream's
// draw number at position t is the count of hotspots before t (d_draw_index,
// -1 = not a hotspot); every other position copies the cached token.
__global__ void replay_tasks_hot_kernel(const int32_t* __restrict__ slot, const int32_t* __restrict__ len,
                                        const int32_t* __restrict__ vocab, const int32_t* __restrict__ draw_index, int64_t n_req, int max_pos, int nb,
                                        const double* __restrict__ temp, const int32_t* __restrict__ topk,
                                        const double* __restrict__ topp, lc_task* __restrict__ tasks) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req * (int64_t)max_pos) return;
  const int64_t r = i / max_pos;
  const int t = (int)(i % max_pos);
  const int s = slot[r];
  const int lim = s >= 0 ? min(len[r], max_pos) : 0;
  const int di = draw_index[i];
  lc_task tk;
  tk.row = -1;
  tk.slot = s;
  tk.pos = t;
  tk.temperature = temp[r];
  tk.top_k = topk[r];
  tk.vocab = (vocab && s >= 0) ? vocab[r] : 0;  // the entry's own width (may be < the slab's)
  tk.top_p = topp[r];
  tk.draw_begin = i * nb;
  tk.draw_end = (t < lim && di >= 0) ? i * nb + nb : i * nb;
  tk.seed_base = r * nb;
  tk.u_index = di >= 0 ? di : 0;
  tasks[i] = tk;
}

// The same tasks for a compact list of hotspot positions only (flat index r * max_pos + t
// and its draw number): the resample sees n_hot tasks instead of n_req * max_pos.
__global__ void replay_tasks_hot_list_kernel(const int32_t* __restrict__ slot, const int32_t* __restrict__ len,
                                             const int32_t* __restrict__ vocab, const int64_t* __restrict__ hot_pos, const int32_t* __restrict__ hot_di,
                                             int64_t n_hot, int max_pos, int nb, const double* __restrict__ temp,
                                             const int32_t* __restrict__ topk, const double* __restrict__ topp,
                                             lc_task* __restrict__ tasks) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_hot) return;
  const int64_t i = hot_pos[j];
  const int64_t r = i / max_pos;
  const int t = (int)(i % max_pos);
  const int s = slot[r];
  const int lim = s >= 0 ? min(len[r], max_pos) : 0;
  lc_task tk;
  tk.row = -1;
  tk.slot = s;
  tk.pos = t;
  tk.temperature = temp[r];
  tk.top_k = topk[r];
  tk.vocab = (vocab && s >= 0) ? vocab[r] : 0;  // the entry's own width (may be < the slab's)
  tk.top_p = topp[r];
  tk.draw_begin = i * nb;
  tk.draw_end = t < lim ? i * nb + nb : i * nb;
  tk.seed_base = r * nb;
  tk.u_index = hot_di[j];
  tasks[j] = tk;
}

// Hotspot acceptance: non-hotspot positions take the cached token (written into
// d_tokens so the output is the engine's `out` list); the replay stops after the
// first hotspot whose sample differs from the cached token.
__global__ void replay_accept_hot_kernel(int32_t* __restrict__ tok, const int32_t* __restrict__ cached,
                                         const int32_t* __restrict__ len, const int32_t* __restrict__ draw_index,
                                         int64_t n_req, int max_pos, int nb, int32_t* __restrict__ replayed,
                                         int32_t* __restrict__ diverged) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req * (int64_t)nb) return;
  const int64_t r = i / nb;
  const int b = (int)(i % nb);
  const int lim = min(len[r], max_pos);
  int rep = 0, div = -1;
  for (int t = 0; t < lim; ++t) {
    const int64_t o = ((r * max_pos) + t) * (int64_t)nb + b;
    const int yc = cached[r * max_pos + t];
    int y = yc;
    if (draw_index[r * max_pos + t] >= 0) y = tok[o];
    else tok[o] = yc;
    rep = t + 1;
    if (y != yc) {
      div = t;
      break;
    }
  }
  replayed[i] = rep;
  if (diverged) diverged[i] = div;
}


// Windowed step-wise replay: the same acceptance (engine.py:296-331), evaluated W positions at a
// time so that rows are resampled only while one of the request's branches is still replaying
// (live[r] = its branches that neither diverged nor reached the limit).  Task j = r * W + k of
// window w0 is row (slot, w0 + k) with the draws of lc_replay_tasks' task r * max_pos + w0 + k,
// so tokens land where the full replay puts them.
__global__ void replay_window_init_kernel(const int32_t* __restrict__ len, int64_t n_req, int max_pos, int nb,
                                          int32_t* __restrict__ replayed, int32_t* __restrict__ diverged,
                                          int32_t* __restrict__ live, int32_t* __restrict__ n_live) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req * (int64_t)nb) return;
  const int64_t r = i / nb;
  replayed[i] = 0;
  diverged[i] = -1;
  if (i % nb == 0) {
    const int lv = min(len[r], max_pos) > 0 ? nb : 0;
    live[r] = lv;
    if (lv) atomicAdd(n_live, lv);
  }
}

__global__ void replay_window_tasks_kernel(const int32_t* __restrict__ slot, const int32_t* __restrict__ len,
                                           const int32_t* __restrict__ vocab, const int32_t* __restrict__ live,
                                           int64_t n_req, int max_pos, int nb, int w0, int W,
                                           const double* __restrict__ temp, const int32_t* __restrict__ topk,
                                           const double* __restrict__ topp, lc_task* __restrict__ tasks) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_req * (int64_t)W) return;
  const int64_t r = j / W;
  const int t = w0 + (int)(j % W);
  const int s = slot[r];
  const int lim = s >= 0 ? min(len[r], max_pos) : 0;
  const int64_t i = r * max_pos + min(t, max_pos - 1);
  lc_task tk;
  tk.row = -1;
  tk.slot = s;
  tk.pos = t;
  tk.temperature = temp[r];
  tk.top_k = topk[r];
  tk.vocab = (vocab && s >= 0) ? vocab[r] : 0;
  tk.top_p = topp[r];
  tk.draw_begin = i * nb;
  tk.draw_end = (t < lim && live[r] > 0) ? i * nb + nb : i * nb;
  tk.seed_base = r * nb;
  tk.u_index = t;
  tasks[j] = tk;
}

__global__ void replay_window_accept_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ cached,
                                            const int32_t* __restrict__ len, int64_t n_req, int max_pos, int nb,
                                            int w0, int W, int32_t* __restrict__ replayed,
                                            int32_t* __restrict__ diverged, int32_t* __restrict__ live,
                                            int32_t* __restrict__ n_live) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req * (int64_t)nb) return;
  const int64_t r = i / nb;
  const int b = (int)(i % nb);
  const int lim = min(len[r], max_pos);
  int rep = replayed[i];
  if (diverged[i] >= 0 || rep != w0 || rep >= lim) return;  // not live in this window
  const int t1 = min(w0 + W, lim);
  int div = -1;
  for (int t = w0; t < t1; ++t) {
    rep = t + 1;
    if (tok[((r * max_pos) + t) * (int64_t)nb + b] != cached[r * max_pos + t]) {
      div = t;
      break;
    }
  }
  replayed[i] = rep;
  if (div >= 0) diverged[i] = div;
  if (div >= 0 || rep >= lim) {
    atomicSub(&live[r], 1);
    atomicSub(n_live, 1);
  }
}

}  // namespace lcb

extern "C" int lc_replay_tasks_hotspot(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab,
                                       const int32_t* d_draw_index,
                                       int64_t n_req, int32_t max_pos, int32_t n_branch,
                                       const double* d_temperature, const int32_t* d_top_k, const double* d_top_p,
                                       lc_task* d_tasks, void* stream) {
  if (n_req < 0 || max_pos < 0 || n_branch < 0) return LC_E_ARG;
  const int64_t n = n_req * (int64_t)max_pos;
  if (n == 0) return LC_OK;
  if (!d_slot || !d_len || !d_draw_index || !d_temperature || !d_top_k || !d_top_p || !d_tasks) return LC_E_ARG;
  lcb::replay_tasks_hot_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_slot, d_len, d_vocab, d_draw_index, n_req, max_pos, n_branch, d_temperature, d_top_k, d_top_p, d_tasks);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_tasks_hotspot_list(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab,
                                            const int64_t* d_hot_pos,
                                            const int32_t* d_hot_draw, int64_t n_hot, int32_t max_pos,
                                            int32_t n_branch, const double* d_temperature, const int32_t* d_top_k,
                                            const double* d_top_p, lc_task* d_tasks, void* stream) {
  if (n_hot < 0 || max_pos < 0 || n_branch < 0) return LC_E_ARG;
  if (n_hot == 0) return LC_OK;
  if (!d_slot || !d_len || !d_hot_pos || !d_hot_draw || !d_temperature || !d_top_k || !d_top_p || !d_tasks)
    return LC_E_ARG;
  lcb::replay_tasks_hot_list_kernel<<<lcb::ceil_div(n_hot, 256), 256, 0, (cudaStream_t)stream>>>(
      d_slot, d_len, d_vocab, d_hot_pos, d_hot_draw, n_hot, max_pos, n_branch, d_temperature, d_top_k, d_top_p, d_tasks);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_accept_hotspot(int32_t* d_tokens, const int32_t* d_cached, const int32_t* d_len,
                                        const int32_t* d_draw_index, int64_t n_req, int32_t max_pos,
                                        int32_t n_branch, int32_t* d_replayed, int32_t* d_diverged, void* stream) {
  if (n_req < 0 || max_pos < 0 || n_branch < 0) return LC_E_ARG;
  const int64_t n = n_req * (int64_t)n_branch;
  if (n == 0) return LC_OK;
  if (!d_tokens || !d_cached || !d_len || !d_draw_index || !d_replayed) return LC_E_ARG;
  lcb::replay_accept_hot_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_tokens, d_cached, d_len, d_draw_index, n_req, max_pos, n_branch, d_replayed, d_diverged);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_tasks(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab, int64_t n_req,
                               int32_t max_pos,
                               int32_t n_branch, const double* d_temperature, const int32_t* d_top_k,
                               const double* d_top_p, lc_task* d_tasks, void* stream) {
  if (n_req < 0 || max_pos < 0 || n_branch < 0) return LC_E_ARG;
  const int64_t n = n_req * (int64_t)max_pos;
  if (n == 0) return LC_OK;
  if (!d_slot || !d_len || !d_temperature || !d_top_k || !d_top_p || !d_tasks) return LC_E_ARG;
  lcb::replay_tasks_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_slot, d_len, d_vocab, n_req, max_pos, n_branch, d_temperature, d_top_k, d_top_p, d_tasks);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_accept(const int32_t* d_tokens, const int32_t* d_cached, const int32_t* d_len, int64_t n_req,
                                int32_t max_pos, int32_t n_branch, int32_t* d_replayed, int32_t* d_diverged,
                                void* stream) {
  if (n_req < 0 || max_pos < 0 || n_branch < 0) return LC_E_ARG;
  const int64_t n = n_req * (int64_t)n_branch;
  if (n == 0) return LC_OK;
  if (!d_tokens || !d_cached || !d_len || !d_replayed) return LC_E_ARG;
  lcb::replay_accept_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_tokens, d_cached, d_len, n_req, max_pos, n_branch, d_replayed, d_diverged);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_window_init(const int32_t* d_len, int64_t n_req, int32_t max_pos, int32_t n_branch,
                                     int32_t* d_replayed, int32_t* d_diverged, int32_t* d_live, int32_t* d_n_live,
                                     void* stream) {
  if (n_req < 0 || max_pos < 0 || n_branch < 0) return LC_E_ARG;
  if (!d_len || !d_replayed || !d_diverged || !d_live || !d_n_live) return LC_E_ARG;
  LCB_CUDA_TRY(cudaMemsetAsync(d_n_live, 0, sizeof(int32_t), (cudaStream_t)stream));
  const int64_t n = n_req * (int64_t)n_branch;
  if (n == 0) return LC_OK;
  lcb::replay_window_init_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_len, n_req, max_pos, n_branch, d_replayed, d_diverged, d_live, d_n_live);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_window_tasks(const int32_t* d_slot, const int32_t* d_len, const int32_t* d_vocab,
                                      const int32_t* d_live, int64_t n_req, int32_t max_pos, int32_t n_branch,
                                      int32_t w0, int32_t window, const double* d_temperature,
                                      const int32_t* d_top_k, const double* d_top_p, lc_task* d_tasks, void* stream) {
  if (n_req < 0 || max_pos <= 0 || n_branch < 0 || w0 < 0 || window <= 0) return LC_E_ARG;
  const int64_t n = n_req * (int64_t)window;
  if (n == 0) return LC_OK;
  if (!d_slot || !d_len || !d_live || !d_temperature || !d_top_k || !d_top_p || !d_tasks) return LC_E_ARG;
  lcb::replay_window_tasks_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_slot, d_len, d_vocab, d_live, n_req, max_pos, n_branch, w0, window, d_temperature, d_top_k, d_top_p, d_tasks);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_replay_window_accept(const int32_t* d_tokens, const int32_t* d_cached, const int32_t* d_len,
                                       int64_t n_req, int32_t max_pos, int32_t n_branch, int32_t w0, int32_t window,
                                       int32_t* d_replayed, int32_t* d_diverged, int32_t* d_live, int32_t* d_n_live,
                                       void* stream) {
  if (n_req < 0 || max_pos < 0 || n_branch < 0 || w0 < 0 || window <= 0) return LC_E_ARG;
  const int64_t n = n_req * (int64_t)n_branch;
  if (n == 0) return LC_OK;
  if (!d_tokens || !d_cached || !d_len || !d_replayed || !d_diverged || !d_live || !d_n_live) return LC_E_ARG;
  lcb::replay_window_accept_kernel<<<lcb::ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_tokens, d_cached, d_len, n_req, max_pos, n_branch, w0, window, d_replayed, d_diverged, d_live, d_n_live);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}
