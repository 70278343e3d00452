// K2 (batched rolling prefix hasher), request uniforms and the synthetic
// logits producer (K5).  All integer-exact w.r.t. the reference:
//   hash_tokens / fold_token  -- mixing.py:63-73
//   RngStream                 -- mixing.py:81-98
//   fill_logits               -- kernels.py:47-60, _mixcore.pyx:27-40,
//                                determinism.md:55-76
#include "lc_common.cuh"

namespace lcb {

// One thread per prompt: the fold is sequential and non-associative
// (hard part 10) so it only parallelises across prompts.
// Tokens are read with a 4-wide vector when aligned to amortise LSU issue.
__global__ void hash_prefix_kernel(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets,
                                   const uint64_t* __restrict__ parent, int64_t n, uint64_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t b = offsets[i], e = offsets[i + 1];
  uint64_t h = parent ? parent[i] : kEmptyHash;
  int64_t t = b;
  for (; t < e && (t & 3); ++t) h = fold_token(h, tokens[t]);
  for (; t + 4 <= e; t += 4) {
    int4 v = *reinterpret_cast<const int4*>(tokens + t);
    h = fold_token(h, v.x);
    h = fold_token(h, v.y);
    h = fold_token(h, v.z);
    h = fold_token(h, v.w);
  }
  for (; t < e; ++t) h = fold_token(h, tokens[t]);
  out[i] = h;
}

__global__ void uniforms_kernel(const uint64_t* __restrict__ seeds, const int64_t* __restrict__ index, int64_t n,
                                double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = request_uniform(seeds[i], (uint64_t)index[i]);
}

// base_v = f32((2*unit_float(stream_u64(state, v)) - 1) * r) evaluated in f64
// (no FMA contraction: __dmul_rn/__dsub_rn keep the reference's two roundings),
// then peak += f32(c*r) in f32.
template <typename OutT>
__global__ void fill_logits_kernel(const uint64_t* __restrict__ states, int64_t n_rows, int64_t vocab, double conc,
                                   double range, OutT* __restrict__ out, int64_t stride) {
  int64_t row = blockIdx.y;
  if (row >= n_rows) return;
  uint64_t st = states[row];
  uint64_t peak = avalanche64(st ^ kPeakSalt) % (uint64_t)vocab;
  float boost = (float)__dmul_rn(conc, range);
  OutT* o = out + row * stride;
  produce_row<OutT>(o, vocab, st, peak, boost, range, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
}

}  // namespace lcb

using namespace lcb;

extern "C" int lc_hash_prefix(const int32_t* d_tokens, const int64_t* d_offsets, const uint64_t* d_parent,
                              int64_t n_prompts, uint64_t* d_out, void* stream) {
  if (n_prompts < 0 || (n_prompts > 0 && (!d_offsets || !d_out))) return LC_E_ARG;
  if (n_prompts == 0) return LC_OK;
  int threads = 128;
  hash_prefix_kernel<<<ceil_div(n_prompts, threads), threads, 0, (cudaStream_t)stream>>>(d_tokens, d_offsets,
                                                                                        d_parent, n_prompts, d_out);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_uniforms(const uint64_t* d_seeds, const int64_t* d_index, int64_t n, double* d_out, void* stream) {
  if (n < 0 || (n > 0 && (!d_seeds || !d_index || !d_out))) return LC_E_ARG;
  if (n == 0) return LC_OK;
  uniforms_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(d_seeds, d_index, n, d_out);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

extern "C" int lc_fill_logits(const uint64_t* d_states, int64_t n_rows, int64_t vocab, double concentration,
                              double logit_range, int dtype, void* d_out, int64_t row_stride, void* stream) {
  if (n_rows < 0 || vocab < 2 || row_stride < vocab || !d_out || !d_states) return LC_E_ARG;
  if (n_rows == 0) return LC_OK;
  if (n_rows > 65535) {
    // split the y-dimension
    for (int64_t r0 = 0; r0 < n_rows; r0 += 65535) {
      int64_t nr = n_rows - r0 < 65535 ? n_rows - r0 : 65535;
      size_t esz = dtype == LC_F32 ? 4 : 2;
      int rc = lc_fill_logits(d_states + r0, nr, vocab, concentration, logit_range, dtype,
                              (char*)d_out + r0 * row_stride * esz, row_stride, stream);
      if (rc) return rc;
    }
    return LC_OK;
  }
  int threads = 256;
  int bx = ceil_div(vocab, threads);
  if (bx > 64) bx = 64;
  dim3 grid(bx, (unsigned)n_rows);
  if (dtype == LC_F32) {
    fill_logits_kernel<float><<<grid, threads, 0, (cudaStream_t)stream>>>(d_states, n_rows, vocab, concentration,
                                                                          logit_range, (float*)d_out, row_stride);
  } else if (dtype == LC_BF16) {
    fill_logits_kernel<uint16_t><<<grid, threads, 0, (cudaStream_t)stream>>>(
        d_states, n_rows, vocab, concentration, logit_range, (uint16_t*)d_out, row_stride);
  } else {
    return LC_E_ARG;
  }
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}
