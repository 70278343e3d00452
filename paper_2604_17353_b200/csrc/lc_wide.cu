// K1w: TMA-staged resample kernel for top-k rows of any width (BASELINE configs 3
// and 5: bf16, V = 151936, top-k 50 + top-p 0.95).
//
// Same CTA shape as lc_stage.cu: three 5-warp groups and a producer warp per SM,
// tasks (resolved rows, parameters, first 32 uniforms) handed over through a
// shared-memory FIFO.  A group streams its row through its 64 KB stage as 16000-id
// chunks in two 32 KB halves: chunk c+2 is loaded (cp.async.bulk + mbarrier) while
// chunk c+1 waits and chunk c is processed, so HBM sees every row once.
//
// Per chunk: the chunk max; while fewer than k candidates are known, a 256-class
// histogram below the chunk max gives a threshold the global k-th largest value
// cannot be below; the chunk mass relative to its max with fp32 MUFU exponentials
// (|a|-weighted bound) and the candidates z >= threshold appended to a shared list
// (compacted to the top k by a bitonic sort when it fills).  After the row: S from
// the chunk masses (fp64 rescale), the top-k by (value desc, id asc) = the
// reference's lexsort order, fp64 table exponentials of the k candidates, the
// nucleus cut on csum(p) certified against S's bound, and the draws over the kept
// set in id order (sampling.py:71-109), each certified; an uncertain task goes to
// the CTA kernel (lc_resample.cu).
#include "lc_common.cuh"
#include "lc_resample.cuh"
#include "lc_stage.cuh"
#include "lc_task.cuh"

namespace lcb {

constexpr int WG_GROUPS = 3;
constexpr int WG_GW = 5;
constexpr int WG_GT = WG_GW * 32;
constexpr int WG_PWARP = WG_GROUPS * WG_GW;
constexpr int WG_THREADS = (WG_PWARP + 1) * 32;
constexpr int WG_CH = 16000;                 // ids per chunk (one half-stage of 32000 B)
constexpr int WG_HALF16 = WG_CH * 2 / 16;    // uint4 per half
constexpr int WG_NCHMAX = 64;                // chunks per row (V <= 1,024,000)
constexpr int WG_K = 64;                     // largest effective top-k handled here
constexpr int WG_CAP = 512;                  // candidate list
constexpr int WG_HB = 256;                   // threshold histogram classes
constexpr int WG_NU = 32;
constexpr int WG_PB = 8;
constexpr int WG_FQ = 6;
constexpr double kLog2eW = 1.4426950408889634;
constexpr double kLn2W = 0.6931471805599453;

struct WgGroup {
  uint32_t hist[WG_HB + 32];  // + one dump bin per lane
  unsigned long long cand[WG_CAP];
  float cmax[WG_NCHMAX];
  double cs[WG_NCHMAX], cw[WG_NCHMAX];
  double su[WG_NU];
  double ke[WG_K];  // kept masses in id order
  int kid[WG_K];
  double rd[2][WG_GW];
  float rf[WG_GW];
  int ri[2][WG_GW];
  TaskView tv;
  int task, ncand, flag;
  float thr;
  unsigned long long thrk;  // after a compaction: the k-th largest key (value desc, id asc)
};

struct __align__(128) WgSmem {
  uint4 ring[WG_GROUPS][2 * WG_HALF16];
  WgGroup g[WG_GROUPS];
  TaskView fq_tv[WG_FQ];
  int fq_task[WG_FQ];
  double fq_u[WG_FQ][WG_NU];
  int fq_tail, fq_head;
  int fq_free[WG_FQ];  // per slot: the sequence number it may next be written for
  TaskView pbv[WG_PB];
  int pbt[WG_PB];
  double pbu[WG_PB][WG_NU];
  double t16[16];
  unsigned long long full[WG_GROUPS][2];
};
static_assert(sizeof(WgSmem) <= 232448, "wide kernel shared memory");

__device__ __forceinline__ void wbar(int g) { gbar_n<WG_GT>(g); }

// eligible: effective top-k <= WG_K, V % 8 == 0, V <= WG_NCHMAX chunks, 16 B rows
__device__ void wg_producer(const StageArgs& a, WgSmem& sm, int lane) {
  bool done = false;
  int sentinels = 0;
  // tasks per grab: WG_PB on big batches; fewer when the batch gives each group only a few rows,
  // so small launches (an engine decode step, a G = 8 rank's share) spread over every SM
  const int pb = max(1, min(WG_PB, a.n_tasks / (int)(gridDim.x * WG_GROUPS * 4)));
  for (;;) {
    int nb = 0;
    if (!done) {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(a.next, pb);
      t0 = __shfl_sync(0xffffffffu, t0, 0);
      if (t0 >= a.n_tasks) {
        done = true;
      } else {
        const int t = t0 + lane;
        bool ok = false;
        TaskView tv;
        if (lane < pb && t < a.n_tasks) {
          const lc_task tk = a.tasks[t];
          if (tk.draw_end > tk.draw_begin) {
            const int Vt = tk.vocab > 0 ? tk.vocab : a.Vdef;
            const bool topk = tk.top_k > 0 && tk.top_k < Vt && tk.top_k <= WG_K;
            ok = topk && !(Vt & 7) && Vt <= WG_NCHMAX * WG_CH &&
                 resolve_task(tk, a.rows, a.row_bytes, a.Vdef, a.cm, tv) && !(reinterpret_cast<uintptr_t>(tv.row) & 15);
            if (!ok) requeue(a, t);
          }
        }
        const unsigned okm = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          const int pos = __popc(okm & ((1u << lane) - 1u));
          sm.pbt[pos] = t;
          sm.pbv[pos] = tv;
        }
        __syncwarp();
        nb = __popc(okm);
        double ub[WG_PB];
#pragma unroll
        for (int j = 0; j < WG_PB; ++j) {
          ub[j] = 0.0;
          if (j < nb) {
            const TaskView& tj = sm.pbv[j];
            if (tj.d0 + lane < tj.d1) ub[j] = draw_u(a.io, tj.d0 + lane, tj);
          }
        }
#pragma unroll
        for (int j = 0; j < WG_PB; ++j) sm.pbu[j][lane] = ub[j];
        __syncwarp();
      }
    }
    const int npush = nb > 0 ? nb : (done ? WG_GROUPS - sentinels : 0);
    for (int j = 0; j < npush; ++j) {
      const int slot_seq = vload(&sm.fq_tail);
      // wait until the slot's previous occupant (sequence slot_seq - WG_FQ) was copied out by
      // its own consumer: consumers finish out of order, so a completion count is not enough
      if (lane == 0)
        // (the FIFO is full for most of a wide row: back off, so the spin takes few issue slots
        // from the group warps on this SM sub-partition)
        for (unsigned ns = 64; vload(&sm.fq_free[slot_seq % WG_FQ]) != slot_seq; ns = min(2 * ns, 2048u)) __nanosleep(ns);
      __syncwarp();
      const int slot = slot_seq % WG_FQ;
      if (nb > 0) {
        sm.fq_u[slot][lane] = sm.pbu[j][lane];
        if (lane == 0) {
          sm.fq_tv[slot] = sm.pbv[j];
          sm.fq_task[slot] = sm.pbt[j];
        }
      } else {
        if (lane == 0) sm.fq_task[slot] = -1;
        ++sentinels;
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) *reinterpret_cast<volatile int*>(&sm.fq_tail) = slot_seq + 1;
      __syncwarp();
    }
    if (done && sentinels >= WG_GROUPS) return;
  }
}

// group warp 0: next task into the group; the group barrier that follows publishes it
__device__ void wg_pop(WgSmem& sm, WgGroup& G, int lane) {
  int h = 0;
  if (lane == 0) {
    h = atomicAdd(&sm.fq_head, 1);
    while (vload(&sm.fq_tail) <= h) __nanosleep(32);
  }
  h = __shfl_sync(0xffffffffu, h, 0);
  __threadfence_block();
  const int slot = h % WG_FQ;
  const int t = sm.fq_task[slot];
  if (t >= 0) G.su[lane] = sm.fq_u[slot][lane];
  __syncwarp();
  if (lane == 0) {
    G.task = t;
    if (t >= 0) G.tv = sm.fq_tv[slot];
    G.ncand = 0;
    G.flag = 0;
    G.thr = -INFINITY;
    G.thrk = 0ull;
    __threadfence_block();
    *reinterpret_cast<volatile int*>(&sm.fq_free[slot]) = h + WG_FQ;  // slot h released
  }
  __syncwarp();
}

// descending sort of the group's candidate list (n <= WG_CAP) by its warp 0: a
// shuffle bitonic network in registers, no group barriers inside
template <int RL>
__device__ __noinline__ void warp_sort(unsigned long long* keys, int n, int lane);

__device__ void wg_sort(WgGroup& G, int g, int gt, int n) {
  static_assert(WG_CAP <= 512, "warp sort covers 512 keys");
  if (gt < 32) {
    if (n <= 128) warp_sort<4>(G.cand, n, gt);
    else if (n <= 256) warp_sort<8>(G.cand, n, gt);
    else warp_sort<16>(G.cand, n, gt);
  }
  wbar(g);
}

// (value order, id) -> descending order = (value desc, id asc), the reference's lexsort
__device__ __forceinline__ unsigned long long wkey(float v, int idx) {
  return ((unsigned long long)f32_order_key(v) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)idx);
}
// descending bitonic sort of up to 32*RL keys by one warp (RL per lane, shuffles only)
template <int RL>
__device__ __noinline__ void warp_sort(unsigned long long* keys, int n, int lane) {
  constexpr int NK = 32 * RL;
  unsigned long long x[RL];
#pragma unroll
  for (int r = 0; r < RL; ++r) x[r] = RL * lane + r < n ? keys[RL * lane + r] : 0ull;
#pragma unroll
  for (int k = 2; k <= NK; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= RL) {
        const int lj = j / RL;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int i = RL * lane + r;
          const bool desc = (i & k) == 0;
          const unsigned long long y = __shfl_xor_sync(0xffffffffu, x[r], lj);
          x[r] = (desc == lower) ? (x[r] > y ? x[r] : y) : (x[r] < y ? x[r] : y);
        }
      } else {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int rp = r ^ j;
          if (rp > r) {
            const int i = RL * lane + r;
            const bool desc = (i & k) == 0;
            const unsigned long long a = x[r], b = x[rp];
            if (desc ? (a < b) : (a > b)) {
              x[r] = b;
              x[rp] = a;
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RL; ++r)
    if (RL * lane + r < n) keys[RL * lane + r] = x[r];
}

__device__ __forceinline__ float key_val(unsigned long long k) {
  const uint32_t o = (uint32_t)(k >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ int key_id(unsigned long long k) { return (int)(0xffffffffu - (uint32_t)k); }

__global__ void __launch_bounds__(WG_THREADS, 1) wide_kernel(StageArgs a) {
  extern __shared__ __align__(128) unsigned char wraw[];
  WgSmem& sm = *reinterpret_cast<WgSmem*>(wraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < WG_GROUPS; ++s) {
      mbar_init(&sm.full[s][0], 1);
      mbar_init(&sm.full[s][1], 1);
    }
    mbar_fence_init();
    sm.fq_tail = sm.fq_head = 0;
    for (int s = 0; s < WG_FQ; ++s) sm.fq_free[s] = s;
  }
  if (tid < 16) sm.t16[tid] = exp2((double)tid / 16.0);
  __syncthreads();
  if (warp == WG_PWARP) {
    wg_producer(a, sm, lane);
    return;
  }
  const int g = warp / WG_GW, gw = warp % WG_GW, gt = tid - g * WG_GT;
  WgGroup& G = sm.g[g];
  const DrawIO& io = a.io;
  uint32_t ph0 = 0, ph1 = 0;  // parity of each half's mbarrier
  const bool prof = a.prof != nullptr && gt == 0;
  unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tp = prof ? clock64() : 0;
#define WG_PH(k)                                \
  do {                                          \
    if (prof) {                                 \
      const unsigned long long t_ = clock64();  \
      pc[k] += t_ - tp;                         \
      tp = t_;                                  \
    }                                           \
  } while (0)
  auto issue = [&](const TaskView& tv, int c) {  // lane 0 of warp 0
    const int len = min(WG_CH, tv.V - c * WG_CH);
    unsigned long long* bar = &sm.full[g][c & 1];
    mbar_expect_tx(bar, (uint32_t)(len * 2));
    bulk_load(sm.ring[g] + (c & 1) * WG_HALF16, tv.row + (size_t)c * WG_CH * 2, (uint32_t)(len * 2), bar);
  };

  for (;;) {
    if (gw == 0) wg_pop(sm, G, lane);
    wbar(g);
    const int task_id = G.task;
    if (task_id < 0) break;
    const TaskView tv = G.tv;
    const int V = tv.V, K = tv.topk;
    const int nch = (V + WG_CH - 1) / WG_CH;
    const int64_t d0 = tv.d0;
    const int nd = (int)(tv.d1 - tv.d0);
    if (gt == 0) {
      issue(tv, 0);
      if (nch > 1) issue(tv, 1);
    }
    const double Ld = tv.Ld;  // log2(e) / T from the producer (0 when T == 0)
    const float Lf = (float)Ld;
    bool bad = false;
    float M_run = -INFINITY;  // running max of the chunks seen
    float mLr = 0.0f;         // largest |reference| L of the chunk masses (their m L roundings)
    for (int c = 0; c < nch; ++c) {
      const int h = c & 1;
      mbar_wait(&sm.full[g][h], h ? ph1 : ph0);
      if (h) ph1 ^= 1u;
      else ph0 ^= 1u;
      WG_PH(0);
      const uint4* R = sm.ring[g] + h * WG_HALF16;
      const int nv = min(WG_CH, V - c * WG_CH) >> 3;
      // the chunk max is needed before the pass only for the first chunk (and while the
      // threshold histogram still runs); later chunks reference the running max M_run
      // and track their own max in the mass pass
      const bool need_thr = G.ncand < K;  // (group-uniform: read after the last barrier)
      float mc = M_run;
      if (c == 0 || need_thr) {
        uint32_t mx2 = 0xff80ff80u;
        for (int v = gt; v < nv; v += WG_GT) {
          const uint4 q = R[v];
          mx2 = bmax2_nan(mx2, bmax2_nan(bmax2_nan(q.x, q.y), bmax2_nan(q.z, q.w)));
        }
        const float tm = max_nan(lo_f(mx2), hi_f(mx2));
        const bool tn = tm != tm;
        const float wm = warp_max(tn ? INFINITY : tm);
        const bool wn = __any_sync(0xffffffffu, tn);
        if (lane == 0) {
          G.rf[gw] = wm;
          G.ri[0][gw] = wn;
        }
        wbar(g);
        mc = -INFINITY;
#pragma unroll
        for (int i = 0; i < WG_GW; ++i) {
          mc = fmaxf(mc, G.rf[i]);
          bad |= G.ri[0][i] != 0;
        }
        bad |= !(mc < INFINITY);
      }
      WG_PH(1);
      if (need_thr && mc > -INFINITY && !bad) {
        // threshold: the k-th largest value of this chunk, from a 256-class histogram
        for (int b = gt; b < WG_HB + 32; b += WG_GT) G.hist[b] = 0u;
        wbar(g);
        const uint32_t km = key16(__float_as_uint(mc));
        for (int v = gt; v < nv; v += WG_GT) {
          const uint4 q = R[v];
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t ol = km - key16(w[k] << 16), oh = km - key16(w[k] & 0xffff0000u);
            atomicAdd(&G.hist[ol < (uint32_t)WG_HB ? ol : WG_HB + lane], 1u);
            atomicAdd(&G.hist[oh < (uint32_t)WG_HB ? oh : WG_HB + lane], 1u);
          }
        }
        wbar(g);
        if (gw == 0) {  // first class where the count from the top reaches k
          int cnt[WG_HB / 32];
          int s8 = 0;
#pragma unroll
          for (int k = 0; k < WG_HB / 32; ++k) {
            cnt[k] = (int)G.hist[lane * (WG_HB / 32) + k];
            s8 += cnt[k];
          }
          int inc = s8;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
          }
          int run = inc - s8, hitb = INT_MAX;
#pragma unroll
          for (int k = 0; k < WG_HB / 32; ++k) {
            run += cnt[k];
            if (hitb == INT_MAX && run >= K) hitb = lane * (WG_HB / 32) + k;
          }
          hitb = warp_min_int(hitb);
          if (lane == 0 && hitb != INT_MAX) G.thr = fmaxf(G.thr, key16_to_f(km - (uint32_t)hitb));
        }
        wbar(g);
      }
      WG_PH(2);
      const float thr = G.thr;
      const unsigned long long thrk = G.thrk;
      // the vector pre-test as one compare: "> thr" once the list was compacted is ">= the next
      // float above thr" (NaN when thr is +inf: nothing passes)
      const float thr_c = !thrk ? thr : (thr < INFINITY ? nextafterf(thr, INFINITY) : __int_as_float(0x7fc00000));
      // mass relative to ref (fp32 MUFU, |a|-weighted bound), the chunk max, candidates >= thr
      const float ref = (c == 0 || need_thr) ? mc : M_run;
      const float nmL = -(ref * Lf);
      mLr = fmaxf(mLr, fabsf(ref) * Lf);
      double acc = 0.0;
      float W = 0.0f;
      uint32_t cm2 = 0xff80ff80u;
      if (!bad && ref > -INFINITY) {
        // two vectors
        // per lane and iteration, so the MUFU / add chains of one hide the other's latency
        auto cand_block = [&](const uint4 q, const uint32_t vm2, const int v) {
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
          // (once the list was compacted, only values above the k-th value can still enter)
          const float vmx = max_nan(lo_f(vm2), hi_f(vm2));
          const bool any_c = vmx >= thr_c;
          if (any_c) {
            // (ties of the k-th value with larger ids than the k-th key cannot enter: ids grow
            // with the chunks, so the list stops growing once it has been compacted).  Few
            // lanes ever get here (~0.3% of the values clear the threshold): one shared
            // atomic per candidate, no warp-wide scan.
            const int id0 = c * WG_CH + 8 * v;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float z = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
              if (z >= thr && z > -INFINITY) {
                const unsigned long long key = wkey(z, id0 + j);
                if (key > thrk) {
                  const int b = atomicAdd(&G.ncand, 1);
                  if (b < WG_CAP) G.cand[b] = key;
                }
              }
            }
          }
        };
        for (int v0 = gw * 32; v0 < nv; v0 += 2 * WG_GT) {
          const int va = v0 + lane, vb = v0 + WG_GT + lane;
          const uint4 ninf = make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);
          const uint4 qa = va < nv ? R[va] : ninf;
          const uint4 qb = vb < nv ? R[vb] : ninf;
          const uint32_t wa[4] = {qa.x, qa.y, qa.z, qa.w};
          const uint32_t wb[4] = {qb.x, qb.y, qb.z, qb.w};
          const uint32_t vma = bmax2_nan(bmax2_nan(wa[0], wa[1]), bmax2_nan(wa[2], wa[3]));
          const uint32_t vmb = bmax2_nan(bmax2_nan(wb[0], wb[1]), bmax2_nan(wb[2], wb[3]));
          cm2 = bmax2_nan(cm2, bmax2_nan(vma, vmb));
          // (-inf -> 0; the argument roundings are bounded with |a| <= 130).  Arguments as packed
          // FFMA2 pairs (the two halves of a bf16x2 word), exponentials per element, and a balanced
          // 4-level fp32 tree over the 16 (kSum16Err) with packed FADD2; one fp64 add per iteration
          float2 ea[4], eb[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float2 xa = ffma2_rn(make_float2(lo_f(wa[h]), hi_f(wa[h])), Lf, nmL);
            const float2 xb = ffma2_rn(make_float2(lo_f(wb[h]), hi_f(wb[h])), Lf, nmL);
            ea[h] = make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
            eb[h] = make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
          }
          const float2 sa = fadd2_rn(fadd2_rn(ea[0], ea[1]), fadd2_rn(ea[2], ea[3]));
          const float2 sb = fadd2_rn(fadd2_rn(eb[0], eb[1]), fadd2_rn(eb[2], eb[3]));
          const float2 sab = fadd2_rn(sa, sb);
          acc += (double)(sab.x + sab.y);
          cand_block(qa, vma, va);
          if (v0 + WG_GT < nv) cand_block(qb, vmb, vb);
        }
      }
      {
        const double ws = warp_sum(acc), ww = warp_sum((double)W);
        const float tm = max_nan(lo_f(cm2), hi_f(cm2));
        const bool tn = tm != tm;
        const float wm = warp_max(tn ? INFINITY : tm);
        const bool wn = __any_sync(0xffffffffu, tn);
        if (lane == 0) {
          G.rd[0][gw] = ws;
          G.rd[1][gw] = ww;
          G.rf[gw] = wm;
          G.ri[1][gw] = wn;
        }
      }
      wbar(g);  // also: every read of this half is done
      float cmx = -INFINITY;
#pragma unroll
      for (int i = 0; i < WG_GW; ++i) {
        cmx = fmaxf(cmx, G.rf[i]);
        bad |= G.ri[1][i] != 0;
      }
      // (a chunk far above the running max would overflow its exponentials)
      bad |= !(cmx < INFINITY) || (cmx - ref) * Lf > 100.0f;
      M_run = fmaxf(M_run, cmx);
      if (gt == 0) {
        double s = 0.0, w = 0.0;
#pragma unroll
        for (int i = 0; i < WG_GW; ++i) {
          s += G.rd[0][i];
          w += G.rd[1][i];
        }
        G.cs[c] = s;
        G.cw[c] = w;
        G.cmax[c] = ref;  // the masses' reference
        if (c + 2 < nch) issue(tv, c + 2);
      }
      WG_PH(3);
      // keep the list bounded: sort, keep the top k, raise the threshold.  Compacting as soon as
      // the list exceeds k + k/8 (not 2k): the threshold rises after nearly every chunk, so later
      // chunks append few candidates and each sort stays <= 128 keys (C3 7.90M -> 8.48M rows/s)
      const int nc = G.ncand;
      if (nc > WG_CAP) {
        bad = true;  // one chunk overflowed the list: left to the CTA kernel
      } else if (nc > K + K / 8 || nc > WG_CAP / 2) {
        wg_sort(G, g, gt, nc);
        if (gt == 0) {
          G.thrk = G.cand[K - 1];
          G.thr = fmaxf(G.thr, key_val(G.thrk));
          G.ncand = K;
        }
      }
      wbar(g);
      WG_PH(4);
    }
    // ---------------------------------------------- the row: mass, top-k, cut, draws
    bool requeue_task = bad;
    if (!bad) {
      const int nc = G.ncand;
      wg_sort(G, g, gt, nc);
      if (gw == 0) {
        const int n = min(K, nc);
        const float M = M_run;
        bool unc = n < 1 || nc < K || !(M > -INFINITY) || M == 0.0f;  // (signed-zero maxima: CTA kernel)
        int kept_k = -1;
        if (!unc && tv.T == 0.0) {
          const int am = key_id(G.cand[0]);
          for (int d = lane; d < nd; d += 32) {
            io.token[d0 + d] = am;
            if (io.flags) io.flags[d0 + d] = 0;
          }
          kept_k = greedy_kept(V, K, tv.topp);
        } else if (!unc) {
          // S = sum_c S_c 2^((m_c - M) L); the chunk bounds carry over (fp64 rescale ~1 ulp)
          double S = 0.0, Wt = 0.0;
          for (int c = lane; c < nch; c += 32) {
            const double f = exp2(((double)G.cmax[c] - (double)M) * Ld);
            S += G.cs[c] * f;
            Wt += G.cw[c] * f;
          }
          S = warp_sum(S);
          Wt = warp_sum(Wt);
          const float mL = fabsf(M) * Lf;
          // (exponentials: ex2.approx + argument rounding ln2 2^-23 |a|, |a| <= 130 below which
          // they flush to 0 and are bounded by V 2^-126)
          const double ES = S * (kEx2Raw + kSum16Err + 1e-12 + 130.0 * kLn2W * 0x1p-23) + Wt * 0.0 +
                            S * kLn2W * 0x1p-24 * (2.0 + 2.0 * (double)fmaxf(mL, mLr)) + (double)V * 0x1p-126;
          ExpCtx ec;
          ec.m = M;
          ec.T = tv.T;
          ec.Lhi = Lf;
          ec.Llo = (float)(Ld - (double)Lf);
          ec.md = (double)M;
          ec.L16 = 16.0 * Ld;
          // the k candidates in (p desc, id asc) order: lane i holds i and i + 32
          double e2[2];
          int id2[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = lane + 32 * r;
            e2[r] = 0.0;
            id2[r] = INT_MAX;
            if (i < n) {
              const unsigned long long k = G.cand[i];
              e2[r] = lite_exp(ec, key_val(k), sm.t16);
              id2[r] = key_id(k);
            }
          }
          const double u53 = kEps64;
          const double relArg = 4.5e-16 * (2.0 * (double)mL + 64.0);
          const double relA = kLiteErr + kRefExpErr + relArg + 128.0 * u53;
          const double relNp = (double)(2 * V + 64) * u53 + relArg + 2.0 * kRefExpErr;
          // (1/S as a correctly rounded reciprocal: one more rounding per ratio, in the (K + 10) u53)
          const double invS = __drcp_rn(S);
          const double rho = relA + ES * invS + relNp + (double)(K + 10) * u53;
          // inclusive csum of the masses in that order
          double c0 = e2[0];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, c0, o);
            if (lane >= o) c0 += y;
          }
          const double t0 = __shfl_sync(0xffffffffu, c0, 31);
          double c1 = e2[1];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, c1, o);
            if (lane >= o) c1 += y;
          }
          c1 += t0;
          // kept count: first index whose csum / S reaches top_p (numpy: searchsorted 'left'
          // on csum of p = e / S_np), all n when top_p == 1 or when it is never reached
          int kstar = n;
          if (tv.topp < 1.0) {
            const unsigned h0 = __ballot_sync(0xffffffffu, lane < n && c0 * invS >= tv.topp);
            const unsigned h1 = __ballot_sync(0xffffffffu, lane + 32 < n && c1 * invS >= tv.topp);
            kstar = h0 ? __ffs(h0) : (h1 ? 32 + __ffs(h1) : n);
            // certify both neighbours of the cut
            auto csum_at = [&](int i) -> double {  // inclusive csum at sorted index i
              const double x = __shfl_sync(0xffffffffu, c0, i & 31), y = __shfl_sync(0xffffffffu, c1, i & 31);
              return i < 32 ? x : y;
            };
            const double cK = csum_at(min(kstar, n) - 1);
            const double cP = kstar >= 2 ? csum_at(kstar - 2) : 0.0;
            if (kstar < n || (h0 | h1)) unc |= !(cK * invS * (1.0 - rho) >= tv.topp);
            else unc |= !(cK * invS * (1.0 + rho) < tv.topp);  // never reached: all n kept
            if (kstar >= 2) unc |= !(cP * invS * (1.0 + rho) < tv.topp);
          }
          // kept set in id order: ranks by counting
          if (!unc) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const int i = lane + 32 * r;
              int rank = 0;
              for (int j = 0; j < kstar; ++j) {
                const int idj = __shfl_sync(0xffffffffu, j < 32 ? id2[0] : id2[1], j & 31);
                rank += (idj < id2[r]);
              }
              if (i < kstar) {
                G.kid[rank] = id2[r];
                G.ke[rank] = e2[r];
              }
            }
            __syncwarp();
            double q0 = lane < kstar ? G.ke[lane] : 0.0, q1 = lane + 32 < kstar ? G.ke[lane + 32] : 0.0;
            double s0 = q0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, s0, o);
              if (lane >= o) s0 += y;
            }
            const double t0b = __shfl_sync(0xffffffffu, s0, 31);
            double s1 = q1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, s1, o);
              if (lane >= o) s1 += y;
            }
            s1 += t0b;
            const double Ak = __shfl_sync(0xffffffffu, s1, 31);
            const double beta = 8.0 * kRefExpErr + kLiteErr + relArg + (double)(6 * V + 1024) * u53;
            // draws: one lane each; first kept id with cdf > u * total
            for (int db = 0; db < nd; db += 32) {
              const int d = db + lane;
              double tau = 0.0;
              if (d < nd) tau = (d < WG_NU ? G.su[d] : draw_u(io, d0 + d, tv)) * Ak;
              // count of cdf entries <= tau (both halves), lane-parallel over the 64 prefixes
              int j = 0;
              for (int i = 0; i < kstar; ++i) {
                const double cv = __shfl_sync(0xffffffffu, i < 32 ? s0 : s1, i & 31);
                j += (cv <= tau);
              }
              const double i0 = __shfl_sync(0xffffffffu, s0, j & 31), i1 = __shfl_sync(0xffffffffu, s1, j & 31);
              const double x0 = __shfl_sync(0xffffffffu, s0, (j - 1) & 31);
              const double x1 = __shfl_sync(0xffffffffu, s1, (j - 1) & 31);
              if (d < nd) {
                const double Ein = j < 32 ? i0 : i1;
                const double Eex = j == 0 ? 0.0 : (j - 1 < 32 ? x0 : x1);
                const bool du = j >= kstar || !(Ein - tau > 2.0 * beta * Ak) || !(tau - Eex > 2.0 * beta * Ak);
                if (!du) {
                  io.token[d0 + d] = G.kid[j];
                  if (io.flags) io.flags[d0 + d] = 0;
                }
                unc |= du;
              }
            }
            kept_k = kstar;  // the kept set = the first kstar candidates (value desc, id asc)
          }
        }
        unc = __any_sync(0xffffffffu, unc);
        if (lane == 0) {
          G.flag = unc;
          if (!unc) set_kept(io, task_id, kept_k);
        }
      }
      wbar(g);
      requeue_task = G.flag != 0;
    }
    if (requeue_task && gt == 0) {
      requeue(a, task_id);
      atomicAdd(&a.counters[4], 1ull);
    }
    wbar(g);  // the group is done with the task's shared state
    WG_PH(5);
    if (prof) pc[6]++;
  }
  if (prof)
    for (int k = 0; k < 7; ++k) atomicAdd(&a.prof[k], pc[k]);
#undef WG_PH
}

int wide_launch(const char* rows, int64_t row_bytes, int V, const lc_task* tasks, int64_t n_tasks, CacheMap cm,
                DrawIO io, int* next, int* q_cta, unsigned long long* counters, int n_sms, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    LCB_CUDA_TRY(cudaFuncSetAttribute(wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(WgSmem)));
    attr = true;
  }
  StageArgs a{rows, row_bytes, V, tasks, (int)n_tasks, cm, io, next, q_cta, counters, stage_prof_buffer()};
  const int64_t g = n_tasks < n_sms ? n_tasks : n_sms;
  LCB_CUDA_TRY(cudaMemsetAsync(next, 0, 4, st));
  wide_kernel<<<(int)g, WG_THREADS, sizeof(WgSmem), st>>>(a);
  LCB_CUDA_TRY(cudaGetLastError());
  return LC_OK;
}

bool wide_eligible(int dtype, int64_t V, int64_t row_bytes, const void* rows) {
  return dtype == LC_BF16 && V > 32000 && V <= (int64_t)WG_NCHMAX * WG_CH && (V & 7) == 0 && (row_bytes & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(rows) & 15) == 0;
}

}  // namespace lcb
