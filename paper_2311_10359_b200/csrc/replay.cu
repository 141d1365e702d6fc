// Gap filling (Algorithm 1 + Algorithm 2), runtime feedback
// and the batch replay (Case B) -- one warp per gap / scenario.
//
// The LP pool of a warp lives in shared memory (predicted duration q = SK of the
// request's row, and a meta byte: level | alive | eligible).  BestPrioFit is a
// warp-parallel argmin of the strict total order (level asc, q desc, index asc)
// over alive eligible requests with q <= R (readings R14-R16): each lane scans
// its strided slice, then a 5-step shuffle reduction.  All time arithmetic is
// u64 and warp-uniform, so the replay is bit-exact with the serial definition.
#include <cuda_runtime.h>

#include "fikit_internal.cuh"

namespace fikit {

constexpr int kReplayWarps = 4;      // warps (scenarios) per CTA
constexpr uint32_t kPoolMax = 1024;  // LP requests per scenario held in shared memory
constexpr uint8_t kAlive = 0x10, kElig = 0x20;

struct Cand {
  uint32_t lk;  // level << 27 | index  (smaller = better at equal q)
  uint64_t q;
};

__device__ __forceinline__ bool better(uint32_t lka, uint64_t qa, uint32_t lkb, uint64_t qb) {
  uint32_t la = lka >> 27, lb = lkb >> 27;
  if (la != lb) return la < lb;
  if (qa != qb) return qa > qb;
  return lka < lkb;
}

// Algorithm 2 (BestPrioFit): index of the best fitting request, or -1 (uniform).
__device__ __forceinline__ int warp_best_prio_fit(const uint64_t* q, const uint8_t* meta, uint32_t m, uint64_t R,
                                                  int lane) {
  uint32_t blk = 0xFFFFFFFFu;
  uint64_t bq = 0;
  for (uint32_t k = lane; k < m; k += 32) {
    uint8_t mt = meta[k];
    uint64_t qk = q[k];
    if ((mt & (kAlive | kElig)) == (kAlive | kElig) && qk <= R) {
      uint32_t lk = ((uint32_t)(mt & 0xF) << 27) | k;
      if (blk == 0xFFFFFFFFu || better(lk, qk, blk, bq)) {
        blk = lk;
        bq = qk;
      }
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    uint32_t olk = __shfl_xor_sync(0xffffffffu, blk, off);
    uint64_t oq = __shfl_xor_sync(0xffffffffu, bq, off);
    if (olk != 0xFFFFFFFFu && (blk == 0xFFFFFFFFu || better(olk, oq, blk, bq))) {
      blk = olk;
      bq = oq;
    }
  }
  return blk == 0xFFFFFFFFu ? -1 : (int)(blk & 0x7FFFFFFu);
}

// load a pool into shared memory; returns false (and flags) on an invalid level
__device__ __forceinline__ bool load_pool(const fikit_table_t& tab, uint32_t K, const uint32_t* __restrict__ row,
                                          const uint8_t* __restrict__ level, uint64_t off, uint32_t m, uint64_t* q,
                                          uint8_t* meta, int lane, fikit_status_t* st) {
  bool ok = true;
  for (uint32_t k = lane; k < m; k += 32) {
    uint32_t r = __ldg(row + off + k);
    uint8_t L = __ldg(level + off + k);
    if (L < 1 || L > 9) {
      flag_record(st, off + k);
      ok = false;
    }
    bool el = r < K && __ldg(tab.sums + (size_t)r * 4) > 0;  // R16: no SK profile -> never a fill
    q[k] = el ? __ldg(tab.mean + (size_t)r * 2) : 0;          // SK of the request's ID
    meta[k] = (uint8_t)((L & 0xF) | kAlive | (el ? kElig : 0));
  }
  __syncwarp();
  return __all_sync(0xffffffffu, ok);
}

// smallest predicted duration among alive eligible requests (UINT64_MAX if none):
// a gap with R < qmin has no candidate, so BestPrioFit's scan is skipped
__device__ __forceinline__ uint64_t warp_min_q(const uint64_t* q, const uint8_t* meta, uint32_t m, int lane) {
  uint64_t mn = ~0ull;
  for (uint32_t k = lane; k < m; k += 32)
    if ((meta[k] & (kAlive | kElig)) == (kAlive | kElig)) mn = min(mn, q[k]);
#pragma unroll
  for (int off = 16; off; off >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  return mn;
}

// ---- sorted pool (fast path) --------------------------------------------------------------
// When every eligible q < 2^50 and m <= 1024, the pool is sorted once per scenario by the
// composite key  level << 60 | (2^50 - 1 - q) << 10 | index  (ineligible: ~0).  Sorted
// order is exactly BestPrioFit's preference order (level asc, q desc, index asc), and since
// the remaining idle time R only shrinks, BestPrioFit(R) = the first alive position whose
// q <= R: a ballot per 32 positions instead of a full argmin.  Lane c holds the alive bits
// of sorted positions [32c, 32c + 32).
constexpr uint64_t kQ50 = (1ull << 50) - 1;

__device__ __forceinline__ uint64_t key_q(uint64_t key) { return kQ50 - ((key >> 10) & kQ50); }

__device__ void warp_bitonic_sort(uint64_t* K, uint32_t P, int lane) {
  for (uint32_t k = 2; k <= P; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = lane; t < P / 2; t += 32) {
        const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const uint32_t l = i + j;
        const uint64_t a = K[i], b = K[l];
        const bool asc = (i & k) == 0;
        if ((a > b) == asc) {
          K[i] = b;
          K[l] = a;
        }
      }
      __syncwarp();
    }
}

// Build the sorted pool in place of q (q[k] by index -> K[p] by sorted position).
// Returns false (pool left by index) if the fast path does not apply.
__device__ __forceinline__ bool make_sorted_pool(uint64_t* q, const uint8_t* meta, uint32_t m, int lane,
                                                 uint32_t& A, uint32_t& nch) {
  bool ok = true;
  for (uint32_t k = lane; k < m; k += 32)
    if ((meta[k] & kElig) && q[k] > kQ50) ok = false;
  if (!__all_sync(0xffffffffu, ok) || m > 1024u) return false;
  uint32_t P = 32;
  while (P < m) P <<= 1;
  for (uint32_t k = lane; k < P; k += 32) {
    uint64_t key = ~0ull;
    if (k < m && (meta[k] & kElig)) key = ((uint64_t)(meta[k] & 0xF) << 60) | ((kQ50 - q[k]) << 10) | k;
    q[k] = key;
  }
  __syncwarp();
  warp_bitonic_sort(q, P, lane);
  nch = (m + 31) / 32;
  A = 0;
  for (uint32_t c = 0; c < nch; c++) {
    const uint32_t p = c * 32 + lane;
    const uint32_t b = __ballot_sync(0xffffffffu, p < m && q[p] != ~0ull);
    if (lane == (int)c) A = b;
  }
  return true;
}

// first alive sorted position with q <= R, or -1 (uniform)
__device__ __forceinline__ int sorted_best(const uint64_t* K, uint32_t A, uint32_t nch, uint64_t R, int lane) {
  for (uint32_t c = 0; c < nch; c++) {
    const uint32_t word = __shfl_sync(0xffffffffu, A, c);
    if (!word) continue;
    const bool fit = ((word >> lane) & 1u) && key_q(K[c * 32 + lane]) <= R;
    const uint32_t b = __ballot_sync(0xffffffffu, fit);
    if (b) return (int)(c * 32 + __ffs(b) - 1);
  }
  return -1;
}

__device__ __forceinline__ uint64_t sorted_min_q(const uint64_t* K, uint32_t A, uint32_t nch, int lane) {
  uint64_t mn = ~0ull;
  for (uint32_t c = 0; c < nch; c++) {
    const uint32_t word = __shfl_sync(0xffffffffu, A, c);
    if ((word >> lane) & 1u) mn = min(mn, key_q(K[c * 32 + lane]));
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  return mn;
}

// One BestPrioFit pick (Alg. 2) on either representation: returns the request index (or -1)
// and its q; dequeues it (alive bit cleared in both views).
__device__ __forceinline__ int pool_pick(bool fast, uint64_t* q, uint8_t* meta, uint32_t m, uint32_t& A,
                                         uint32_t nch, uint64_t R, int lane, uint64_t& qk) {
  int k;
  if (fast) {
    const int p = sorted_best(q, A, nch, R, lane);
    if (p < 0) return -1;
    const uint64_t key = q[p];
    k = (int)(key & 1023u);
    qk = key_q(key);
    if (lane == (p >> 5)) A &= ~(1u << (p & 31));
  } else {
    k = warp_best_prio_fit(q, meta, m, R, lane);
    if (k < 0) return -1;
    qk = q[k];
  }
  if (lane == 0) meta[k] &= (uint8_t)~kAlive;
  __syncwarp();
  return k;
}

__device__ __forceinline__ uint64_t pool_min_q(bool fast, const uint64_t* q, const uint8_t* meta, uint32_t m,
                                               uint32_t A, uint32_t nch, int lane) {
  return fast ? sorted_min_q(q, A, nch, lane) : warp_min_q(q, meta, m, lane);
}

__device__ __forceinline__ uint64_t digest_term(uint32_t k, int32_t fg, uint64_t start) {
  return mix64((uint64_t)k ^ ((uint64_t)(uint32_t)(fg + 1) << 32) ^ mix64(start));
}

// ---- fikit_fill: G independent gaps ----------------------------------------------------------
__global__ void __launch_bounds__(kReplayWarps * 32)
    k_fill(fikit_table_t tab, const uint64_t* __restrict__ R0, const uint64_t* __restrict__ deadline,
           const uint32_t* __restrict__ pool_row, const uint64_t* __restrict__ pool_dur,
           const uint8_t* __restrict__ pool_level, const uint32_t* __restrict__ pool_off,
           const uint32_t* __restrict__ pool_len, uint32_t G, fikit_fill_params_t prm, uint32_t* __restrict__ picks,
           const uint32_t* __restrict__ picks_off, uint32_t* __restrict__ n_picks, uint64_t* __restrict__ R_left,
           uint64_t* __restrict__ t_used, fikit_status_t* st) {
  __shared__ uint64_t s_q[kReplayWarps][kPoolMax];
  __shared__ uint8_t s_meta[kReplayWarps][kPoolMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  for (uint32_t g = blockIdx.x * kReplayWarps + w; g < G; g += gridDim.x * kReplayWarps) {
    uint32_t m = pool_len[g], off = pool_off[g];
    uint64_t* q = s_q[w];
    uint8_t* meta = s_meta[w];
    __syncwarp();
    if (m > kPoolMax) {
      if (lane == 0) atomicOr(&st->flags, kStatusArg);
      continue;
    }
    if (!load_pool(tab, K, pool_row, pool_level, off, m, q, meta, lane, st)) continue;
    uint64_t R = R0[g], t = 0, dl = deadline[g];
    uint32_t np = 0, po = picks_off[g];
    if (R >= prm.threshold_ns) {  // Alg. 1 lines 6-8
      uint32_t A = 0, nch = 0;
      const bool fast = make_sorted_pool(q, meta, m, lane, A, nch);
      uint64_t qmin = pool_min_q(fast, q, meta, m, A, nch, lane);
      for (;;) {                             // lines 9-16
        if (prm.feedback && t >= dl) break;  // early stop on the HP launch
        if (R < qmin) break;                 // nothing can fit
        uint64_t qk;
        const int k = pool_pick(fast, q, meta, m, A, nch, R, lane, qk);  // Alg. 2
        if (k < 0) break;
        if (lane == 0) picks[po + np] = (uint32_t)k;
        np++;
        t += __ldg(pool_dur + off + k);  // launched (line 14)
        R -= qk;                           // revised by the predicted duration (line 15, R17)
        if (qk == qmin) qmin = pool_min_q(fast, q, meta, m, A, nch, lane);
      }
    }
    if (lane == 0) {
      n_picks[g] = np;
      R_left[g] = R;
      t_used[g] = t;
    }
  }
}

// ---- fikit_simulate_batch: one warp per scenario ------------------------------------------------
__global__ void __launch_bounds__(kReplayWarps * 32)
    k_simulate(fikit_table_t tab, const uint32_t* __restrict__ hp_row, const uint64_t* __restrict__ hp_dur,
               const uint64_t* __restrict__ hp_gap, const uint32_t* __restrict__ lp_row,
               const uint64_t* __restrict__ lp_dur, const uint8_t* __restrict__ lp_level,
               const fikit_scenario_t* __restrict__ sc, uint32_t S, fikit_fill_params_t prm,
               fikit_result_t* __restrict__ out, int32_t* __restrict__ fill_gap, uint64_t* __restrict__ lp_start,
               const uint64_t* __restrict__ sched_off, fikit_status_t* st) {
  __shared__ uint64_t s_q[kReplayWarps][kPoolMax];
  __shared__ uint8_t s_meta[kReplayWarps][kPoolMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  const bool sched = fill_gap != nullptr && lp_start != nullptr && sched_off != nullptr;
  for (uint32_t s = blockIdx.x * kReplayWarps + w; s < S; s += gridDim.x * kReplayWarps) {
    fikit_scenario_t c = sc[s];
    uint32_t m = c.lp_len, nh = c.hp_len;
    uint64_t* q = s_q[w];
    uint8_t* meta = s_meta[w];
    __syncwarp();
    if (m > kPoolMax) {
      if (lane == 0) atomicOr(&st->flags, kStatusArg);
      continue;
    }
    if (!load_pool(tab, K, lp_row, lp_level, c.lp_off, m, q, meta, lane, st)) continue;
    const uint64_t so = sched ? sched_off[s] : 0;
    const uint64_t scale = c.gap_scale_q16;
    uint32_t A = 0, nch = 0;
    const bool fast = make_sorted_pool(q, meta, m, lane, A, nch);
    uint64_t qmin = pool_min_q(fast, q, meta, m, A, nch, lane);
    uint64_t t = 0, hp_delay = 0, fill_work = 0, lp_end = 0, dig = 0;
    uint32_t n_fills = 0;
    // t = start of the next HP kernel.  Without a fill, kernel i+1 starts at
    // T_i + d_i + a'_i; only gaps whose gate can open (p >= tau, p >= qmin, and
    // with feedback a' > 0) need the serial Alg. 1 loop, so each chunk of 32 HP
    // kernels is advanced by a prefix sum and visits just its open gates.
    for (uint32_t base = 0; base < nh; base += 32) {
      uint32_t i_l = base + lane;
      uint64_t d_l = 0, a_l = 0, p_l = 0;
      bool valid = i_l < nh, last = i_l == nh - 1;
      if (valid) {
        d_l = __ldg(hp_dur + c.hp_off + i_l);
        a_l = last ? 0 : (__ldg(hp_gap + c.hp_off + i_l) * scale) >> 16;  // R24; no gap after the last
        uint32_t r = __ldg(hp_row + c.hp_off + i_l);
        p_l = r < K ? ((__ldg(tab.mean + (size_t)r * 2 + 1) * scale) >> 16) : 0;  // SG (Alg.1 3-5, R12)
      }
      const uint64_t x_l = d_l + a_l;
      uint64_t X = x_l;  // inclusive prefix over the chunk
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, X, dd);
        if (lane >= dd) X += y;
      }
      const bool gate = valid && !last && p_l >= prm.threshold_ns && p_l >= qmin && (!prm.feedback || a_l > 0);
      uint32_t gmask = __ballot_sync(0xffffffffu, gate);
      const uint64_t T0 = t;
      uint64_t shift = 0;  // delays imposed by fills earlier in this chunk
      while (gmask) {
        const int j = __ffs(gmask) - 1;
        gmask &= gmask - 1;
        const uint32_t i = base + j;
        const uint64_t Xj = __shfl_sync(0xffffffffu, X, j);
        const uint64_t a = __shfl_sync(0xffffffffu, a_l, j);
        const uint64_t p = __shfl_sync(0xffffffffu, p_l, j);
        t = T0 + shift + Xj - a;  // end of HP kernel i
        const uint64_t r = t + a;   // the HP client's next launch arrives (R20)
        uint64_t R = p;
        for (;;) {
          if (prm.feedback && t >= r) break;
          if (R < qmin) break;  // no alive eligible request fits: BestPrioFit returns none
          uint64_t qk;
          const int k = pool_pick(fast, q, meta, m, A, nch, R, lane, qk);  // Alg. 2
          if (k < 0) break;
          const uint64_t e = __ldg(lp_dur + c.lp_off + k);
          if (lane == 0) {
            if (sched) {
              fill_gap[so + k] = (int32_t)i;
              lp_start[so + k] = t;
            }
            dig += digest_term((uint32_t)k, (int32_t)i, t);
          }
          R -= qk;
          t += e;
          if (qk == qmin) qmin = pool_min_q(fast, q, meta, m, A, nch, lane);
          fill_work += e;
          n_fills++;
          lp_end = max(lp_end, t);
        }
        if (t > r) {  // overhead 2: kernel i+1 starts at max(t, r_{i+1})
          hp_delay += t - r;
          shift += t - r;
        }
      }
      t = T0 + shift + __shfl_sync(0xffffffffu, X, 31);  // next kernel's start (or the HP end)
    }
    const uint64_t hp_jct = t;
    // tail: remaining requests in Q1..Q9 order, FIFO within a queue (R22)
    uint32_t n_tail = 0;
    for (uint32_t L = 1; L <= 9; L++) {
      for (uint32_t b = 0; b < m; b += 32) {
        uint32_t k = b + lane;
        bool sel = k < m && (meta[k] & kAlive) && (meta[k] & 0xF) == L;
        uint32_t bal = __ballot_sync(0xffffffffu, sel);
        if (!bal) continue;
        uint64_t e = sel ? __ldg(lp_dur + c.lp_off + k) : 0;
        uint64_t x = e;  // inclusive scan
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          uint64_t y = __shfl_up_sync(0xffffffffu, x, dd);
          if (lane >= dd) x += y;
        }
        if (sel) {
          uint64_t start = t + x - e;
          if (sched) {
            fill_gap[so + k] = -1;
            lp_start[so + k] = start;
          }
          dig += digest_term(k, -1, start);
        }
        t += __shfl_sync(0xffffffffu, x, 31);
        n_tail += __popc(bal);
      }
    }
    if (n_tail) lp_end = max(lp_end, t);
#pragma unroll
    for (int off = 16; off; off >>= 1) dig += __shfl_xor_sync(0xffffffffu, dig, off);
    if (lane == 0) {
      fikit_result_t o;
      o.hp_jct = hp_jct;
      o.lp_jct = m ? lp_end : 0;
      o.hp_delay = hp_delay;
      o.fill_work = fill_work;
      o.digest = dig;
      o.n_fills = n_fills;
      o.n_tail = n_tail;
      out[s] = o;
    }
  }
}

}  // namespace fikit
