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

constexpr int kReplayWarps = kSimThreads / 32;  // warps (scenarios) per CTA
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

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t a) {
  const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(a >> 32));
  const uint32_t lo = __reduce_max_sync(0xffffffffu, (uint32_t)(a >> 32) == hi ? (uint32_t)a : 0u);
  return ((uint64_t)hi << 32) | lo;
}

// warp minimum of a u64 (all lanes): REDUX on the high words, then on the low words of the
// lanes holding the minimal high word
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t a) {
  const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(a >> 32));
  const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(a >> 32) == hi ? (uint32_t)a : 0xFFFFFFFFu);
  return ((uint64_t)hi << 32) | lo;
}


__device__ __forceinline__ uint64_t key_q(uint64_t key) { return kQ50 - ((key >> 10) & kQ50); }

// Warp bitonic sort of P (power of two, >= 32) keys in shared memory.  Consecutive stages j and
// j/2 of one merge are fused: each thread loads a group of 4 keys {b, b+h, b+j, b+j+h} (h = j/2),
// does both compare-exchange rounds in registers and stores them (half the shared-memory
// round trips and warp syncs of one stage at a time).
__device__ void warp_bitonic_sort(uint64_t* K, uint32_t P, int lane) {
  auto cx = [](uint64_t& a, uint64_t& b, bool asc) {
    if ((a > b) == asc) {
      const uint64_t x = a;
      a = b;
      b = x;
    }
  };
  for (uint32_t k = 2; k <= P; k <<= 1) {
    uint32_t j = k >> 1;
    while (j > 0) {
      if (j >= 2) {
        const uint32_t h = j >> 1;
        for (uint32_t t = lane; t < P / 4; t += 32) {
          const uint32_t b = ((t & ~(h - 1)) << 2) | (t & (h - 1));
          const bool asc = (b & k) == 0;
          uint64_t a0 = K[b], a1 = K[b + h], a2 = K[b + j], a3 = K[b + j + h];
          cx(a0, a2, asc);
          cx(a1, a3, asc);
          cx(a0, a1, asc);
          cx(a2, a3, asc);
          K[b] = a0;
          K[b + h] = a1;
          K[b + j] = a2;
          K[b + j + h] = a3;
        }
        j >>= 2;
      } else {
        for (uint32_t t = lane; t < P / 2; t += 32) {
          const uint32_t i = t << 1;
          const bool asc = (i & k) == 0;
          uint64_t a = K[i], b = K[i + 1];
          cx(a, b, asc);
          K[i] = a;
          K[i + 1] = b;
        }
        j = 0;
      }
      __syncwarp();
    }
  }
}

// Build the sorted pool in place of q (q[k] by index -> K[p] by sorted position).
// Returns false (pool left by index) if the fast path does not apply.
// epack: every eligible request's duration e < 2^22 ns, so the sorted entry carries it too
// (q << 32 | e << 10 | index): a pick reads q, e and the index in one shared load instead of
// waiting on a global load of e.
__device__ __forceinline__ bool make_sorted_pool(uint64_t* q, const uint8_t* meta, uint32_t m, int lane,
                                                 uint32_t& A, uint32_t& nch, uint32_t& CM,
                                                 const uint64_t* __restrict__ dur, bool& epack) {
  bool ok = true, small = true;
  for (uint32_t k = lane; k < m; k += 32)
    if (meta[k] & kElig) {
      if (q[k] >= 0xFFFFFFFFull) ok = false;  // fast path: every q < 2^32 - 1
      if (__ldg(dur + k) >= (1ull << 22)) small = false;
    }
  epack = __all_sync(0xffffffffu, small);
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
  // sorted: the order is the position now; each entry becomes q << 32 | index (q = the high
  // word, one 32-bit load), dead / ineligible entries stay ~0
  for (uint32_t p = lane; p < P; p += 32) {
    const uint64_t key = q[p];
    if (key != ~0ull)
      q[p] = (key_q(key) << 32) | (epack ? (__ldg(dur + (key & 1023u)) << 10) : 0ull) | (key & 1023u);
  }
  __syncwarp();
  const uint32_t* qh = reinterpret_cast<const uint32_t*>(q) + 1;  // qh[2 p] = q at position p
  nch = (m + 31) / 32;
  A = 0;
  CM = 0xFFFFFFFFu;
  for (uint32_t c = 0; c < nch; c++) {
    const uint32_t p = c * 32 + lane;
    const bool alive = p < m && q[p] != ~0ull;
    const uint32_t b = __ballot_sync(0xffffffffu, alive);
    const uint32_t mn = __reduce_min_sync(0xffffffffu, alive ? qh[2 * p] : 0xFFFFFFFFu);
    if (lane == (int)c) {
      A = b;
      CM = mn;
    }
  }
  return true;
}

// chunk c's minimum q over its alive positions, after its alive word changed (to lane c)
__device__ __forceinline__ void chunk_min_refresh(const uint64_t* K, uint32_t A, uint32_t c, uint32_t& CM,
                                                  int lane) {
  const uint32_t word = __shfl_sync(0xffffffffu, A, c);
  const uint32_t* qh = reinterpret_cast<const uint32_t*>(K) + 1;
  const uint32_t mn = __reduce_min_sync(0xffffffffu, ((word >> lane) & 1u) ? qh[2 * (c * 32 + lane)] : 0xFFFFFFFFu);
  if (lane == (int)c) CM = mn;
}

// first alive sorted position with q <= R, or -1 (uniform): the first chunk whose alive minimum
// fits (one ballot over the chunk lanes), then the first fitting position inside it
__device__ __forceinline__ int sorted_best(const uint64_t* K, uint32_t A, uint32_t CM, uint32_t nch, uint64_t R,
                                           int lane) {
  // every q <= 2^32 - 2, so q <= R iff q <= min(R, 2^32 - 2); an empty chunk's minimum
  // 0xFFFFFFFF then never passes the chunk ballot
  const uint32_t Rc = R >= 0xFFFFFFFFull ? 0xFFFFFFFEu : (uint32_t)R;
  const uint32_t cb = __ballot_sync(0xffffffffu, (uint32_t)lane < nch && CM <= Rc);
  FK_CHECK(cb != 0u);  // (the caller's R >= qmin, the exact pool minimum, guarantees a fit)
  const uint32_t c = __ffs(cb) - 1;
  const uint32_t word = __shfl_sync(0xffffffffu, A, c);
  const uint32_t* qh = reinterpret_cast<const uint32_t*>(K) + 1;
  const bool fit = ((word >> lane) & 1u) && qh[2 * (c * 32 + lane)] <= Rc;
  const uint32_t b = __ballot_sync(0xffffffffu, fit);  // != 0: the chunk's minimum fits
  return (int)(c * 32 + __ffs(b) - 1);
}

__device__ __forceinline__ uint64_t sorted_min_q(uint32_t CM, uint32_t nch, int lane) {
  const uint32_t v = __reduce_min_sync(0xffffffffu, (uint32_t)lane < nch ? CM : 0xFFFFFFFFu);
  return v == 0xFFFFFFFFu ? ~0ull : (uint64_t)v;
}

// One BestPrioFit pick (Alg. 2) on either representation: returns the request index (or -1)
// and its q; dequeues it (alive bit cleared in both views).
// ek: the pick's actual duration, its global load issued as soon as the index is known (the
// dequeue bookkeeping below overlaps its latency)
__device__ __forceinline__ bool qk_fits(uint64_t q, uint64_t R) { return q <= R; }  // (FK_CHECK: R14)
__device__ __forceinline__ int pool_pick(bool fast, uint64_t* q, uint8_t* meta, uint32_t m, uint32_t& A,
                                         uint32_t& CM, uint32_t nch, uint64_t R, int lane, uint64_t& qk,
                                         const uint64_t* __restrict__ dur, uint64_t& ek, bool epack = false) {
  int k;
  if (fast) {
    const int p = sorted_best(q, A, CM, nch, R, lane);  // (always a fit: see sorted_best)
    const uint64_t x = q[p];  // q << 32 | [e << 10 |] index
    k = (int)(x & 1023u);
    FK_CHECK((uint32_t)p < m && (uint32_t)k < m && qk_fits(x >> 32, R));
    ek = epack ? ((x >> 10) & 0x3FFFFFull) : __ldg(dur + k);
    qk = x >> 32;
    if (lane == (p >> 5)) A &= ~(1u << (p & 31));
    // the chunk's alive minimum changes only if the pick was it (a pick is the largest fitting q
    // of its level: usually not the minimum)
    if (__shfl_sync(0xffffffffu, CM, (uint32_t)p >> 5) == (uint32_t)qk) chunk_min_refresh(q, A, (uint32_t)p >> 5, CM, lane);
  } else {
    k = warp_best_prio_fit(q, meta, m, R, lane);
    if (k < 0) return -1;
    ek = __ldg(dur + k);
    qk = q[k];
    if (lane == 0) meta[k] &= (uint8_t)~kAlive;  // (the fast path's dequeues: sync_meta_alive)
    __syncwarp();
  }
  return k;
}

// after a sorted-pool replay: clear the alive bit (by index) of every request a fill dequeued
// (eligible positions whose bit in A is clear), once instead of one shared RMW per pick
__device__ __forceinline__ void sync_meta_alive(const uint64_t* q, uint8_t* meta, uint32_t A, uint32_t nch, int lane) {
  for (uint32_t c = 0; c < nch; c++) {
    const uint32_t word = __shfl_sync(0xffffffffu, A, c);
    const uint64_t x = q[c * 32 + lane];
    if (x != ~0ull && !((word >> lane) & 1u)) meta[x & 1023u] &= (uint8_t)~kAlive;
  }
  __syncwarp();
}

__device__ __forceinline__ uint64_t pool_min_q(bool fast, const uint64_t* q, const uint8_t* meta, uint32_t m,
                                               uint32_t CM, uint32_t nch, int lane) {
  return fast ? sorted_min_q(CM, nch, lane) : warp_min_q(q, meta, m, lane);
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
  pdl_entry();
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
      uint32_t CM;
      bool epack = false;
      const bool fast = make_sorted_pool(q, meta, m, lane, A, nch, CM, pool_dur + off, epack);
      uint64_t qmin = pool_min_q(fast, q, meta, m, CM, nch, lane);
      for (;;) {                             // lines 9-16
        if (prm.feedback && t >= dl) break;  // early stop on the HP launch
        if (R < qmin) break;                 // nothing can fit
        uint64_t qk, ek;
        const int k = pool_pick(fast, q, meta, m, A, CM, nch, R, lane, qk, pool_dur + off, ek, epack);  // Alg. 2
        if (k < 0) break;
        if (lane == 0) picks[po + np] = (uint32_t)k;
        np++;
        t += ek;  // launched (line 14)
        R -= qk;                           // revised by the predicted duration (line 15, R17)
        if (qk == qmin) qmin = pool_min_q(fast, q, meta, m, CM, nch, lane);
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
// Digest terms are batched: lane (n % 32) keeps the n-th fill's (k, gap, start) and every 32
// fills the warp evaluates 32 terms in one SIMT pass (the digest is a sum: order-free).
struct DigestBatch {
  uint32_t n = 0, k = 0;
  int32_t fg = 0;
  uint64_t start = 0, sum = 0;
  __device__ __forceinline__ void add(uint32_t kk, int32_t g, uint64_t t, int lane) {
    if (lane == (int)(n & 31u)) {
      k = kk;
      fg = g;
      start = t;
    }
    if ((++n & 31u) == 0) sum += digest_term(k, fg, start);
  }
  __device__ __forceinline__ void drain(int lane) {
    if (lane < (int)(n & 31u)) sum += digest_term(k, fg, start);
  }
};

// LP pool of at most 64 requests in registers, by request index: lane l holds requests l and
// 32 + l.  Requires every eligible q < 2^22 ns and every LP duration < 2^32 ns.
// BestPrioFit (Alg. 2) is one warp argmin: the strict total order (level asc, q desc, index asc)
// of R14-R16 is the order of the 32-bit key  level << 28 | (2^22 - 1 - q) << 6 | index, so the
// best fitting request is the REDUX minimum of the keys of the alive eligible requests with
// q <= R (no sort, no per-scenario setup beyond the loads).
constexpr uint32_t kQ22 = (1u << 22) - 1;
struct RegPool {
  static constexpr bool kOwnerStats = true;  // fill_work / n_fills from the owning lanes at the end
  // the order key and q << 6 | index of requests lane, 32 + lane (both 0xFFFFFFFF if not
  // eligible; a dequeue sets pq alone to 0xFFFFFFFF, which no Rc <= 0xFFFFFFFE admits):
  // q <= R <=> pq <= R << 6 | 63
  uint32_t key0, key1;
  uint32_t pq0, pq1;
  uint64_t elig;        // eligible requests by index (warp-uniform)
  uint32_t dur0, dur1;  // LP duration of requests lane, 32 + lane (< 2^32 ns)
  uint32_t lvl0, lvl1;  // level of requests lane, 32 + lane
  uint64_t alive;       // alive requests by index (warp-uniform)
  uint32_t ek;          // the last pick's duration

  // smallest alive eligible q, 0xFFFFFFFF if none
  __device__ __forceinline__ uint32_t min_q32() const {
    const uint32_t v = __reduce_min_sync(0xffffffffu, min(pq0, pq1));
    return v == 0xFFFFFFFFu ? v : v >> 6;
  }
  // Alg. 2: the best alive eligible request with q <= R, dequeued; returns its index.  The caller
  // guarantees one fits (R >= qmin, the exact smallest alive eligible q), so there is no "none"
  // branch here or after the call (3.7 % of the replay).
  // q <= R  <=>  q << 6 | k <= R << 6 | 63  (k < 64), and every q < 2^22 fits an R >= 2^22.
  __device__ __forceinline__ int pick32(uint32_t R, int lane, uint32_t& qk) {
    const uint32_t Rc = R >= (1u << 22) ? 0xFFFFFFFEu : (R << 6) | 63u;  // (a cleared pq never fits)
    const uint32_t c0 = pq0 <= Rc ? key0 : 0xFFFFFFFFu, c1 = pq1 <= Rc ? key1 : 0xFFFFFFFFu;
    const uint32_t best = __reduce_min_sync(0xffffffffu, min(c0, c1));
    FK_CHECK(best != 0xFFFFFFFFu);
    const uint32_t k = best & 63u;
    FK_CHECK((uint32_t)lane != (k & 31u) || (k < 32u ? pq0 : pq1) != 0xFFFFFFFFu);  // (alive when picked)
    qk = kQ22 - ((best >> 6) & kQ22);
    ek = __shfl_sync(0xffffffffu, k < 32u ? dur0 : dur1, (int)(k & 31u));
    if ((uint32_t)lane == (k & 31u)) {
      if (k < 32u) pq0 = 0xFFFFFFFFu; else pq1 = 0xFFFFFFFFu;  // (dequeued: only pq is cleared)
    }
    return (int)k;
  }
  __device__ __forceinline__ uint64_t dur_of(uint32_t) const { return ek; }  // (of the last pick)
  // the schedule of a filled request kk (gap, start): lane 0 logs it in the warp's shared slot
  // kk (one store, no per-lane selects); the owning lanes read it back for the digest at the end
  uint4* log;
  __device__ __forceinline__ void record(uint32_t kk, int32_t g, uint64_t t, int lane, DigestBatch&) {
    if (lane == 0) log[kk] = make_uint4((uint32_t)g, (uint32_t)t, (uint32_t)(t >> 32), 0u);
  }
  // the tail start of requests lane, 32 + lane (set by replay_tail_reg; fg = -1 there)
  int32_t fg0, fg1;
  uint64_t st0, st1;
  // requests dequeued by fills, by index
  __device__ __forceinline__ uint64_t picked_mask() const {
    const uint32_t lo = __ballot_sync(0xffffffffu, pq0 == 0xFFFFFFFFu);
    const uint32_t hi = __ballot_sync(0xffffffffu, pq1 == 0xFFFFFFFFu);
    return elig & (((uint64_t)hi << 32) | lo);
  }
};

// load a pool of m <= 64 requests into registers.  Returns 0 ok, 1 invalid level (flagged),
// 2 the register pool does not apply (some eligible q >= 2^22 or duration >= 2^32: pass 2).
__device__ __forceinline__ int load_reg_pool(const fikit_table_t& tab, uint32_t K, const uint32_t* __restrict__ row,
                                             const uint8_t* __restrict__ level, const uint64_t* __restrict__ dur,
                                             uint64_t off, uint32_t m, int lane, fikit_status_t* st, RegPool& P) {
  bool ok = true, small = true;
  auto one = [&](uint32_t kk, uint32_t& key, uint32_t& pq, uint32_t& d, uint32_t& lv) {
    key = pq = 0xFFFFFFFFu;
    d = 0;
    lv = 0;
    if (kk < m) {
      const uint32_t r = __ldg(row + off + kk);
      const uint32_t L = __ldg(level + off + kk);
      const uint64_t d64 = __ldg(dur + off + kk);
      if (d64 >> 32) small = false;
      d = (uint32_t)d64;
      lv = L;
      if (L < 1 || L > 9) {
        flag_record(st, off + kk);
        ok = false;
      }
      const bool el = r < K && __ldg(tab.sums + (size_t)r * 4) > 0;  // R16: no SK profile -> never a fill
      if (el) {
        const uint64_t q = __ldg(tab.mean + (size_t)r * 2);  // SK of the request's ID
        if (q > kQ22) small = false;
        const uint32_t q22 = (uint32_t)(q & kQ22);
        key = ((L & 0xFu) << 28) | ((kQ22 - q22) << 6) | kk;
        pq = (q22 << 6) | kk;
      }
    }
  };
  one((uint32_t)lane, P.key0, P.pq0, P.dur0, P.lvl0);
  one(32u + (uint32_t)lane, P.key1, P.pq1, P.dur1, P.lvl1);
  if (!__all_sync(0xffffffffu, ok)) return 1;
  if (!__all_sync(0xffffffffu, small)) return 2;
  P.elig = ((uint64_t)__ballot_sync(0xffffffffu, P.pq1 != 0xFFFFFFFFu) << 32) |
           __ballot_sync(0xffffffffu, P.pq0 != 0xFFFFFFFFu);
  P.alive = m >= 64 ? ~0ull : ((1ull << m) - 1);
  return 0;
}

// shared-memory pool (any m <= kPoolMax): the sorted fast path or the full argmin
struct SmemPool {
  static constexpr bool kOwnerStats = false;
  uint64_t* q;
  uint8_t* meta;
  const uint64_t* dur;  // lp_dur + lp_off
  uint32_t m, A, nch;
  bool fast;
  uint32_t CM;  // lane c: chunk c's alive minimum q (sorted fast path; q < 2^32 there)
  __device__ __forceinline__ uint64_t min_q(int lane) const { return pool_min_q(fast, q, meta, m, CM, nch, lane); }
  uint64_t ek;  // the last pick's duration (loaded by pool_pick)
  bool epack;   // durations packed into the sorted entries (make_sorted_pool)
  __device__ __forceinline__ int pick(uint64_t R, int lane, uint64_t& qk) {
    return pool_pick(fast, q, meta, m, A, CM, nch, R, lane, qk, dur, ek, epack);
  }
  __device__ __forceinline__ uint64_t dur_of(uint32_t) const { return ek; }  // (of the last pick)
  __device__ __forceinline__ void record(uint32_t kk, int32_t g, uint64_t t, int lane, DigestBatch& dig) {
    dig.add(kk, g, t, lane);
  }
};

// inclusive warp prefix sum of u64 values; 32-bit shuffles and adds when every value is
// < 2^27 (the sum of 32 then stays below 2^32), the common case for nanosecond chunk times
__device__ __forceinline__ uint64_t warp_inclusive_scan(uint64_t v, int lane) {
  if (__all_sync(0xffffffffu, v < (1ull << 27))) {
    uint32_t x = (uint32_t)v;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, dd);
      if (lane >= dd) x += y;
    }
    return x;
  }
  uint64_t x = v;
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, dd);
    if (lane >= dd) x += y;
  }
  return x;
}

// warp sum of u64 values (all lanes): one REDUX when every value is < 2^27 (the common case)
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
  if (__all_sync(0xffffffffu, v < (1ull << 27))) return __reduce_add_sync(0xffffffffu, (uint32_t)v);
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

struct HpOut {
  uint64_t t, hp_delay, fill_work, lp_end;
  uint32_t n_fills;
};

// The HP template with gap filling (Alg. 1 + Alg. 2 + feedback, Case B).  t = start of the next
// HP kernel.  Without a fill, kernel i+1 starts at T_i + d_i + a'_i; only gaps whose gate can
// open (p >= tau, p >= qmin, and with feedback a' > 0) need the serial Alg. 1 loop, so each
// chunk of 32 HP kernels is advanced by a prefix sum and visits just its open gates.  The next
// chunk's inputs are loaded while this one is processed.
// kLazyScan: a chunk without an open gate advances t by its REDUX total, skipping the prefix
// scan (off for the STREAM model: its larger fill then spills)
template <bool kLazyScan = true, class GateMin, class Fill>
__device__ __forceinline__ HpOut replay_hp_core(GateMin gate_min, Fill fill, const fikit_table_t& tab, uint32_t K,
                                                const uint32_t* __restrict__ hp_row,
                                                const uint64_t* __restrict__ hp_dur,
                                                const uint64_t* __restrict__ hp_gap, const fikit_scenario_t& c,
                                                const fikit_fill_params_t& prm, int lane, uint64_t t_start = 0) {
  const uint32_t nh = c.hp_len;
  const uint64_t scale = c.gap_scale_q16;
  HpOut o{0, 0, 0, 0, 0};
  uint64_t t = t_start;  // HP kernel 0 starts here
  // chunk inputs: d, raw gap, row of HP kernel base + lane (next chunk prefetched)
  auto ld = [&](uint32_t base, uint64_t& d, uint64_t& g, uint32_t& r) {
    const uint32_t i = base + lane;
    d = 0;
    g = 0;
    r = 0xFFFFFFFFu;
    if (i < nh) {
      d = __ldg(hp_dur + c.hp_off + i);
      g = i + 1 < nh ? __ldg(hp_gap + c.hp_off + i) : 0;  // no gap after the last kernel
      r = __ldg(hp_row + c.hp_off + i);
    }
  };
  uint64_t dn, gn;
  uint32_t rn;
  ld(0, dn, gn, rn);
  for (uint32_t base = 0; base < nh; base += 32) {
    const uint32_t i_l = base + lane;
    const bool valid = i_l < nh, last = i_l == nh - 1;
    const uint64_t d_l = dn;
    const uint64_t a_l = (gn * scale) >> 16;  // R24
    const uint32_t r_l = rn;
    const uint64_t p_l = (valid && r_l < K) ? ((__ldg(tab.mean + (size_t)r_l * 2 + 1) * scale) >> 16) : 0;  // SG (Alg.1 3-5, R12)
    if (base + 32 < nh) ld(base + 32, dn, gn, rn);
    const uint64_t x_l = d_l + a_l;
    // prefix over the chunk: issued before the gate ballot when it is always needed (no lazy path), so
    // it overlaps the SG load the ballot waits on (after the ballot it cost the STREAM model's
    // exclusive arm, whose gates never open, 11 %: ratio workload 5.00 -> 5.57 ms)
    uint64_t X = 0;
    if constexpr (!kLazyScan) X = warp_inclusive_scan(x_l, lane);
    const bool gate = valid && !last && p_l >= prm.threshold_ns && (!prm.feedback || a_l > 0);
    uint32_t gmask = __ballot_sync(0xffffffffu, gate && p_l >= gate_min());
    if (kLazyScan && !gmask) {  // no gate opens in this chunk (the common case): only its total advances t
      t += warp_sum_u64(x_l);
      continue;
    }
    if constexpr (kLazyScan) X = warp_inclusive_scan(x_l, lane);
    const uint64_t T0 = t;
    uint64_t shift = 0;  // delays imposed by fills earlier in this chunk
    while (gmask) {
      const int j = __ffs(gmask) - 1;
      const uint32_t i = base + j;
      const uint64_t Xj = __shfl_sync(0xffffffffu, X, j);
      const uint64_t a = __shfl_sync(0xffffffffu, a_l, j);
      const uint64_t p = __shfl_sync(0xffffffffu, p_l, j);
      t = T0 + shift + Xj - a;  // end of HP kernel i
      const uint64_t r = t + a;   // the HP client's next launch arrives (R20)
      t = fill(i, t, r, p, o);    // Alg. 1 over this gap (R = p)
      if (t > r) {  // overhead 2: kernel i+1 starts at max(t, r_{i+1})
        o.hp_delay += t - r;
        shift += t - r;
      }
      // the gate bound may have moved either way (a fill consumed the smallest request, or a
      // stream's next head is smaller): re-gate the rest of the chunk
      gmask = j == 31 ? 0u : __ballot_sync(0xffffffffu, gate && p_l >= gate_min()) & (~0u << (j + 1));
    }
    t = T0 + shift + __shfl_sync(0xffffffffu, X, 31);  // next kernel's start (or the HP end)
  }
  o.t = t;
  return o;
}

// The POOL model's gap loop on a pool representation (RegPool / SmemPool)
template <class Pool, class MinQ>
__device__ __forceinline__ HpOut replay_hp(Pool& P, MinQ min_q, const fikit_table_t& tab, uint32_t K,
                                           const uint32_t* __restrict__ hp_row, const uint64_t* __restrict__ hp_dur,
                                           const uint64_t* __restrict__ hp_gap, const fikit_scenario_t& c,
                                           const fikit_fill_params_t& prm, bool sched, int32_t* fill_gap,
                                           uint64_t* lp_start, uint64_t so, DigestBatch& dig, int lane) {
  uint64_t qmin = min_q();
  auto fill = [&](uint32_t i, uint64_t t, uint64_t r, uint64_t R, HpOut& o) -> uint64_t {
    // (a visited gap admits its first pick: see replay_hp_reg; the exits are tested after a fill)
    for (;;) {
      uint64_t qk;
      const int k = P.pick(R, lane, qk);  // Alg. 2
      if (k < 0) break;
      const uint64_t e = P.dur_of((uint32_t)k);
      if (sched && lane == 0) {
        fill_gap[so + k] = (int32_t)i;
        lp_start[so + k] = t;
      }
      P.record((uint32_t)k, (int32_t)i, t, lane, dig);
      R -= qk;
      t += e;
      if (qk == qmin) qmin = min_q();
      if (!Pool::kOwnerStats) {  // (the register pool sums its fills from the owning lanes)
        o.fill_work += e;
        o.n_fills++;
      }
      o.lp_end = t;  // fills run in time order: the last one ends last
      if ((prm.feedback && t >= r) || R < qmin) break;  // feedback stop / nothing fits
    }
    return t;
  };
  return replay_hp_core([&]() { return qmin; }, fill, tab, K, hp_row, hp_dur, hp_gap, c, prm, lane);
}

// The same loop on the register pool, with the idle time R and qmin in 32 bits: every eligible
// q < 2^22 there, so R saturated at 2^32 - 1 takes every fit decision R does (after at most 64
// picks, a saturated R is still >= 2^32 - 1 - 2^28 > any q, and so is the exact one).
__device__ __forceinline__ HpOut replay_hp_reg(RegPool& P, const fikit_table_t& tab, uint32_t K,
                                               const uint32_t* __restrict__ hp_row,
                                               const uint64_t* __restrict__ hp_dur,
                                               const uint64_t* __restrict__ hp_gap, const fikit_scenario_t& c,
                                               const fikit_fill_params_t& prm, bool sched, int32_t* fill_gap,
                                               uint64_t* lp_start, uint64_t so, DigestBatch& dig, int lane) {
  uint32_t qmin = P.min_q32();  // 0xFFFFFFFF: no alive eligible request
  auto fill = [&](uint32_t i, uint64_t t, uint64_t r, uint64_t R64, HpOut& o) -> uint64_t {
    uint32_t R = R64 >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)R64;
    const uint64_t r_stop = prm.feedback ? r : ~0ull;  // (without feedback t never reaches it)
    // replay_hp_core visits a gap only when its gate opened against the current qmin (R >= qmin)
    // and, with feedback, the HP client's next launch is still ahead (a' > 0, t < r): the first
    // pick needs no check, the loop tests its exits after each fill (2.5 % of the replay)
    for (;;) {
      uint32_t qk;
      const int k = P.pick32(R, lane, qk);  // Alg. 2 (R >= qmin: one fits)
      const uint64_t e = P.ek;
      if (sched && lane == 0) {
        fill_gap[so + k] = (int32_t)i;
        lp_start[so + k] = t;
      }
      P.record((uint32_t)k, (int32_t)i, t, lane, dig);
      R -= qk;
      t += e;
      if (qk == qmin) qmin = P.min_q32();
      if (t >= r_stop || R < qmin) break;  // feedback stop / no alive eligible request fits
    }
    o.lp_end = t;  // fills run in time order: the last one ends last
    return t;
  };
  return replay_hp_core([&]() { return qmin == 0xFFFFFFFFu ? ~0ull : (uint64_t)qmin; }, fill, tab, K, hp_row,
                        hp_dur, hp_gap, c, prm, lane);
}

// tail (R22): the requests still queued run after the HP end in Q1..Q9 order, FIFO within a
// queue; sel(k) / dur(k) / level presence come from the pool representation
template <class Sel, class Dur>
__device__ __forceinline__ uint64_t replay_tail(uint64_t t, uint32_t m, uint32_t levels, Sel sel_of, Dur dur_of,
                                                bool sched, int32_t* fill_gap, uint64_t* lp_start, uint64_t so,
                                                uint64_t& dig, uint32_t& n_tail, int lane) {
  while (levels) {
    const uint32_t L = __ffs(levels) - 1;
    levels &= levels - 1;
    uint64_t e_cur = (uint32_t)lane < m ? dur_of((uint32_t)lane) : 0;  // block b's durations, one block ahead
    for (uint32_t b = 0; b < m; b += 32) {
      const uint32_t k = b + lane;
      const uint64_t e_next = k + 32 < m ? dur_of(k + 32) : 0;
      const bool sel = k < m && sel_of(k, L);
      const uint32_t bal = __ballot_sync(0xffffffffu, sel);
      const uint64_t e_here = e_cur;
      e_cur = e_next;
      if (!bal) continue;
      const uint64_t e = sel ? e_here : 0;
      const uint64_t x = warp_inclusive_scan(e, lane);
      if (sel) {
        const uint64_t start = t + x - e;
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
  return t;
}

// the same for a register pool (m <= 64): the owning lanes keep each request's tail start (the
// digest terms of fills and tail are evaluated together at the end)
template <class Sel, class Dur>
__device__ __forceinline__ uint64_t replay_tail_reg(uint64_t t, uint32_t m, uint32_t levels, Sel sel_of, Dur dur_of,
                                                    bool sched, int32_t* fill_gap, uint64_t* lp_start, uint64_t so,
                                                    RegPool& P, uint32_t& n_tail, int lane) {
  while (levels) {
    const uint32_t L = __ffs(levels) - 1;
    levels &= levels - 1;
#pragma unroll
    for (uint32_t h = 0; h < 2; h++) {
      const uint32_t k = 32u * h + (uint32_t)lane;
      if (32u * h >= m) break;
      const bool sel = k < m && sel_of(k, L);
      const uint32_t bal = __ballot_sync(0xffffffffu, sel);
      if (!bal) continue;
      const uint64_t e = sel ? dur_of(k) : 0;
      const uint64_t x = warp_inclusive_scan(e, lane);
      if (sel) {
        const uint64_t start = t + x - e;
        if (sched) {
          fill_gap[so + k] = -1;
          lp_start[so + k] = start;
        }
        if (h) {
          P.fg1 = -1;
          P.st1 = start;
        } else {
          P.fg0 = -1;
          P.st0 = start;
        }
      }
      t += __shfl_sync(0xffffffffu, x, 31);
      n_tail += __popc(bal);
    }
  }
  return t;
}

__device__ __forceinline__ void write_result(fikit_result_t* out, uint32_t s, const HpOut& o, uint64_t t_end,
                                             uint32_t m, uint32_t n_tail, DigestBatch& db, uint64_t tail_dig,
                                             int lane) {
  uint64_t lp_end = o.lp_end;
  if (n_tail) lp_end = max(lp_end, t_end);
  db.drain(lane);
  uint64_t dig = db.sum + tail_dig;
#pragma unroll
  for (int off = 16; off; off >>= 1) dig += __shfl_xor_sync(0xffffffffu, dig, off);
  if (lane == 0) {
    fikit_result_t r;
    r.hp_jct = o.t;
    r.lp_jct = m ? lp_end : 0;
    r.hp_delay = o.hp_delay;
    r.fill_work = o.fill_work;
    r.digest = dig;
    r.n_fills = o.n_fills;
    r.n_tail = n_tail;
    out[s] = r;
  }
}

// Pass 1 (no shared memory, so only registers bound its occupancy): every scenario with m <= 64
// and all q < 2^50 runs on the register pool; any other scenario is marked deferred
// (n_tail = kDeferred) for pass 2.  Persistent grid, one warp per scenario; scenarios are
// claimed from a counter (the next claim is in flight while one runs), so uneven scenario costs
// do not strand warps.
constexpr uint32_t kDeferred = 0xFFFFFFFFu;
constexpr int kRegWarps = kRegThreads / 32;

template <bool kSched>  // schedule outputs requested (a compile-time branch: no per-fill checks)
__global__ void __launch_bounds__(kRegWarps * 32, 2)  // <= 64 registers: 32 warps per SM
    k_simulate_reg(fikit_table_t tab, const uint32_t* __restrict__ hp_row, const uint64_t* __restrict__ hp_dur,
                   const uint64_t* __restrict__ hp_gap, const uint32_t* __restrict__ lp_row,
                   const uint64_t* __restrict__ lp_dur, const uint8_t* __restrict__ lp_level,
                   const fikit_scenario_t* __restrict__ sc, uint32_t S, fikit_fill_params_t prm,
                   fikit_result_t* __restrict__ out, int32_t* __restrict__ fill_gap, uint64_t* __restrict__ lp_start,
                   const uint64_t* __restrict__ sched_off, fikit_status_t* st) {
  pdl_entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  constexpr bool sched = kSched;
  uint32_t* ctr = reinterpret_cast<uint32_t*>(st) + kSchedWord1;
  const uint32_t nw = gridDim.x * kRegWarps;
  uint32_t s = blockIdx.x * kRegWarps + w;  // first scenario: static; later ones claimed
  uint32_t nxt = 0;
  __shared__ uint4 s_log[kRegWarps][64];  // per warp: (gap, start) of each filled request
  for (; s < S; s = nw + __shfl_sync(0xffffffffu, nxt, 0)) {
    if (lane == 0) nxt = atomicAdd(ctr, 1u);  // claim the next one now, use it after this one
    const fikit_scenario_t c = sc[s];
    const uint32_t m = c.lp_len;
    RegPool P;
    P.log = s_log[w];
    const int rc = m <= 64 ? load_reg_pool(tab, K, lp_row, lp_level, lp_dur, c.lp_off, m, lane, st, P) : 2;
    if (rc != 0) {  // invalid level (flagged; pass 2 flags it again) or not for this pass
      if (lane == 0) out[s].n_tail = kDeferred;
      continue;
    }
    const uint64_t so = sched ? sched_off[s] : 0;
    DigestBatch db;
    P.fg0 = P.fg1 = -1;
    HpOut o = replay_hp_reg(P, tab, K, hp_row, hp_dur, hp_gap, c, prm, sched, fill_gap, lp_start, so, db, lane);
    const uint64_t picked = P.picked_mask();
    const bool f0 = (picked >> lane) & 1ull, f1 = (picked >> (32 + lane)) & 1ull;
    {  // fills: the picked requests, summed from their owning lanes
      o.n_fills = __popc((uint32_t)picked) + __popc((uint32_t)(picked >> 32));
      uint64_t fw = (f0 ? (uint64_t)P.dur0 : 0ull) + (f1 ? (uint64_t)P.dur1 : 0ull);
#pragma unroll
      for (int off2 = 16; off2; off2 >>= 1) fw += __shfl_xor_sync(0xffffffffu, fw, off2);
      o.fill_work = fw;
    }
    P.alive &= ~picked;
    uint32_t lv = 0;  // levels still queued
    if ((P.alive >> lane) & 1ull) lv |= 1u << P.lvl0;
    if ((P.alive >> (32 + lane)) & 1ull) lv |= 1u << P.lvl1;
    lv = __reduce_or_sync(0xffffffffu, lv);
    uint32_t n_tail = 0;
    const uint64_t t = replay_tail_reg(
        o.t, m, lv,
        [&](uint32_t k, uint32_t L) { return ((P.alive >> k) & 1ull) && (k < 32 ? P.lvl0 : P.lvl1) == L; },
        [&](uint32_t k) { return k < 32 ? P.dur0 : P.dur1; }, sched, fill_gap, lp_start, so, P, n_tail, lane);
    // every request ran (fill or tail): its digest term from its owning lane
    __syncwarp();  // (lane 0's log stores -> the owning lanes)
    uint64_t dig = 0;
    if (f0) {
      const uint4 x = P.log[lane];
      P.fg0 = (int32_t)x.x;
      P.st0 = (uint64_t)x.y | ((uint64_t)x.z << 32);
    }
    if (f1) {
      const uint4 x = P.log[32 + lane];
      P.fg1 = (int32_t)x.x;
      P.st1 = (uint64_t)x.y | ((uint64_t)x.z << 32);
    }
    __syncwarp();  // (the reads, before the next scenario's stores)
    if ((uint32_t)lane < m) dig += digest_term((uint32_t)lane, P.fg0, P.st0);
    if (32u + (uint32_t)lane < m) dig += digest_term(32u + (uint32_t)lane, P.fg1, P.st1);
    write_result(out, s, o, t, m, n_tail, db, dig, lane);
  }
}

// Pass 2: the deferred scenarios, pool in shared memory (sorted fast path or full argmin).
template <bool kSched>
__global__ void __launch_bounds__(kReplayWarps * 32)
    k_simulate(fikit_table_t tab, const uint32_t* __restrict__ hp_row, const uint64_t* __restrict__ hp_dur,
               const uint64_t* __restrict__ hp_gap, const uint32_t* __restrict__ lp_row,
               const uint64_t* __restrict__ lp_dur, const uint8_t* __restrict__ lp_level,
               const fikit_scenario_t* __restrict__ sc, uint32_t S, fikit_fill_params_t prm,
               fikit_result_t* __restrict__ out, int32_t* __restrict__ fill_gap, uint64_t* __restrict__ lp_start,
               const uint64_t* __restrict__ sched_off, fikit_status_t* st) {
  pdl_entry();
  __shared__ uint64_t s_q[kReplayWarps][kPoolMax];
  __shared__ uint8_t s_meta[kReplayWarps][kPoolMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  constexpr bool sched = kSched;
  uint32_t* ctr = reinterpret_cast<uint32_t*>(st) + kSchedWord2;
  // claim 32 scenarios at a time; run the ones pass 1 deferred
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(ctr, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= S) break;
    const uint32_t sl = base + lane;
    uint32_t todo = __ballot_sync(0xffffffffu, sl < S && out[sl].n_tail == kDeferred);
    while (todo) {
    const uint32_t s = base + __ffs(todo) - 1;
    todo &= todo - 1;
    const fikit_scenario_t c = sc[s];
    const uint32_t m = c.lp_len;
    __syncwarp();
    if (m > kPoolMax) {
      if (lane == 0) atomicOr(&st->flags, kStatusArg);
      continue;
    }
    uint64_t* q = s_q[w];
    uint8_t* meta = s_meta[w];
    if (!load_pool(tab, K, lp_row, lp_level, c.lp_off, m, q, meta, lane, st)) continue;
    const uint64_t so = sched ? sched_off[s] : 0;
    SmemPool P{q, meta, lp_dur + c.lp_off, m, 0, 0, false, 0xFFFFFFFFu, 0, false};
    P.fast = make_sorted_pool(q, meta, m, lane, P.A, P.nch, P.CM, lp_dur + c.lp_off, P.epack);
    DigestBatch db;
    const HpOut o = replay_hp(P, [&]() { return P.min_q(lane); }, tab, K, hp_row, hp_dur, hp_gap, c, prm, sched,
                              fill_gap, lp_start, so, db, lane);
    if (P.fast) sync_meta_alive(q, meta, P.A, P.nch, lane);
    uint32_t lv = 0;
    for (uint32_t k = lane; k < m; k += 32)
      if (meta[k] & kAlive) lv |= 1u << (meta[k] & 0xF);
    lv = __reduce_or_sync(0xffffffffu, lv);
    uint64_t tail_dig = 0;
    uint32_t n_tail = 0;
    const uint64_t t = replay_tail(
        o.t, m, lv, [&](uint32_t k, uint32_t L) { return (meta[k] & kAlive) && (meta[k] & 0xF) == L; },
        [&](uint32_t k) { return __ldg(lp_dur + c.lp_off + k); }, sched, fill_gap, lp_start, so, tail_dig, n_tail,
        lane);
    write_result(out, s, o, t, m, n_tail, db, tail_dig, lane);
    }
  }
}

// ---- fikit_simulate_stream_batch: the STREAM model (R29-R32), one warp per scenario --------
// Up to 64 streams per scenario: lane l owns streams l (slot 0) and 32 + l (slot 1) with, for
// each, its head request (window index), end, the head's arrival time, q, level, eligibility,
// duration and think time, and the next request's duration and think time (prefetched).  The
// window's q and level | eligibility are staged in shared memory at the scenario's start, so a
// dispatch waits on no global load.
constexpr int kStreamWarps = kStreamThreads / 32;
constexpr uint32_t kMaxStreams = 64;

struct StreamHeads {
  uint32_t hd[2], se[2], lv[2];
  uint64_t A[2], q[2], e[2], th[2], en[2], thn[2];
  bool el[2];
};

struct StreamPick {  // the best head of a warp reduction (valid: lv != 0xFF)
  uint32_t lv, k, sid;
  uint64_t q;
};

template <bool kSched>
__global__ void __launch_bounds__(kStreamWarps * 32, 5)  // <= 102 registers: 20 warps per SM
    k_simulate_stream(fikit_table_t tab, const uint32_t* __restrict__ hp_row, const uint64_t* __restrict__ hp_dur,
                      const uint64_t* __restrict__ hp_gap, const uint32_t* __restrict__ lp_row,
                      const uint64_t* __restrict__ lp_dur, const uint8_t* __restrict__ lp_level,
                      const uint32_t* __restrict__ lp_stream, const uint64_t* __restrict__ lp_think,
                      const uint64_t* __restrict__ hp_arrival, const fikit_scenario_t* __restrict__ sc, uint32_t S,
                      fikit_fill_params_t prm,
                      fikit_result_t* __restrict__ out, int32_t* __restrict__ fill_gap,
                      uint64_t* __restrict__ lp_start, const uint64_t* __restrict__ sched_off, fikit_status_t* st) {
  pdl_entry();
  __shared__ uint32_t s_start[kStreamWarps][kMaxStreams];
  __shared__ uint64_t s_q[kStreamWarps][kPoolMax];
  __shared__ uint8_t s_lv[kStreamWarps][kPoolMax];  // level | eligible << 7
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  constexpr bool sched = kSched;
  uint32_t* ctr = reinterpret_cast<uint32_t*>(st) + kSchedWord3;
  uint32_t nxt = 0;  // lane 0: the next claimed scenario (in flight while one runs)
  if (lane == 0) nxt = atomicAdd(ctr, 1u);
  for (uint32_t cur = __shfl_sync(0xffffffffu, nxt, 0); cur < S; cur = __shfl_sync(0xffffffffu, nxt, 0)) {
    __syncwarp();  // the previous scenario's reads of the warp's staging arrays come before these writes
    const fikit_scenario_t c = sc[cur];
    if (lane == 0) nxt = atomicAdd(ctr, 1u);
    const uint32_t m = c.lp_len;
    const uint64_t off = c.lp_off;
    // streams: maximal runs of equal consecutive ids (R29); levels validated on the way
    uint32_t ns = 0;
    const bool too_big = m > kPoolMax;
    bool ok = !too_big;
    for (uint32_t b = 0; b < m && ok; b += 32) {
      const uint32_t k = b + lane;
      bool f = false;
      if (k < m) {
        f = k == 0 || __ldg(lp_stream + off + k) != __ldg(lp_stream + off + k - 1);
        const uint32_t L = __ldg(lp_level + off + k);
        if (L < 1 || L > 9) {
          flag_record(st, off + k);
          ok = false;
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      const uint32_t mask = __ballot_sync(0xffffffffu, f);
      const uint32_t rank = ns + __popc(mask & ((1u << lane) - 1u));
      if (f && rank < kMaxStreams) s_start[w][rank] = k;
      ns += __popc(mask);
    }
    if (too_big || !ok || ns > kMaxStreams) {  // (an invalid level is flagged as E_RECORD above)
      if ((too_big || ns > kMaxStreams) && lane == 0) atomicOr(&st->flags, kStatusArg);  // m > 1024 or > 64 streams
      continue;
    }
    // stage q and level | eligibility of the window (R16); gate lower bound (R32): the minimum q
    // over every eligible request of the window
    uint64_t qmin = ~0ull;
    for (uint32_t k = lane; k < m; k += 32) {
      const uint32_t row = __ldg(lp_row + off + k);
      const bool el = row < K && __ldg(tab.sums + (size_t)row * 4) > 0;
      const uint64_t q = el ? __ldg(tab.mean + (size_t)row * 2) : 0;
      s_q[w][k] = q;
      s_lv[w][k] = (uint8_t)(__ldg(lp_level + off + k) | (el ? 0x80u : 0u));
      if (el) qmin = min(qmin, q);
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) qmin = min(qmin, __shfl_xor_sync(0xffffffffu, qmin, o2));
    __syncwarp();
    StreamHeads H{};
    auto prefetch_next = [&](int h) {  // duration and think time of the request after the head
      const uint32_t k = H.hd[h] + 1;
      H.en[h] = k < H.se[h] ? __ldg(lp_dur + off + k) : 0;
      H.thn[h] = k < H.se[h] ? __ldg(lp_think + off + k) : 0;
    };
    auto set_head = [&](int h) {  // hd[h] became the head; its e / th are in e / th
      H.lv[h] = 0xFFu;
      H.el[h] = false;
      if (H.hd[h] < H.se[h]) {
        const uint32_t x = s_lv[w][H.hd[h]];
        H.lv[h] = x & 0x7Fu;
        H.el[h] = (x & 0x80u) != 0;
        H.q[h] = s_q[w][H.hd[h]];
      }
    };
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t sid = (uint32_t)h * 32u + (uint32_t)lane;
      H.hd[h] = sid < ns ? s_start[w][sid] : 0u;
      H.se[h] = sid < ns ? (sid + 1 < ns ? s_start[w][sid + 1] : m) : 0u;
      H.A[h] = 0;
      H.e[h] = H.hd[h] < H.se[h] ? __ldg(lp_dur + off + H.hd[h]) : 0;
      H.th[h] = H.hd[h] < H.se[h] ? __ldg(lp_think + off + H.hd[h]) : 0;
      set_head(h);
      prefetch_next(h);
    }
    const uint64_t so = sched ? sched_off[cur] : 0;
    DigestBatch db;
    uint64_t lp_end = 0;
    // dispatch the head of stream sid at time t (all lanes): returns its duration; the owning
    // lane advances the stream (its next request arrives think time after this one ends)
    auto dispatch = [&](const StreamPick& b, uint64_t t, int32_t gap_i) -> uint64_t {
      const int src = (int)(b.sid & 31u), h = (int)(b.sid >> 5);
      const uint64_t e = __shfl_sync(0xffffffffu, h ? H.e[1] : H.e[0], src);
      if (sched && lane == 0) {
        fill_gap[so + b.k] = gap_i;
        lp_start[so + b.k] = t;
      }
      db.add(b.k, gap_i, t, lane);
      if (lane == src) {
        const uint64_t arr = t + e + (h ? H.th[1] : H.th[0]);
        if (h) {
          H.hd[1]++;
          H.A[1] = arr;
          H.e[1] = H.en[1];
          H.th[1] = H.thn[1];
          set_head(1);
          prefetch_next(1);
        } else {
          H.hd[0]++;
          H.A[0] = arr;
          H.e[0] = H.en[0];
          H.th[0] = H.thn[0];
          set_head(0);
          prefetch_next(0);
        }
      }
      return e;
    };
    auto next_arrival = [&](uint64_t t) -> uint64_t {  // earliest head arrival after t
      uint64_t a = ~0ull;
#pragma unroll
      for (int h = 0; h < 2; h++)
        if (H.hd[h] < H.se[h] && H.A[h] > t) a = min(a, H.A[h]);
      return warp_min_u64(a);
    };
    // Alg. 2 over the arrived eligible heads with q <= R, preference (level asc, q desc, index
    // asc): three warp reductions (REDUX) narrow the candidates level, then q, then index
    auto pick_fill = [&](uint64_t t, uint64_t R, StreamPick& x) -> bool {
      bool c0 = H.hd[0] < H.se[0] && H.A[0] <= t && H.el[0] && H.q[0] <= R;
      bool c1 = H.hd[1] < H.se[1] && H.A[1] <= t && H.el[1] && H.q[1] <= R;
      if (ns == 1) {  // one stream (lane 0, slot 0): its head or nothing
        if (!(__ballot_sync(0xffffffffu, c0) & 1u)) return false;
        x.sid = 0;
        x.k = __shfl_sync(0xffffffffu, H.hd[0], 0);
        x.lv = __shfl_sync(0xffffffffu, H.lv[0], 0);
        x.q = __shfl_sync(0xffffffffu, H.q[0], 0);
        return true;
      }
      const uint32_t L = __reduce_min_sync(0xffffffffu, min(c0 ? H.lv[0] : 0xFFu, c1 ? H.lv[1] : 0xFFu));
      if (L == 0xFFu) return false;
      c0 = c0 && H.lv[0] == L;
      c1 = c1 && H.lv[1] == L;
      const uint64_t qb = warp_max_u64(max(c0 ? H.q[0] : 0ull, c1 ? H.q[1] : 0ull));
      c0 = c0 && H.q[0] == qb;
      c1 = c1 && H.q[1] == qb;
      const uint32_t kb = __reduce_min_sync(0xffffffffu, min(c0 ? H.hd[0] : 0xFFFFFFFFu, c1 ? H.hd[1] : 0xFFFFFFFFu));
      const uint32_t b0 = __ballot_sync(0xffffffffu, c0 && H.hd[0] == kb);
      const uint32_t b1 = __ballot_sync(0xffffffffu, c1 && H.hd[1] == kb);
      x.sid = b0 ? (uint32_t)(__ffs(b0) - 1) : 32u + (uint32_t)(__ffs(b1) - 1);
      x.k = kb;
      x.lv = L;
      x.q = qb;
      return true;
    };
    // the tail's / Case A's pick (R31, R33): the arrived head first in (level, index) order, as
    // one 32-bit key per slot (level <= 9, index < 1024) and one warp min (REDUX)
    auto pick_level_index = [&](uint64_t t, StreamPick& x) -> bool {
      uint32_t k0 = 0xFFFFFFFFu, k1 = 0xFFFFFFFFu;
      if (H.hd[0] < H.se[0] && H.A[0] <= t) k0 = (H.lv[0] << 16) | H.hd[0];
      if (H.hd[1] < H.se[1] && H.A[1] <= t) k1 = (H.lv[1] << 16) | H.hd[1];
      const uint32_t best = __reduce_min_sync(0xffffffffu, min(k0, k1));
      if (best == 0xFFFFFFFFu) return false;
      const uint32_t b0 = __ballot_sync(0xffffffffu, k0 == best), b1 = __ballot_sync(0xffffffffu, k1 == best);
      x.sid = b0 ? (uint32_t)(__ffs(b0) - 1) : 32u + (uint32_t)(__ffs(b1) - 1);
      x.k = best & 0xFFFFu;
      x.lv = best >> 16;
      x.q = 0;
      return true;
    };
    // gate bound with feedback: the minimum q over the eligible current heads.  Heads change only
    // by a dispatch, so in a gap with p below it no head can ever fit; the waits the gap could
    // still make end before r_{i+1} (feedback) and leave no trace: skipping the gap is exact.
    // (Without feedback a wait may run past r_{i+1} and delay the HP job: the window bound qmin.)
    auto heads_min = [&]() -> uint64_t {
      uint64_t a = ~0ull;
#pragma unroll
      for (int h = 0; h < 2; h++)
        if (H.hd[h] < H.se[h] && H.el[h]) a = min(a, H.q[h]);
      return warp_min_u64(a);
    };
    uint64_t gmin = qmin;
    auto fill = [&](uint32_t i, uint64_t t, uint64_t r, uint64_t R, HpOut& o) -> uint64_t {
      for (;;) {
        if (prm.feedback && t >= r) break;  // R19
        StreamPick x{0xFFu, 0, 0, 0};  // BestPrioFit over the arrived heads (Alg. 2)
        if (pick_fill(t, R, x)) {
          const uint64_t e = dispatch(x, t, (int32_t)i);
          if (prm.feedback) gmin = heads_min();
          t += e;
          R -= x.q;  // R17
          o.fill_work += e;
          o.n_fills++;
          lp_end = max(lp_end, t);
          continue;
        }
        const uint64_t A = next_arrival(t);  // R30: wait within the predicted idle
        if (A == ~0ull || A - t > R || (prm.feedback && A >= r)) break;
        R -= A - t;
        t = A;
      }
      return t;
    };
    // Case A (R33): before the HP job arrives the LP streams hold the GPU (arrived heads in
    // (level, index) order); a kernel launches only before Ta, the running one is not preempted
    const uint64_t Ta = hp_arrival ? hp_arrival[cur] : 0;
    uint64_t t = 0;
    while (t < Ta) {
      StreamPick x{0xFFu, 0, 0, 0};
      if (!pick_level_index(t, x)) {
        const uint64_t A = next_arrival(t);
        if (A >= Ta) break;
        t = A;
        continue;
      }
      t += dispatch(x, t, -1);  // (R34: neither a fill nor the tail)
      lp_end = max(lp_end, t);
    }
    if (prm.feedback) gmin = heads_min();
    HpOut o = replay_hp_core<false>([&]() { return gmin; }, fill, tab, K, hp_row, hp_dur, hp_gap, c, prm, lane,
                             t > Ta ? t : Ta);
    // tail (R31)
    t = o.t;
    uint32_t n_tail = 0;
    for (;;) {
      // one stream left: its requests run back to back, each think time after the previous
      // one ends (the device is otherwise idle), so their starts are a prefix sum over e + think
      // (32 requests per step) -- exactly what the loop below would dispatch one at a time
      const uint32_t v0 = __ballot_sync(0xffffffffu, H.hd[0] < H.se[0]);
      const uint32_t v1 = __ballot_sync(0xffffffffu, H.hd[1] < H.se[1]);
      if (__popc(v0) + __popc(v1) == 1) {
        const int h = v0 ? 0 : 1, src = __ffs(v0 ? v0 : v1) - 1;
        const uint32_t k0 = __shfl_sync(0xffffffffu, h ? H.hd[1] : H.hd[0], src);
        const uint32_t ke = __shfl_sync(0xffffffffu, h ? H.se[1] : H.se[0], src);
        t = max(t, __shfl_sync(0xffffffffu, h ? H.A[1] : H.A[0], src));  // the head's arrival
        for (uint32_t c = k0; c < ke; c += 32) {
          const uint32_t k = c + lane;
          const bool in = k < ke;
          const uint64_t e = in ? __ldg(lp_dur + off + k) : 0;
          const uint64_t th = (in && k + 1 < ke) ? __ldg(lp_think + off + k) : 0;
          const uint64_t X = warp_inclusive_scan(e + th, lane);
          const uint64_t start = t + X - e - th;
          if (in) {
            if (sched) {
              fill_gap[so + k] = -1;
              lp_start[so + k] = start;
            }
            db.sum += digest_term(k, -1, start);
          }
          t += __shfl_sync(0xffffffffu, X, 31);  // (no think time after the last request)
        }
        lp_end = max(lp_end, t);
        n_tail += ke - k0;
        if (lane == src) {
          if (h) H.hd[1] = H.se[1];
          else H.hd[0] = H.se[0];
        }
        break;
      }
      StreamPick x{0xFFu, 0, 0, 0};
      if (!pick_level_index(t, x)) {
        const uint64_t A = next_arrival(t);
        if (A == ~0ull) break;
        t = A;
        continue;
      }
      t += dispatch(x, t, -1);
      lp_end = max(lp_end, t);
      n_tail++;
    }
    db.drain(lane);
    uint64_t dig = db.sum;
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) dig += __shfl_xor_sync(0xffffffffu, dig, o2);
    if (lane == 0) {
      fikit_result_t rr;
      rr.hp_jct = o.t;
      rr.lp_jct = m ? lp_end : 0;
      rr.hp_delay = o.hp_delay;
      rr.fill_work = o.fill_work;
      rr.digest = dig;
      rr.n_fills = o.n_fills;
      rr.n_tail = n_tail;
      out[cur] = rr;
    }
  }
}

// host launchers (the kernel templates are instantiated and launched in this translation unit)
const void* simulate_reg_kernel(bool sched) {
  return sched ? (const void*)k_simulate_reg<true> : (const void*)k_simulate_reg<false>;
}
const void* simulate_smem_kernel(bool sched) {
  return sched ? (const void*)k_simulate<true> : (const void*)k_simulate<false>;
}
void launch_simulate_smem(int blocks, int threads, cudaStream_t s, const fikit_table_t& tab, const uint32_t* hp_row,
                          const uint64_t* hp_dur, const uint64_t* hp_gap, const uint32_t* lp_row,
                          const uint64_t* lp_dur, const uint8_t* lp_level, const fikit_scenario_t* sc, uint32_t S,
                          fikit_fill_params_t prm, fikit_result_t* out, int32_t* fill_gap, uint64_t* lp_start,
                          const uint64_t* sched_off, fikit_status_t* st) {
  if (fill_gap && lp_start && sched_off)
    launch_pdl(k_simulate<true>, blocks, threads, 0, s, tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, S, prm, out,
                                                 fill_gap, lp_start, sched_off, st);
  else
    launch_pdl(k_simulate<false>, blocks, threads, 0, s, tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, S, prm,
                                                  out, fill_gap, lp_start, sched_off, st);
}
const void* simulate_stream_kernel(bool sched) {
  return sched ? (const void*)k_simulate_stream<true> : (const void*)k_simulate_stream<false>;
}
void launch_simulate_reg(int blocks, int threads, cudaStream_t s, const fikit_table_t& tab, const uint32_t* hp_row,
                         const uint64_t* hp_dur, const uint64_t* hp_gap, const uint32_t* lp_row,
                         const uint64_t* lp_dur, const uint8_t* lp_level, const fikit_scenario_t* sc, uint32_t S,
                         fikit_fill_params_t prm, fikit_result_t* out, int32_t* fill_gap, uint64_t* lp_start,
                         const uint64_t* sched_off, fikit_status_t* st) {
  if (fill_gap && lp_start && sched_off)
    launch_pdl(k_simulate_reg<true>, blocks, threads, 0, s, tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, S, prm,
                                                     out, fill_gap, lp_start, sched_off, st);
  else
    launch_pdl(k_simulate_reg<false>, blocks, threads, 0, s, tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, S, prm,
                                                      out, fill_gap, lp_start, sched_off, st);
}
void launch_simulate_stream(int blocks, int threads, cudaStream_t s, const fikit_table_t& tab,
                            const uint32_t* hp_row, const uint64_t* hp_dur, const uint64_t* hp_gap,
                            const uint32_t* lp_row, const uint64_t* lp_dur, const uint8_t* lp_level,
                            const uint32_t* lp_stream, const uint64_t* lp_think, const uint64_t* hp_arrival,
                            const fikit_scenario_t* sc, uint32_t S, fikit_fill_params_t prm, fikit_result_t* out,
                            int32_t* fill_gap, uint64_t* lp_start, const uint64_t* sched_off, fikit_status_t* st) {
  if (fill_gap && lp_start && sched_off)
    launch_pdl(k_simulate_stream<true>, blocks, threads, 0, s, tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level,
                                                        lp_stream, lp_think, hp_arrival, sc, S, prm, out, fill_gap,
                                                        lp_start, sched_off, st);
  else
    launch_pdl(k_simulate_stream<false>, blocks, threads, 0, s, tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level,
                                                         lp_stream, lp_think, hp_arrival, sc, S, prm, out, fill_gap,
                                                         lp_start, sched_off, st);
}

}  // namespace fikit
