// finalize / means / lookup / resolve / multi-GPU dictionary kernels.
#include <cuda_runtime.h>

#include "fikit_internal.cuh"

namespace fikit {

__device__ __forceinline__ bool key_less(uint32_t ta, uint64_t ka, uint32_t tb, uint64_t kb) {
  return ta < tb || (ta == tb && ka < kb);
}

// R8: floor(sum/cnt) + [2 (sum mod cnt) >= cnt]; cnt = 0 -> 0
__device__ __forceinline__ uint64_t mean_half_up(uint64_t sum, uint64_t cnt) {
  if (cnt == 0) return 0;
  uint64_t q = sum / cnt, r = sum - q * cnt;
  return q + ((2 * r >= cnt) ? 1 : 0);
}

// fikit_table_finalize in two launches.  The canonical row of measured row r (R11) is its rank
// among the K distinct (task, kernel ID) keys.
//   k_fin_sort     one block per group of G keys (G = 256 for tables of <= 8192 rows, else kFinGroup =
//                  2048): a shared-memory bitonic sort (G / 2 threads, one compare-exchange per thread
//                  and stage), the sorted group to the workspace.
//   k_fin_scatter  block b owns rows [b R, (b + 1) R): a row's rank is the sum over the sorted
//                  groups of the keys below it (one branch-free (log2 G + 1)-step binary search per row and
//                  group in the L2-resident sorted keys, four groups interleaved per thread; staging
//                  every group in each block's shared memory had cost more than the searches, and
//                  the search loop 4 M warp-instructions per 8192 rows); then the block writes its
//                  rows into the caller's table at their ranks, a warp per half row (32 histogram
//                  bins: the count is their sum), with the sums, extremes and
//                  SK_j / SG_j (R8).
// Grids follow the capacity (the row count K is on the device); blocks past K return at once.
__device__ __forceinline__ bool fin_less(uint32_t ta, uint64_t ka, uint32_t tb, uint64_t kb) {
  return (ta < tb) | ((ta == tb) & (ka < kb));  // (branch-free: the sort network selects, never branches)
}

template <uint32_t G>  // keys per sorted group (256 up to 8192 rows, kFinGroup above)
__device__ __forceinline__ void fin_sort_body(const fikit_status_t* __restrict__ st, const RawRow* __restrict__ raw,
                                              uint32_t cap, fikit_table_t tab, FinKey* __restrict__ skeys,
                                              const uint32_t* __restrict__ misc) {
  pdl_entry();
  __shared__ uint64_t sk[G];
  __shared__ uint32_t stk[G];
  const uint32_t K = (uint32_t)umin64(st->n_rows_needed, cap);
  const uint32_t tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) *tab.n_rows = K;
  if (misc[kMiscDict]) return;  // dictionary mode: the rows are already canonical
  const uint32_t g0 = blockIdx.x * G;
  if (g0 >= K) return;
  const uint32_t m = min(G, K - g0);
  for (uint32_t i = tid; i < G; i += blockDim.x) {
    const bool in = i < m;
    sk[i] = in ? raw[g0 + i].kid : ~0ull;  // padding sorts last
    stk[i] = in ? raw[g0 + i].task : 0xFFFFFFFFu;
  }
  __syncthreads();
  // bitonic network: one compare-exchange per thread and stage (branch-free selects)
#pragma unroll
  for (uint32_t kk = 2; kk <= G; kk <<= 1)
#pragma unroll
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      const uint32_t a = ((tid & ~(j - 1)) << 1) | (tid & (j - 1)), b = a + j;
      const bool asc = (a & kk) == 0;
      const uint64_t ka = sk[a], kb = sk[b];
      const uint32_t ta = stk[a], tb = stk[b];
      const bool sw = asc ? fin_less(tb, kb, ta, ka) : fin_less(ta, ka, tb, kb);
      sk[a] = sw ? kb : ka;
      sk[b] = sw ? ka : kb;
      stk[a] = sw ? tb : ta;
      stk[b] = sw ? ta : tb;
      __syncthreads();
    }
  for (uint32_t i = tid; i < m; i += blockDim.x) skeys[g0 + i] = FinKey{sk[i], stk[i], 0u};
}
__global__ void __launch_bounds__(128) k_fin_sort256(const fikit_status_t* __restrict__ st,
                                                   const RawRow* __restrict__ raw, uint32_t cap, fikit_table_t tab,
                                                   FinKey* __restrict__ skeys, const uint32_t* __restrict__ misc) {
  fin_sort_body<256>(st, raw, cap, tab, skeys, misc);
}
__global__ void __launch_bounds__(kFinGroup / 2) k_fin_sort(const fikit_status_t* __restrict__ st,
                                                            const RawRow* __restrict__ raw, uint32_t cap,
                                                            fikit_table_t tab, FinKey* __restrict__ skeys,
                                                            const uint32_t* __restrict__ misc) {
  fin_sort_body<kFinGroup>(st, raw, cap, tab, skeys, misc);
}

__global__ void __launch_bounds__(256) k_fin_scatter(const fikit_status_t* __restrict__ st,
                                                     const RawRow* __restrict__ raw, uint32_t cap, uint32_t R,
                                                     const FinKey* __restrict__ skeys, uint32_t G, fikit_table_t tab,
                                                     uint32_t* __restrict__ rank, const uint32_t* __restrict__ misc) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char fin_sm[];
  FinKey* rk = reinterpret_cast<FinKey*>(fin_sm);              // [R] this block's row keys
  uint32_t* srank = reinterpret_cast<uint32_t*>(rk + R);       // [R]
  const uint32_t K = (uint32_t)umin64(st->n_rows_needed, cap);
  // rows per block for this K (R_max: the shared arrays' size, >= cap / gridDim): K spread over the
  // grid (one block per SM), at least 16 rows per block
  const uint32_t R_max = R;
  R = min(R_max, max(16u, ((K + gridDim.x - 1) / gridDim.x + 15u) & ~15u));
  const uint32_t r0 = blockIdx.x * R;
  if (r0 >= K) return;
  const uint32_t nr = min(R, K - r0), tid = threadIdx.x;
  const bool dict = misc[kMiscDict] != 0u;  // dictionary mode: rank = row
  for (uint32_t i = tid; i < nr; i += blockDim.x) {
    srank[i] = dict ? r0 + i : 0u;
    rk[i] = FinKey{raw[r0 + i].kid, raw[r0 + i].task, 0u};
  }
  __syncthreads();
  if (!dict) {
    // rank = the keys below the row's in every sorted group: Q threads per row, each a share of the
    // groups, four groups' branch-free binary searches interleaved (log2 G + 1 steps each: 16-B loads of the
    // L2-resident sorted keys; positions past a partial last group read as +infinity)
    const uint32_t ng = (K + G - 1) / G;
    const uint32_t Q = max(1u, (uint32_t)blockDim.x / nr);
    for (uint32_t it = tid; it < nr * Q; it += blockDim.x) {
      const uint32_t i = it / Q, q = it - i * Q;
      const uint64_t xk = rk[i].kid;
      const uint32_t xt = rk[i].task;
      uint32_t below = 0;
      for (uint32_t g0 = q * 4; g0 < ng; g0 += Q * 4) {
        uint32_t lo[4] = {0u, 0u, 0u, 0u}, m[4];
#pragma unroll
        for (int u = 0; u < 4; u++) m[u] = g0 + u < ng ? min(G, K - (g0 + u) * G) : 0u;
#pragma unroll
        for (uint32_t half = G; half; half >>= 1) {  // (log2 G + 1 steps: G + 1 possible counts)
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const uint32_t idx = lo[u] + half - 1;
            if (idx < m[u]) {
              const uint4 v = __ldg(reinterpret_cast<const uint4*>(skeys + (size_t)(g0 + u) * G + idx));
              if (fin_less(v.z, ((uint64_t)v.y << 32) | v.x, xt, xk)) lo[u] += half;
            }
          }
        }
        below += lo[0] + lo[1] + lo[2] + lo[3];
      }
      if (below) atomicAdd(&srank[i], below);
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < nr; i += blockDim.x) rank[r0 + i] = srank[i];  // (the out_row remap)
  // a warp per half row h = 2 i + j (j = 0 duration, 1 gap): 32 bins, count, sum, extremes, mean;
  // U half rows in flight per warp
  constexpr uint32_t U = 4;
  const uint32_t lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nh = 2 * nr;
  for (uint32_t h0 = warp * U; h0 < nh; h0 += nw * U) {
    // every load of the U half rows first: lane l's bin, and one 8-B word per lane -- lanes 0, 1
    // the extremes, lane 2 the sum, lane 3 the key (j = 0) -- so no load waits on a store
    uint32_t bin[U], d[U];
    uint64_t x[U];
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint32_t h = h0 + u, j = h & 1;
      const RawRow* f = raw + r0 + (h >> 1);
      const bool in = h < nh;
      bin[u] = in ? f->hist[32 * j + lane] : 0u;
      d[u] = in ? srank[h >> 1] : 0u;
      x[u] = !in ? 0ull : lane < 2 ? f->ext[2 * j + lane] : lane == 2 ? f->sums[2 * j + 1] : lane == 3 ? f->kid : 0ull;
    }
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint32_t h = h0 + u;
      if (h >= nh) break;
      const uint32_t j = h & 1;
      FK_CHECK(d[u] < K);
      tab.hist[(size_t)d[u] * 64 + 32 * j + lane] = bin[u];
      // row counts < 2^32 (a call measures < 2^32 launches)
      const uint64_t c = __reduce_add_sync(0xffffffffu, bin[u]);
      if (lane < 2) tab.ext[(size_t)d[u] * 4 + 2 * j + lane] = x[u];
      if (lane == 2) {
        tab.sums[(size_t)d[u] * 4 + 2 * j] = c;
        tab.sums[(size_t)d[u] * 4 + 2 * j + 1] = x[u];
        tab.mean[(size_t)d[u] * 2 + j] = mean_half_up(x[u], c);  // SK_j, SG_j
      }
      if (lane == 3 && j == 0) {
        tab.kernel_id[d[u]] = x[u];
        tab.task_id[d[u]] = rk[h >> 1].task;
      }
    }
  }
}

__global__ void k_remap_rows(uint32_t* rows, uint64_t n, const uint32_t* __restrict__ rank, const uint32_t* n_ptr) {
  pdl_entry();
  uint32_t K = *n_ptr;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t r = rows[i];
    rows[i] = (r < K) ? rank[r] : FIKIT_NO_ROW;
  }
}

// counts from histograms + means of an already canonical table
__global__ void k_means(fikit_table_t tab) {
  uint32_t K = min(*tab.n_rows, tab.capacity);
  uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= K) return;
  uint64_t dc = 0, gc = 0;
  for (int b = 0; b < 32; b++) {
    dc += tab.hist[(size_t)r * 64 + b];
    gc += tab.hist[(size_t)r * 64 + 32 + b];
  }
  tab.sums[(size_t)r * 4 + 0] = dc;
  tab.sums[(size_t)r * 4 + 2] = gc;
  tab.mean[(size_t)r * 2 + 0] = mean_half_up(tab.sums[(size_t)r * 4 + 1], dc);
  tab.mean[(size_t)r * 2 + 1] = mean_half_up(tab.sums[(size_t)r * 4 + 3], gc);
}

// binary search of (task, kid) in the canonical table
__device__ __forceinline__ uint32_t find_row(const uint64_t* __restrict__ kid, const uint32_t* __restrict__ task,
                                             uint32_t K, uint32_t t, uint64_t k) {
  uint32_t lo = 0, hi = K;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    uint32_t tm = __ldg(task + mid);
    uint64_t km = __ldg(kid + mid);
    if (key_less(tm, km, t, k))
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < K && __ldg(task + lo) == t && __ldg(kid + lo) == k) ? lo : FIKIT_NO_ROW;
}

// Predictor variants (R26-R28): a warp per row; lane b holds histogram bin b, a 64-bit
// inclusive scan gives cum(b), and b_P = the first lane with 100*cum >= P*count (a ballot).
__global__ void k_predict(fikit_table_t tab, uint32_t mode, uint32_t pct) {
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= K) return;
  const uint64_t dc = tab.sums[(size_t)r * 4], ds = tab.sums[(size_t)r * 4 + 1];
  const uint64_t gc = tab.sums[(size_t)r * 4 + 2], gs = tab.sums[(size_t)r * 4 + 3];
  const uint64_t dmax = tab.ext[(size_t)r * 4], gmin = ~tab.ext[(size_t)r * 4 + 3];
  uint64_t d = 0, g = 0;
  if (mode == FIKIT_PREDICT_MEAN) {
    d = mean_half_up(ds, dc);
    g = mean_half_up(gs, gc);
  } else if (mode == FIKIT_PREDICT_PERCENTILE) {
    uint64_t cd = tab.hist[(size_t)r * 64 + lane], cg = tab.hist[(size_t)r * 64 + 32 + lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t yd = __shfl_up_sync(0xffffffffu, cd, o), yg = __shfl_up_sync(0xffffffffu, cg, o);
      if ((int)lane >= o) {
        cd += yd;
        cg += yg;
      }
    }
    const uint32_t md = __ballot_sync(0xffffffffu, cd >= 1 && 100 * cd >= (uint64_t)pct * dc);
    const uint32_t mg = __ballot_sync(0xffffffffu, cg >= 1 && 100 * cg >= (uint64_t)(100 - pct) * gc);
    if (dc) {  // md != 0: at bin 31, cum = count
      const uint32_t b = __ffs(md) - 1;
      const uint64_t up = b == 0 ? 0 : (b < 31 ? (1ull << b) - 1 : dmax);
      d = up < dmax ? up : dmax;
    }
    if (gc) {
      const uint32_t b = __ffs(mg) - 1;
      const uint64_t lo = b == 0 ? 0 : (1ull << (b - 1));
      g = lo > gmin ? lo : gmin;
    }
  } else {
    d = dc ? dmax : 0;
    g = gc ? gmin : 0;
  }
  if (lane == 0) {
    tab.mean[(size_t)r * 2] = d;
    tab.mean[(size_t)r * 2 + 1] = g;
  }
}

__global__ void k_lookup(fikit_table_t tab, const uint64_t* __restrict__ kid, const uint32_t* __restrict__ task,
                         uint64_t n, uint32_t* __restrict__ out) {
  uint32_t K = min(*tab.n_rows, tab.capacity);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = find_row(tab.kernel_id, tab.task_id, K, task[i], kid[i]);
}

// profile lookup + duration + following gap of fresh launches (Alg. 1 lines 3-5).
// Persistent, one 1024-thread block per SM.  The canonical table's keys (task, kernel ID) are
// staged once per block in shared memory when K <= kResolveSmemKeys (96 KB: a lookup is a
// binary search in shared memory, ~13 steps of ~30 cycles, instead of 13 dependent L2 loads);
// larger tables are searched in global memory.  (A shared-memory hash of the keys measured no
// faster: the kernel waits on its record loads, so each warp keeps two chunks in flight.)  Each warp streams 32-launch tiles (+ the next
// launch) through its shared-memory staging buffer (coalesced 16-B loads), and writes row,
// duration and following gap.
__global__ void __launch_bounds__(kResolveThreads, 1) k_resolve(
    const uint4* __restrict__ recs, uint64_t n, const fikit_record_t* __restrict__ halo,
    const uint64_t* __restrict__ name_hash, const uint64_t* __restrict__ sig_hash, uint32_t n_names, uint32_t n_sigs,
    fikit_table_t tab, uint32_t* __restrict__ out_row, uint64_t* __restrict__ out_dur,
    uint64_t* __restrict__ out_gap, fikit_status_t* st) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char rs_sm[];
  constexpr int W = kResolveThreads / 32;
  uint4* sbuf = reinterpret_cast<uint4*>(rs_sm);                          // [W][99]
  uint64_t* skid = reinterpret_cast<uint64_t*>(sbuf + W * 99);            // [kResolveSmemKeys]
  uint32_t* stask = reinterpret_cast<uint32_t*>(skid + kResolveSmemKeys);  // [kResolveSmemKeys]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = min(*tab.n_rows, tab.capacity);
  const bool in_smem = K <= kResolveSmemKeys;
  if (in_smem) {
    constexpr uint32_t U = kResolveSmemKeys / kResolveThreads;  // keys per thread, loads in flight
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint32_t i = threadIdx.x + u * blockDim.x;
      if (i < K) {
        skid[i] = __ldg(tab.kernel_id + i);
        stask[i] = __ldg(tab.task_id + i);
      }
    }
  }
  __syncthreads();
  auto lookup = [&](uint32_t t, uint64_t k) -> uint32_t {
    const uint64_t* kid = in_smem ? skid : tab.kernel_id;
    const uint32_t* task = in_smem ? stask : tab.task_id;
    uint32_t lo = 0, hi = K;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint32_t tm = task[mid];
      const uint64_t km = kid[mid];
      if ((tm < t) | ((tm == t) & (km < k)))
        lo = mid + 1;
      else
        hi = mid;
    }
    return (lo < K && task[lo] == t && kid[lo] == k) ? lo : FIKIT_NO_ROW;
  };
  uint4* wb = sbuf + wid * 99;
  const uint64_t nchunks = (n + 31) / 32;
  const uint64_t cstride = (uint64_t)gridDim.x * W;
  uint32_t ov = 0;
  // the next chunk's 16-B words (lane, lane + 32, lane + 64, lane + 96 of its <= 99) are loaded
  // into registers before the current chunk is processed: two chunks in flight per warp
  uint4 pre[4];
  auto fetch = [&](uint64_t c) {
    const uint64_t first = c * 32;
    const uint32_t cnt3 = 3u * (uint32_t)umin64(33, n - first);
    const uint4* src = recs + first * 3;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t j = (uint32_t)lane + 32u * q;
      pre[q] = j < cnt3 ? __ldcs(src + j) : make_uint4(0, 0, 0, 0);
    }
  };
  uint64_t c = (uint64_t)blockIdx.x * W + wid;
  if (c < nchunks) fetch(c);
  for (; c < nchunks; c += cstride) {
    const uint64_t first = c * 32;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t j = (uint32_t)lane + 32u * q;
      if (j < 99) wb[j] = pre[q];
    }
    __syncwarp();
    if (c + cstride < nchunks) fetch(c + cstride);
    if (lane < (int)umin64(32, n - first)) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&wb[lane * 3]);
      const uint64_t gi = first + lane;
      if (record_valid(w, n_names, n_sigs)) {
        const uint64_t kid = kernel_id_from(__ldg(name_hash + w[4]), __ldg(sig_hash + w[5]), w[6], w[7], w[8], w[9]);
        const uint64_t start = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        const uint64_t end = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
        bool has_next = false;
        uint64_t nstart = 0;
        uint32_t nrun = 0, ntask = 0;
        if (gi + 1 < n) {
          const uint32_t* nx = reinterpret_cast<const uint32_t*>(&wb[(lane + 1) * 3]);
          nstart = (uint64_t)nx[0] | ((uint64_t)nx[1] << 32);
          nrun = nx[10];
          ntask = nx[11];
          has_next = true;
        } else if (halo) {
          nstart = halo->start_ns;
          nrun = halo->run_id;
          ntask = halo->task_id;
          has_next = true;
        }
        const bool gap = has_next && ntask == w[11] && nrun == w[10];
        const bool o = gap && nstart < end;
        ov += o;
        __stcs(out_row + gi, lookup(w[11], kid));
        __stcs(out_dur + gi, end - start);
        __stcs(out_gap + gi, (gap && !o) ? nstart - end : 0ull);
      } else {
        flag_record(st, gi);
      }
    }
  }
  ov = __reduce_add_sync(0xffffffffu, ov);
  if (lane == 0 && ov) atomicAdd((unsigned long long*)&st->n_overlap_gaps, (unsigned long long)ov);
}

// ---- multi-GPU dictionary union ----------------------------------------------
// P sorted unique key lists (stride Kmax).  Element (r, j) is canonical iff no
// list r' < r holds the same key; the union position of key x is
//   sum_r' #{canonical y in list r' : y < x} = sum_r' cpre_r'[lower_bound_r'(x)].
__device__ __forceinline__ uint32_t lower_bound_list(const uint64_t* kid, const uint32_t* task, uint32_t len,
                                                     uint32_t t, uint64_t k) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (key_less(task[mid], kid[mid], t, k))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void k_union_flags(const uint64_t* __restrict__ all_kid, const uint32_t* __restrict__ all_task,
                              const uint32_t* __restrict__ n_list, uint32_t P, uint32_t Kmax, uint32_t* canon) {
  uint32_t r = blockIdx.y;
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Kmax) return;
  uint32_t len = n_list[r];
  if (j >= len) {
    canon[(size_t)r * Kmax + j] = 0;
    return;
  }
  uint64_t k = all_kid[(size_t)r * Kmax + j];
  uint32_t t = all_task[(size_t)r * Kmax + j];
  uint32_t c = 1;
  for (uint32_t q = 0; q < r && c; q++) {
    const uint64_t* kq = all_kid + (size_t)q * Kmax;
    const uint32_t* tq = all_task + (size_t)q * Kmax;
    uint32_t lb = lower_bound_list(kq, tq, n_list[q], t, k);
    if (lb < n_list[q] && kq[lb] == k && tq[lb] == t) c = 0;
  }
  canon[(size_t)r * Kmax + j] = c;
}

// exclusive prefix of canon per list (one CTA per list); cpre has Kmax + 1 entries per list
__global__ void __launch_bounds__(1024) k_union_scan(const uint32_t* __restrict__ canon, uint32_t Kmax,
                                                     uint32_t* cpre) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  uint32_t r = blockIdx.x;
  const uint32_t* c = canon + (size_t)r * Kmax;
  uint32_t* o = cpre + (size_t)r * (Kmax + 1);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < Kmax; base += 1024) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < Kmax ? c[i] : 0;
    uint32_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t t = warp_tot[lane];
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
        if (lane >= d) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    uint32_t excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
    if (i < Kmax) o[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) o[Kmax] = carry;
}

__global__ void k_union_place(const uint64_t* __restrict__ all_kid, const uint32_t* __restrict__ all_task,
                              const uint32_t* __restrict__ n_list, uint32_t P, uint32_t Kmax, uint32_t self_rank,
                              const uint32_t* __restrict__ canon, const uint32_t* __restrict__ cpre,
                              uint64_t* out_kid, uint32_t* out_task, uint32_t cap_out, uint32_t* out_n,
                              uint32_t* local_to_union, fikit_status_t* st) {
  uint32_t r = blockIdx.y;
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0 && j == 0) {
    uint32_t tot = 0;
    for (uint32_t q = 0; q < P; q++) tot += cpre[(size_t)q * (Kmax + 1) + Kmax];
    *out_n = min(tot, cap_out);
    if (tot > cap_out) {
      atomicOr(&st->flags, kStatusCapacity);
      atomicMax((unsigned long long*)&st->n_rows_needed, (unsigned long long)tot);
    }
  }
  if (j >= n_list[r]) return;
  uint64_t k = all_kid[(size_t)r * Kmax + j];
  uint32_t t = all_task[(size_t)r * Kmax + j];
  uint32_t pos = 0;
  for (uint32_t q = 0; q < P; q++) {
    uint32_t lb = lower_bound_list(all_kid + (size_t)q * Kmax, all_task + (size_t)q * Kmax, n_list[q], t, k);
    pos += cpre[(size_t)q * (Kmax + 1) + lb];
  }
  if (canon[(size_t)r * Kmax + j] && pos < cap_out) {
    out_kid[pos] = k;
    out_task[pos] = t;
  }
  if (r == self_rank) local_to_union[j] = pos < cap_out ? pos : FIKIT_NO_ROW;
}

// local canonical rows -> dense union rows (dense table zero-initialised by the caller)
__global__ void k_table_remap(fikit_table_t local, const uint32_t* __restrict__ l2u,
                              const uint64_t* __restrict__ ukid, const uint32_t* __restrict__ utask,
                              const uint32_t* __restrict__ un, fikit_table_t dense) {
  uint32_t U = min(*un, dense.capacity);
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *dense.n_rows = U;
  if (i < U) {
    dense.kernel_id[i] = ukid[i];
    dense.task_id[i] = utask[i];
  }
  uint32_t K = min(*local.n_rows, local.capacity);
  if (i >= K) return;
  uint32_t d = l2u[i];
  if (d >= U) return;
  for (int j = 0; j < 4; j++) dense.sums[(size_t)d * 4 + j] = local.sums[(size_t)i * 4 + j];
  for (int j = 0; j < 4; j++) dense.ext[(size_t)d * 4 + j] = local.ext[(size_t)i * 4 + j];
  for (int b = 0; b < 64; b++) dense.hist[(size_t)d * 64 + b] = local.hist[(size_t)i * 64 + b];
}

__global__ void k_table_bias(fikit_table_t tab) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 4ull * tab.capacity;
       i += (uint64_t)gridDim.x * blockDim.x)
    tab.ext[i] ^= 0x8000000000000000ULL;
}

}  // namespace fikit
