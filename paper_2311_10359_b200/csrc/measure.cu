// identify + measure kernels for sm_100a.
//
// Data path of fikit_measure:
//   k_strtab_hash    FNV-1a-64 of every name / signature once (not per launch)
//   k_sample         a strided sample of launches -> (task, KID) rows in the global
//                    index, with sample counts (picks the rows worth caching)
//   k_hot_select     the <= kHotMax most-sampled rows -> hot dictionary (raw tuple -> row)
//   k_measure        persistent, one CTA per SM, 24 warps: each warp streams its own
//                    64-launch tiles global->shared with 1-D TMA (cp.async.bulk, one
//                    mbarrier stage per warp), validates each launch, looks its raw
//                    identity up in the shared hot dictionary (per task-bucket hot sets,
//                    dynamic admission) and accumulates duration and following-gap
//                    statistics into shared memory (u32 histograms, 32-bit sums with carry
//                    counters, 32-bit min/max), flushed into the table once per phase;
//                    launches of cold rows take the global path (tuple index, KID index,
//                    L2 reductions).
#include <cuda_runtime.h>

#include <type_traits>

#include "fikit_internal.cuh"

namespace fikit {

// Per-CTA timeline of k_measure for diagnosis builds only (nvcc -DFIKIT_TRACE, scripts/trace_measure.py):
// 16 u64 per CTA -- 0 entry, 1 streaming start, 2 exit (globaltimer ns), 3 phases, 4 tiles, 5 ns loading
// hot sets, 6 ns from the first warp's last tile to the phase barrier, 7 ns flushing / picking the
// next bucket, 8 cold-batch resolutions.  The product build compiles none of it.
#ifdef FIKIT_TRACE
__device__ unsigned long long g_trace[kMaxCTAs * 16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_trace_pre[2048 * 8];  // k_prep / k_plan blocks: role, stamps
#define FK_TP(slot) (g_trace_pre[blockIdx.x * 8 + (slot)] = gtime())
#define FK_TQ(slot) (g_trace_pre[(1024 + blockIdx.x) * 8 + (slot)] = gtime())
#define FK_TR_SET(slot, v) (g_trace[blockIdx.x * 16 + (slot)] = (unsigned long long)(v))
#define FK_TR_ADD(slot, v) atomicAdd(&g_trace[blockIdx.x * 16 + (slot)], (unsigned long long)(v))
#define FK_TR(x) x
#else
#define FK_TR_SET(slot, v)
#define FK_TR_ADD(slot, v)
#define FK_TR(x)
#define FK_TP(slot)
#define FK_TQ(slot)
#endif

// ------------------------------------------------------------------------------------
__device__ __forceinline__ void k_reset_status_body(fikit_status_t* st) {
  if (threadIdx.x == 0) {
    st->code = 0;
    st->flags = 0;
    st->first_bad_index = ~0ull;
    st->n_rows_needed = 0;
    st->n_overlap_gaps = 0;
    st->schedule = 0;
    st->n_task_buckets = 0;
    st->first_missing_index = ~0ull;
    reinterpret_cast<uint32_t*>(st)[kSchedWord1] = 0;
    reinterpret_cast<uint32_t*>(st)[kSchedWord2] = 0;
    reinterpret_cast<uint32_t*>(st)[kSchedWord3] = 0;
  }
}
__global__ void k_reset_status(fikit_status_t* st) {
  pdl_entry();
  k_reset_status_body(st);
}

// Zero up to kZeroRegions device regions (4-B multiples) in one launch, and (block 0) reset
// the status as k_reset_status does: the measure call's table / index / sample zeroing.
__global__ void k_zero(ZeroList z, fikit_status_t* st) {
  pdl_entry();
  if (blockIdx.x == 0 && threadIdx.x < 32) k_reset_status_body(st);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < z.k; r++) {
    unsigned char* p = static_cast<unsigned char*>(z.p[r]);
    const uint64_t n = z.n[r];
    const uint64_t mis = (16u - ((uintptr_t)p & 15u)) & 15u, head = n < mis ? n : mis;  // to 16-B alignment
    const uint64_t nv = (n - head) / 16;
    if (tid < head / 4) reinterpret_cast<uint32_t*>(p)[tid] = 0u;
    uint4* v = reinterpret_cast<uint4*>(p + head);
    for (uint64_t i = tid; i < nv; i += nt) v[i] = make_uint4(0, 0, 0, 0);
    const uint64_t done = head + 16 * nv;
    if (tid < (n - done) / 4) reinterpret_cast<uint32_t*>(p + done)[tid] = 0u;
  }
}

// Dictionary mode (fikit_measure_dict): row j of the table is dictionary key j.  Each key is
// placed in the KID index with row j (its raw row's key set; the statistics were zeroed by
// k_zero); a key not strictly above its predecessor flags E_ARG.  Thread 0 sets the row counter
// to dict_n and the workspace's dictionary word (read by finalize).
__global__ void k_dict_load(const uint64_t* __restrict__ dkid, const uint32_t* __restrict__ dtask, uint32_t K,
                            IndexEntry* idx, uint32_t slots, RawRow* raw, fikit_status_t* st, uint32_t* misc,
                            uint32_t keep_index) {
  pdl_entry();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) {
    st->n_rows_needed = K;
    misc[kMiscDict] = K + 1;
  }
  {  // the dictionary's hash (XOR of per-key mixes with their positions): a reused plan must match
     // it.  Warp-reduced first: one 64-bit atomic per warp, not per key.
    const uint64_t x = j < K ? mix64(dkid[j] ^ (0x9E3779B97F4A7C15ULL * (uint64_t)(dtask[j] + 1)) ^ ((uint64_t)j << 40))
                             : 0ull;
    const uint32_t lo = __reduce_xor_sync(0xffffffffu, (uint32_t)x), hi = __reduce_xor_sync(0xffffffffu, (uint32_t)(x >> 32));
    if ((threadIdx.x & 31) == 0 && (lo | hi))
      atomicXor(reinterpret_cast<unsigned long long*>(misc + kMiscDictHash), ((unsigned long long)hi << 32) | lo);
  }
  if (j >= K) return;
  const uint64_t kid = dkid[j];
  const uint32_t task = dtask[j];
  if (j > 0) {
    const uint32_t pt = dtask[j - 1];
    const uint64_t pk = dkid[j - 1];
    if (!(pt < task || (pt == task && pk < kid))) atomicOr(&st->flags, kStatusArg);
  }
  raw[j].kid = kid;
  raw[j].task = task;
  if (keep_index) return;  // (a reused plan: the index already maps this dictionary; the hash checks it)
  uint32_t h = key_hash(kid, task) & (slots - 1);
  for (uint32_t probe = 0; probe < slots; probe++, h = (h + 1) & (slots - 1)) {
    if (atomicCAS(&idx[h].state, 0u, kBusy) == 0u) {
      idx[h].kid = kid;
      idx[h].task = task;
      __threadfence();
      atomicExch(&idx[h].state, j + 1);
      return;
    }
  }
}

// FNV-1a 64 of one string of a table, by the whole warp: the lanes stage the string's aligned
// 16-B blocks in shared memory (buf: 64 blocks) with coalesced loads, then lane 0 runs FNV-1a
// over the bytes (serial by definition) from shared memory.  Returns the hash on lane 0.
// A malformed entry (offsets decreasing) flags E_ARG; an empty name flags E_NAME.
__device__ __forceinline__ uint64_t warp_fnv_string(const fikit_strtab_t& t, uint32_t j, bool is_name, uint4* buf,
                                                    uint32_t lane, fikit_status_t* st) {
  constexpr uint32_t CH = 64;  // 16-B blocks staged per pass (1 KB per warp)
  const uint32_t a = t.offsets[j], b = t.offsets[j + 1];
  if (b < a) {
    if (lane == 0) atomicOr(&st->flags, kStatusArg);
    return 0;
  }
  if (is_name && a == b && lane == 0) atomicOr(&st->flags, kStatusName);
  uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a 64 (R2), bytes in order
  const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<uintptr_t>(t.bytes) & ~uintptr_t(15));
  const uint32_t skew = (uint32_t)(reinterpret_cast<uintptr_t>(t.bytes) & 15);
  const uint32_t lo = a + skew, hi = b + skew;  // byte range relative to base
  const uint32_t c_end = (hi + 15) >> 4;
  for (uint32_t c0 = lo >> 4; c0 < c_end; c0 += CH) {
    const uint32_t nch = min(CH, c_end - c0);
    for (uint32_t i = lane; i < nch; i += 32) buf[i] = __ldg(base + c0 + i);
    __syncwarp();
    if (lane == 0) {
      // one 16-B shared load per block, then its bytes in order from registers (the serial
      // multiply chain is the only latency left)
      for (uint32_t i = 0; i < nch; i++) {
        const uint4 v = buf[i];
        const uint32_t q[4] = {v.x, v.y, v.z, v.w};
        const uint32_t b0 = (c0 + i) * 16;
        if (b0 >= lo && b0 + 16 <= hi) {
#pragma unroll
          for (int k = 0; k < 16; k++) {
            h ^= (uint64_t)((q[k >> 2] >> (8 * (k & 3))) & 0xFFu);
            h *= 0x100000001b3ULL;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16; k++) {
            if (b0 + k >= lo && b0 + k < hi) {
              h ^= (uint64_t)((q[k >> 2] >> (8 * (k & 3))) & 0xFFu);
              h *= 0x100000001b3ULL;
            }
          }
        }
      }
    }
    __syncwarp();
  }
  return h;
}

// FNV-1a 64 of one string by one thread (the sample's representatives: a few per block)
__device__ __forceinline__ uint64_t thread_fnv_string(const fikit_strtab_t& t, uint32_t j) {
  uint64_t h = 0xcbf29ce484222325ULL;
  const uint32_t a = __ldg(t.offsets + j), b = __ldg(t.offsets + j + 1);
  if (b <= a) return h;  // (malformed: flagged by the hash role)
  const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<uintptr_t>(t.bytes) & ~uintptr_t(15));
  const uint32_t skew = (uint32_t)(reinterpret_cast<uintptr_t>(t.bytes) & 15);
  const uint32_t lo = a + skew, hi = b + skew;
  uint4 nx = __ldg(base + (lo >> 4));
  for (uint32_t c = lo >> 4; c < (hi + 15) >> 4; c++) {
    const uint4 v = nx;
    if (c + 1 < (hi + 15) >> 4) nx = __ldg(base + c + 1);  // next block in flight
    const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const uint32_t pos = c * 16 + k;
      if (pos >= lo && pos < hi) {
        h ^= (uint64_t)((q[k >> 2] >> (8 * (k & 3))) & 0xFFu);
        h *= 0x100000001b3ULL;
      }
    }
  }
  return h;
}

// One warp per string (blockIdx.y: 0 names, 1 signatures): identify / resolve
__global__ void __launch_bounds__(128) k_strtab_hash(fikit_strtab_t names, uint64_t* __restrict__ name_out,
                                                     fikit_strtab_t sigs, uint64_t* __restrict__ sig_out,
                                                     fikit_status_t* st) {
  pdl_entry();
  __shared__ uint4 buf[4][64];
  const bool is_name = blockIdx.y == 0;
  const fikit_strtab_t t = is_name ? names : sigs;
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t j = blockIdx.x * 4 + w;
  if (j >= t.count) return;
  const uint64_t h = warp_fnv_string(t, j, is_name, buf[w], lane, st);
  if (lane == 0) (is_name ? name_out : sig_out)[j] = h;
}

// warp-cooperative coalesced load of up to 32 records (1536 B) into a per-warp
// shared buffer; lane l then reads record l with three 16-B shared loads
__device__ __forceinline__ void warp_stage_records(const uint4* __restrict__ g, uint64_t first, uint32_t cnt,
                                                   uint4* sbuf, int lane) {
  const uint4* src = g + first * 3;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    uint32_t c = lane + 32 * k;
    if (c < cnt * 3) sbuf[c] = __ldcs(src + c);  // streaming: read once
  }
  __syncwarp();
}

__device__ __forceinline__ void read_rec_words(const uint4* sbuf, int j, uint32_t* w) {
  uint4 a = sbuf[j * 3 + 0], b = sbuf[j * 3 + 1], c = sbuf[j * 3 + 2];
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
}

// ---- identify: 48 B in, 8 B out per launch (HBM-bound streaming) ---------------------
__global__ void __launch_bounds__(256) k_identify(const uint4* __restrict__ recs, uint64_t n,
                                                  const uint64_t* __restrict__ name_hash,
                                                  const uint64_t* __restrict__ sig_hash, uint32_t n_names,
                                                  uint32_t n_sigs, uint64_t* __restrict__ out, fikit_status_t* st) {
  pdl_entry();
  __shared__ uint4 sbuf[8][96];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t nchunks = (n + 31) / 32;
  for (uint64_t c = (uint64_t)blockIdx.x * 8 + wid; c < nchunks; c += (uint64_t)gridDim.x * 8) {
    uint64_t first = c * 32;
    uint32_t cnt = (uint32_t)umin64(32, n - first);
    __syncwarp();
    warp_stage_records(recs, first, cnt, sbuf[wid], lane);
    if (lane < (int)cnt) {
      uint32_t w[12];
      read_rec_words(sbuf[wid], lane, w);
      uint64_t kid = 0;
      if (record_valid(w, n_names, n_sigs)) {
        kid = kernel_id_from(__ldg(name_hash + w[4]), __ldg(sig_hash + w[5]), w[6], w[7], w[8], w[9]);
      } else {
        flag_record(st, first + lane);
      }
      __stcs(out + first + lane, kid);
    }
  }
}

// ---- the measure call's preamble: two launches (k_prep, k_plan) ---------------------------------
// k_prep, one launch with three independent roles by block range (256 threads each):
//   hash    the FNV-1a hashes of every name and signature (one warp per string), used by the
//           cold path of k_measure;
//   sample  a jittered strided sample of ~64k launches -> (task, kernel ID) rows in the global
//           index with sample counts (picks the rows worth caching; the representatives hash
//           their strings themselves, so this role does not wait for the hash role);
//   group   the task bucket of every tile group (kGroupTiles warp-tiles = 256 launches, bucketed
//           by their first launch's task: one sector read per group) and per-block bucket counts
//           (the counting sort of the task-partitioned schedule).
// k_plan, one launch (1024 threads per block) with two roles:
//   hot     per task bucket (and one global set), the <= kHotMax most-sampled rows and the
//           sample coverage that decides the schedule mode;
//   scatter the stable counting-sort scatter of the tile groups by bucket (each block derives its
//           own offsets from every block's counts), and (block 0) the buckets' ranges and the
//           first bucket of every k_measure CTA.

__device__ __forceinline__ void prep_sample(const PrepArgs& a, uint32_t blk, uint32_t nblk, unsigned char* sm) {
  // The sample counts raw launch identities (no kernel IDs, no rows: k_plan resolves only the
  // identities it keeps).  Per-block deduplication first: the block's samples are counted per
  // distinct identity in shared memory (keyed by a 64-bit fingerprint), then one representative
  // per identity adds the count to the global sample table (one CAS claims a slot and publishes
  // its fingerprint; the identity words are read only by the next kernel).  A skewed sample hits
  // a few identities thousands of times; this keeps the global table to one access per distinct
  // identity per block.
  constexpr uint32_t HS = 1024;  // (<= 512 samples per block: load <= 1/2)
  unsigned long long* sfp = reinterpret_cast<unsigned long long*>(sm);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sfp + HS);
  uint32_t* stw = scnt + HS;  // [HS][7]
  uint32_t* snew = stw + 7 * HS;  // [2 * kPrepThreads] sample slots this block claimed, then a count
  uint32_t* snew_n = snew + 2 * kPrepThreads;
  for (uint32_t i = threadIdx.x; i < HS; i += blockDim.x) {
    sfp[i] = 0;
    scnt[i] = 0;
  }
  if (threadIdx.x == 0) *snew_n = 0;
  __syncthreads();
  auto global_add = [&](const uint32_t* tw, unsigned long long fp, uint32_t cnt) {
    uint32_t h = (uint32_t)(fp >> 20) & (kSampSlots - 1);
    for (uint32_t probe = 0; probe < 64; probe++, h = (h + 1) & (kSampSlots - 1)) {
      const unsigned long long old = atomicCAS(&a.samp[h].fp, 0ull, fp);
      if (old == 0ull) {
#pragma unroll
        for (int q = 0; q < 6; q++) a.samp[h].w[q] = tw[q];
        a.samp[h].task = tw[6];
        snew[atomicAdd(snew_n, 1u)] = h;  // (listed once per block below: no global counter per slot)
      }
      if (old == 0ull || old == fp) {
        atomicAdd(&a.samp[h].cnt, cnt);
        return;
      }
    }  // (a full neighbourhood: the sample is dropped)
  };
  const uint32_t nn = a.names.count, ns = a.sigs.count;
  for (uint64_t j = blk * (uint64_t)blockDim.x + threadIdx.x; j < a.n_samples; j += (uint64_t)nblk * blockDim.x) {
    // jittered stride: a fixed stride aliases with periodic traces (a 300-kernel template
    // sampled every 1525 launches sees only 12 of its positions); a hashed offset inside each
    // stride window covers every position
    const uint64_t i = j * a.stride + (a.stride > 1 ? mix64(j + 0x9E3779B97F4A7C15ULL) % a.stride : 0);
    if (i >= a.n) break;
    const uint4 x = __ldg(a.recs + i * 3), y = __ldg(a.recs + i * 3 + 1), z = __ldg(a.recs + i * 3 + 2);
    const uint32_t w[12] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w, z.x, z.y, z.z, z.w};
    if (!record_valid(w, nn, ns)) continue;  // reported by k_measure
    const uint32_t tw[7] = {w[4], w[5], w[6], w[7], w[8], w[9] & 0xFFFFu, w[11]};
    const uint32_t h1 = tuple_hash(tw);
    const unsigned long long fp = (((unsigned long long)h1 << 32) | (mix64(((uint64_t)tw[0] << 32 | tw[1]) ^
                                   ((uint64_t)tw[2] << 32 | tw[3]) * 0x9E3779B97F4A7C15ULL ^
                                   ((uint64_t)tw[4] << 32 | tw[5]) * 0xC2B2AE3D27D4EB4FULL ^ tw[6]) >> 32)) | 1ull;
    uint32_t p = h1 & (HS - 1);
    bool counted = false;
    for (uint32_t probe = 0; probe < HS; probe++, p = (p + 1) & (HS - 1)) {
      const unsigned long long old = atomicCAS(&sfp[p], 0ull, fp);
      if (old == 0ull) {  // first sample of this identity in the block: the representative
#pragma unroll
        for (int q = 0; q < 7; q++) stw[p * 7 + q] = tw[q];
      }
      if (old == 0ull || old == fp) {
        atomicAdd(&scnt[p], 1u);
        counted = true;
        break;
      }
    }
    if (!counted) global_add(tw, fp, 1u);  // the block saw > HS identities: count it directly
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < HS; q += blockDim.x)
    if (scnt[q]) global_add(stw + q * 7, sfp[q], scnt[q]);
  // the block's new slots join the dense list with one global atomic
  __syncthreads();
  const uint32_t nnew = *snew_n;
  __shared__ uint32_t s_base;
  if (threadIdx.x == 0 && nnew) s_base = atomicAdd(a.samp_n, nnew);
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < nnew; q += blockDim.x) a.samp_list[s_base + q] = snew[q];
}

__device__ __forceinline__ void prep_groups(const PrepArgs& a, uint32_t blk, uint32_t* h) {
  for (int i = threadIdx.x; i < (int)kBuckets; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t C = (a.ngroups + a.sb - 1) / a.sb;
  const uint32_t g0 = blk * C, g1 = min(a.ngroups, g0 + C);
  constexpr int U = 4;  // independent one-sector loads in flight per thread
  for (uint32_t q = g0 + threadIdx.x; q < g1; q += U * blockDim.x) {
    uint32_t task[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t qu = q + u * blockDim.x;
      task[u] = qu < g1 ? __ldcs(&a.recs_t[(uint64_t)qu * kGroupTiles * kTileLaunches].task_id) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t qu = q + u * blockDim.x;
      if (qu < g1) {
        const uint32_t b = bucket_of(task[u]);
        a.grp_bucket[qu] = (uint8_t)b;
        atomicAdd(&h[b], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)kBuckets; i += blockDim.x) a.blkcnt[blk * kBuckets + i] = h[i];
}

__global__ void __launch_bounds__(kPrepThreads) k_prep(PrepArgs a) {
  pdl_entry();
  __shared__ __align__(16) unsigned char sm[1024 * 8 + 1024 * 4 + 1024 * 28 + 2 * kPrepThreads * 4 + 4];  // sample role's
  const uint32_t b = blockIdx.x;
  FK_TR(if (threadIdx.x == 0) { FK_TP(0); g_trace_pre[blockIdx.x * 8 + 7] = b < a.nb_hash ? 1 : b < a.nb_hash + a.nb_samp ? 2 : 3; })
  FK_TR(struct TrEnd { __device__ ~TrEnd() { __syncthreads(); if (threadIdx.x == 0) FK_TP(1); } } tr_end;)
  if (b < a.nb_hash) {  // names, then signatures: one warp per string
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t j = b * (kPrepThreads / 32) + w;
    const uint32_t nn = a.names.count;
    if (j < nn + a.sigs.count) {
      const bool is_name = j < nn;
      const uint64_t h = warp_fnv_string(is_name ? a.names : a.sigs, is_name ? j : j - nn, is_name,
                                         reinterpret_cast<uint4*>(sm) + w * 64, lane, a.st);
      if (lane == 0) (is_name ? a.name_hash[j] : a.sig_hash[j - nn]) = h;
    }
  } else if (b < a.nb_hash + a.nb_samp) {
    prep_sample(a, b - a.nb_hash, a.nb_samp, sm);
  } else {
    // a reused plan in address-order mode needs no task buckets (k_measure sweeps the tiles in order)
    if (a.reused_plan && !use_task_buckets(a.hot_hdr)) return;
    prep_groups(a, b - a.nb_hash - a.nb_samp, reinterpret_cast<uint32_t*>(sm));
  }
}


// hot sets: per task bucket, the most-sampled identities (block bkt; block kBuckets: the global
// set over all tasks), each resolved to its row (kernel ID from the string hashes k_prep wrote,
// then the KID index: find or insert).  Each block also counts the samples its set covers.
__device__ __forceinline__ void plan_hot(const PlanArgs& a, uint32_t bkt, unsigned char* sm) {
  constexpr int NB = 4096;
  uint32_t* h = reinterpret_cast<uint32_t*>(sm);
  uint32_t* wsum = h + NB;  // [32]
  uint32_t* s_misc = wsum + 32;  // chosen, hot n, T, claims, first claimed row
  Tuple* hot = a.hot_all + (size_t)bkt * kHotMax;
  auto mine = [&](uint32_t task) { return bkt == kGlobalSet || bucket_of(task) == bkt; };
  const uint32_t nd = min(a.hot_hdr[kSampN], kSampSlots);  // distinct sampled identities
  FK_TR(if (threadIdx.x == 0) { FK_TQ(0); g_trace_pre[(1024 + blockIdx.x) * 8 + 7] = 10; })
  for (int i = threadIdx.x; i < NB; i += blockDim.x) h[i] = 0;
  __syncthreads();
  // (count, task) of 4 listed identities per thread in flight; the loop bound is warp-uniform
  // (the histogram update below is a full-warp match).  The first two rounds stay in registers
  // for the selection pass (no second read of the list for nd <= 8192).
  constexpr uint32_t U = 4;
  const uint32_t lane_id = threadIdx.x & 31u;
  uint32_t e0[U], e1[U];
  uint2 c0[U], c1[U];
  auto load_round = [&](uint32_t i0, uint32_t* ent, uint2* ct) {
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint32_t i = i0 + u * blockDim.x;
      ent[u] = i < nd ? __ldg(a.samp_list + i) : 0u;
    }
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint32_t i = i0 + u * blockDim.x;
      ct[u] = i < nd ? *reinterpret_cast<const uint2*>(a.samp + ent[u]) : make_uint2(0u, 0u);
    }
  };
  auto count_round = [&](const uint2* ct) {
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {  // warp-aggregated: skewed samples give many equal counts
      const bool in = ct[u].x && mine(ct[u].y);
      const uint32_t bin = in ? min(ct[u].x, (uint32_t)NB - 1) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (in && (peers & ((1u << lane_id) - 1u)) == 0) atomicAdd(&h[bin], (uint32_t)__popc(peers));
    }
  };
  {
    uint32_t r = 0;
    for (uint32_t i0 = threadIdx.x; i0 - lane_id < nd; i0 += U * blockDim.x, r++) {
      if (r == 0) {
        load_round(i0, e0, c0);
        count_round(c0);
      } else if (r == 1) {
        load_round(i0, e1, c1);
        count_round(c1);
      } else {
        uint32_t ent[U];
        uint2 ct[U];
        load_round(i0, ent, ct);
        count_round(ct);
      }
    }
  }
  if (threadIdx.x == 0) {
    s_misc[0] = 0;
    s_misc[1] = 0;
    s_misc[2] = NB;
  }
  __syncthreads();
  // T = smallest count c >= 1 whose suffix S(c) = #identities with count >= c fits kHotMax:
  // a block-wide suffix scan of the 4096-bin count histogram (4 bins per thread)
  {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    uint32_t loc[4], x = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      loc[j] = h[4 * t + j];
      x += loc[j];
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_down_sync(0xffffffffu, x, d);
      if (lane + d < 32) x += y;
    }
    if (lane == 0) wsum[wid] = x;
    __syncthreads();
    uint32_t later = 0;
    for (int w2 = wid + 1; w2 < 32; w2++) later += wsum[w2];
    uint32_t S = x + later;  // suffix from bin 4t
#pragma unroll
    for (int j = 0; j < 4; j++) {
      uint32_t c = 4 * t + j;
      if (c >= 1 && S <= kHotMax) atomicMin(&s_misc[2], c);
      S -= loc[j];
    }
    __syncthreads();
  }
  const uint32_t T = s_misc[2];
  FK_TR(if (threadIdx.x == 0) FK_TQ(2);)
  uint32_t* chosen = h;  // (the histogram is no longer needed) [kHotMax] sample slots
  uint32_t tot = 0;
  auto choose_round = [&](const uint32_t* ent, const uint2* ct) {
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint32_t c = ct[u].x;
      if (c == 0 || !mine(ct[u].y)) continue;
      tot += c;
      if (c >= T) {
        const uint32_t e = atomicAdd(&s_misc[0], 1u);
        if (e < kHotMax) chosen[e] = ent[u];
      }
    }
  };
  {
    uint32_t r = 0;
    for (uint32_t i0 = threadIdx.x; i0 - lane_id < nd; i0 += U * blockDim.x, r++) {
      if (r == 0) {
        choose_round(e0, c0);
      } else if (r == 1) {
        choose_round(e1, c1);
      } else {
        uint32_t ent[U];
        uint2 ct[U];
        load_round(i0, ent, ct);
        choose_round(ent, ct);
      }
    }
  }
  __syncthreads();
  FK_TR(if (threadIdx.x == 0) FK_TQ(3);)
  // Resolve the chosen identities to rows, one per thread (nc <= kHotMax < blockDim.x), the new
  // rows allocated with ONE global atomic per block: (1) probe the KID index, claiming an empty
  // slot by CAS without waiting on anyone (a slot another thread is writing: pending); (2) the
  // block counts its claims, one thread reserves their rows; (3) the claimers publish (release
  // store); (4) pending threads finish with the ordinary find-or-insert, whose waits can only be
  // on other blocks' claimers, which never wait.  (One row counter hit by every new row had
  // serialised ~8k L2 atomics.)
  const uint32_t nc = min(s_misc[0], kHotMax);
  uint32_t* s_claims = s_misc + 3;  // claims of this block; s_misc[4]: first reserved row
  if (threadIdx.x == 0) *s_claims = 0;
  __syncthreads();
  const uint32_t q = threadIdx.x;
  Tuple t;
  uint64_t kid = 0;
  uint32_t cnt = 0, slot = 0, mine_n = 0;
  int state = -1;  // -1 none, 0 row known, 1 claimed slot, 2 pending
  if (q < nc) {
    const SampEntry& se = a.samp[chosen[q]];
    const uint2 ct = *reinterpret_cast<const uint2*>(&se);
#pragma unroll
    for (int w = 0; w < 6; w++) t.w[w] = se.w[w];
    t.w[6] = ct.y;
    cnt = ct.x;
    kid = kernel_id_from(__ldg(a.name_hash + t.w[0]), __ldg(a.sig_hash + t.w[1]), t.w[2], t.w[3], t.w[4], t.w[5]);
    uint32_t h = key_hash(kid, t.w[6]) & (a.slots - 1);
    state = 2;
    for (uint32_t probe = 0; probe < a.slots; probe++, h = (h + 1) & (a.slots - 1)) {
      uint4 v = ld_relaxed_v4(&a.idx[h]);
      uint32_t st_w = v.w;
      if (st_w == 0u) {
        if (a.dict) {  // dictionary mode: an absent key has no row
          t.row = FIKIT_NO_ROW;
          state = 0;
          break;
        }
        st_w = atomicCAS(&a.idx[h].state, 0u, kBusy);
        if (st_w == 0u) {
          a.idx[h].kid = kid;
          a.idx[h].task = t.w[6];
          slot = h;
          state = 1;
          mine_n = atomicAdd(s_claims, 1u);
          break;
        }
        v = ld_relaxed_v4(&a.idx[h]);
      }
      if (st_w == kBusy) break;  // pending: resolved after this block's claims are published
      if ((((uint64_t)v.y << 32) | v.x) == kid && v.z == t.w[6]) {
        t.row = st_w - 1;
        state = 0;
        break;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && *s_claims) s_misc[4] = (uint32_t)atomicAdd((unsigned long long*)&a.st->n_rows_needed,
                                                                   (unsigned long long)*s_claims);
  __syncthreads();
  if (state == 1) {  // publish: the row's key, a representative tuple, then the slot
    t.row = s_misc[4] + mine_n;
    if (t.row < a.cap) {
      a.raw[t.row].kid = kid;
      a.raw[t.row].task = t.w[6];
      a.row_tuple[t.row] = t;
    } else {
      atomicOr(&a.st->flags, kStatusCapacity);
    }
    st_release_u32(&a.idx[slot].state, t.row + 1);
  } else if (state == 2) {
    t.row = index_find_or_insert(a.idx, a.slots, kid, t.w[6], t.w, a.st, a.raw, a.row_tuple, a.cap, a.dict == 0u);
  }
  uint32_t cov = 0;
  if (state >= 0 && t.row < a.cap) {  // (E_CAPACITY is flagged; the row is not materialised)
    const uint32_t e = atomicAdd(&s_misc[1], 1u);
    hot[e] = t;
    cov = cnt;
  }
  cov = __reduce_add_sync(0xffffffffu, cov);
  tot = __reduce_add_sync(0xffffffffu, tot);
  if ((threadIdx.x & 31) == 0) {
    if (cov) atomicAdd(&a.hot_hdr[bkt == kGlobalSet ? kCovGlobal : kCovTask], cov);
    if (tot && bkt == kGlobalSet) atomicAdd(&a.hot_hdr[kCovTotal], tot);
  }
  __syncthreads();
  if (threadIdx.x == 0) a.hot_hdr[bkt] = min(s_misc[1], kHotMax);
  FK_TR(if (threadIdx.x == 0) FK_TQ(4);)
}

// stable counting-sort scatter of block k's chunk of tile groups: its offsets are the buckets'
// starts plus the counts of the chunks before it (every block reads every block's counts); the
// chunk is walked in address order 1024 groups per step, a group's position = its bucket's
// running cursor + same-bucket groups of lower warps in the step + same-bucket lanes below it
// (match_any).  Groups of a bucket keep address order.  Block 0 also publishes the buckets'
// ranges and assigns every k_measure CTA its first bucket.
__device__ __forceinline__ void plan_scatter(const PlanArgs& a, uint32_t k, unsigned char* sm) {
  constexpr uint32_t SEGS = 16, W = 32;
  uint32_t* ptot = reinterpret_cast<uint32_t*>(sm);  // [SEGS][kBuckets]
  uint32_t* ppre = ptot + SEGS * kBuckets;           // [SEGS][kBuckets]
  uint32_t* cur = ppre + SEGS * kBuckets;            // [kBuckets]
  uint32_t* tot = cur + kBuckets;                    // [kBuckets]
  uint32_t* wcnt = tot + kBuckets;                   // [W][kBuckets]
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {  // thread (seg, b): counts of bucket b over a segment of the blocks, all of them and those before k
    const uint32_t b = tid % kBuckets, seg = tid / kBuckets;
    const uint32_t per = (a.sb + SEGS - 1) / SEGS, k0 = seg * per, k1 = min(a.sb, k0 + per);
    uint32_t x = 0, y = 0;
    for (uint32_t kk = k0; kk < k1; kk++) {
      const uint32_t c = a.blkcnt[kk * kBuckets + b];
      x += c;
      y += kk < k ? c : 0u;
    }
    ptot[seg * kBuckets + b] = x;
    ppre[seg * kBuckets + b] = y;
  }
  for (uint32_t i = tid; i < W * kBuckets; i += blockDim.x) wcnt[i] = 0;
  __syncthreads();
  if (tid < kBuckets) {
    uint32_t x = 0, y = 0;
#pragma unroll
    for (uint32_t seg = 0; seg < SEGS; seg++) {
      x += ptot[seg * kBuckets + tid];
      y += ppre[seg * kBuckets + tid];
    }
    tot[tid] = x;
    cur[tid] = y;  // (+ the bucket's start, below)
  }
  __syncthreads();
  if (warp == 0) {  // bucket starts: exclusive scan of the totals (2 buckets per lane)
    const uint32_t c0 = tot[2 * lane], c1 = tot[2 * lane + 1];
    uint32_t x = c0 + c1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= (uint32_t)d) x += y;
    }
    const uint32_t s0 = x - c0 - c1;
    cur[2 * lane] += s0;
    cur[2 * lane + 1] += s0 + c0;
    if (k == 0) {
      a.bstart[2 * lane] = s0;
      a.bstart[2 * lane + 1] = s0 + c0;
      a.btot[2 * lane] = c0;
      a.btot[2 * lane + 1] = c1;
      // first bucket of every CTA: g_b = ceil(c_b / L) CTAs for the smallest per-CTA load L with
      // sum_b g_b <= G (at least one CTA per non-empty bucket when nb <= G; else every CTA
      // starts on its own bucket); unassigned CTAs start by stealing (kNoBucket)
      const uint32_t G = a.grid_measure;
      const uint32_t nb = __reduce_add_sync(0xffffffffu, (c0 ? 1u : 0u) + (c1 ? 1u : 0u));
      const uint32_t ng = __shfl_sync(0xffffffffu, x, 31);  // all groups
      uint32_t g0, g1;
      if (nb <= G) {
        uint32_t lo = (ng + G - 1) / G, hi = ng > 0 ? ng : 1;
        if (lo < 1) lo = 1;
        while (lo < hi) {
          const uint32_t mid = lo + (hi - lo) / 2;
          const uint32_t need = __reduce_add_sync(0xffffffffu, (c0 + mid - 1) / mid + (c1 + mid - 1) / mid);
          if (need <= G) hi = mid; else lo = mid + 1;
        }
        g0 = (c0 + lo - 1) / lo;
        g1 = (c1 + lo - 1) / lo;
      } else {
        g0 = c0 ? 1u : 0u;
        g1 = c1 ? 1u : 0u;
      }
      uint32_t gx = g0 + g1;  // CTA ranges: exclusive scan of g
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, gx, d);
        if (lane >= (uint32_t)d) gx += y;
      }
      const uint32_t cs = gx - g0 - g1;
      for (uint32_t c = lane; c < G; c += 32) a.first[c] = kNoBucket;
      __syncwarp();
      for (uint32_t i = 0; i < g0 && cs + i < G; i++) a.first[cs + i] = 2 * lane;
      for (uint32_t i = 0; i < g1 && cs + g0 + i < G; i++) a.first[cs + g0 + i] = 2 * lane + 1;
    }
  }
  __syncthreads();
  const uint32_t C = (a.ngroups + a.sb - 1) / a.sb;
  const uint32_t t0 = k * C, t1 = min(a.ngroups, t0 + C);
  auto ldb = [&](uint32_t t) -> uint32_t { return t < t1 ? (uint32_t)a.grp_bucket[t] : kBuckets; };
  uint32_t bnext = ldb(t0 + tid);  // software-pipelined one step ahead
  for (uint32_t base = t0; base < t1; base += blockDim.x) {
    const uint32_t t = base + tid;
    const uint32_t b = bnext;  // kBuckets: no group (tail)
    bnext = ldb(t + blockDim.x);
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (b < kBuckets && rank == 0) wcnt[warp * kBuckets + b] = __popc(peers);
    __syncthreads();
    if (b < kBuckets) {
      uint32_t pos = cur[b] + rank;
      for (uint32_t v = 0; v < warp; v++) pos += wcnt[v * kBuckets + b];
      FK_CHECK(pos < a.ngroups && t < a.ngroups);
      a.order[pos] = t;
    }
    __syncthreads();
    if (tid < kBuckets) {
      uint32_t add = 0;
#pragma unroll
      for (uint32_t v = 0; v < W; v++) {
        add += wcnt[v * kBuckets + tid];
        wcnt[v * kBuckets + tid] = 0;
      }
      cur[tid] += add;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_plan(PlanArgs a) {
  pdl_entry();
  __shared__ __align__(16) unsigned char sm[(4096 + 32 + 8) * 4 > (2 * 16 + 2 + 32) * kBuckets * 4
                                                ? (4096 + 32 + 8) * 4
                                                : (2 * 16 + 2 + 32) * kBuckets * 4];
  unsigned long long* stamp = reinterpret_cast<unsigned long long*>(a.hot_hdr + kPlanStamp);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (a.hot_blocks) {  // a new plan: stamp it with this call's dictionary (0: no dictionary)
      *stamp = a.dict ? *a.dict_hash : 0ull;
    } else if (*stamp == 0ull || *stamp != *a.dict_hash) {  // reused plan of another dictionary
      atomicOr(&a.st->flags, kStatusArg);
    }
  }
  if (blockIdx.x < a.hot_blocks) {
    plan_hot(a, blockIdx.x, sm);
  } else {
    FK_TR(if (threadIdx.x == 0) { FK_TQ(0); g_trace_pre[(1024 + blockIdx.x) * 8 + 7] = 11; })
    if (a.hot_blocks == 0 && !use_task_buckets(a.hot_hdr)) return;  // (a reused address-order plan)
    plan_scatter(a, blockIdx.x - a.hot_blocks, sm);
    FK_TR(if (threadIdx.x == 0) FK_TQ(4);)
  }
}

// ---- the fused identify + measure kernel ----------------------------------------------------
namespace mk {
constexpr int TILE = 32;                  // launches per half-tile (one per lane)
constexpr int CH = 2 * TILE;              // launches per warp-tile: one TMA, one wait, two per lane
static_assert(CH == (int)kTileLaunches, "the schedule's tile is the kernel's warp-tile");
constexpr int WARPS = 24;                 // warps per CTA; every warp streams and consumes its own tiles (<= 85 registers)
constexpr int CONSUMERS = WARPS * 32;
constexpr int THREADS = CONSUMERS;
constexpr uint32_t TAG_W = 2;             // one-word tags per bucket (one 8-B load per probe)
constexpr uint32_t TAG_Q = 4096 / TAG_W;  // buckets (4096 tags, load <= 0.16)
constexpr uint32_t TAG_HB = 0xFFFFF800u;  // tag = hash bits 11..31 (bit 31 forced to 1) | (slot + 1)
static_assert(kHotMax < 2048, "slot + 1 must fit the 11 tag bits");
constexpr int STAGE_BYTES = (CH + 1) * 48;  // the tile + the next launch (the tile's last gap)

struct Smem {
  uint4 ring[WARPS][STAGE_BYTES / 16];  // one stage per warp (refilled as soon as it is read)
  uint64_t full[WARPS];
  // Bucket q = hash % TAG_Q holds up to TAG_W tags, filled in order (the filled tags are a
  // prefix); a full bucket continues in the next one.  0 = empty.
  alignas(16) uint32_t tagw[TAG_Q * TAG_W];
  // slot -> identity in 5 words: name | sig << 16, grid_x, grid_y | grid_z << 16,
  // block_x | block_y << 16, block_z | task << 16 (one 16-B + one 4-B load verify).  Only
  // identities with name, sig, task < 2^16 are kept hot; the others always take the cold path.
  // Indexed by slot + 1 (the tag's low bits): entry 0 is never admitted, so the speculative
  // verification of a launch without a matching tag reads it without a race.
  uint4 tq[kHotMax + 1];
  uint32_t tq4[kHotMax + 1];
  // Odd row strides (33 and 9 words) spread the slots of a warp over all 32 banks.
  uint32_t hist[kHotMax][2 * kBins + 1];  // 64 u32 bins (32 duration, 32 gap) (+1 pad)
  uint32_t st[kHotMax][5];        // duration: 0 sum mod 2^32, 1 carries out of it; gap: 2, 3 (v < 2^32); 4: pad
  uint4 mm[kHotMax];              // min, max (u32) of duration, then of gap (values < 2^32): one 16-B load
  uint32_t grow[kHotMax];         // slot -> global row
  uint32_t hot_n;
  uint32_t next_bucket;
  unsigned long long overlap;
};
static_assert(sizeof(Smem) <= 227 * 1024, "shared memory budget (227 KB per CTA)");
static_assert(THREADS <= 1024, "a CTA has at most 1024 threads");
// Each warp owns its stage and is its only producer and consumer, so the stage's mbarrier
// phase can never be waited on two uses ahead (no parity aliasing) and no slow warp can
// stall another warp's prefetch.
}  // namespace mk

// fire-and-forget reductions (no return value, no dependent latency)
__device__ __forceinline__ void red_shared_add(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_shared_min(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_shared_max(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
// predicated forms (no branch, no reconvergence point): the reduction happens where p holds
__device__ __forceinline__ void red_shared_add_if(bool p, uint32_t saddr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.add.u32 [%1], %2;\n\t}" ::"r"((uint32_t)p),
               "r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_shared_min_if(bool p, uint32_t saddr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.min.u32 [%1], %2;\n\t}" ::"r"((uint32_t)p),
               "r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_shared_max_if(bool p, uint32_t saddr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.max.u32 [%1], %2;\n\t}" ::"r"((uint32_t)p),
               "r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// one duration (j = 0) or gap (j = 1, on: the launch has a gap) value of a hot row, without
// branches for values < 2^32.  Histogram and split sums are fire-and-forget shared reductions;
// min/max are read first (a broadcast when several lanes hit the same row) and reduced only when
// the value improves them.  Values >= 2^32 ns (4.3 s, rare) go straight to the table.
__device__ __forceinline__ uint32_t atom_shared_add(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}

// mn, mx: the slot's current min / max for j, loaded before any of the launch's reductions.
// The sum of values < 2^32 is kept mod 2^32 with a carry counter: the add returns the old
// word and a wrap (old + v < old, exact: the atomic serializes) adds one carry.  Returns the
// old word (the caller checks the carry after its other reductions, off the critical path).
// The split sum gets a (v, or 0 when off or >= 2^32: every lane adds, the old word is returned
// for the carry check, which the caller makes after its other reductions).
// kSmall: the caller checked v < 2^32 for the whole warp (no per-value check, no >= 2^32 path).
template <bool kSmall, class RowOf>  // row_of(): the slot's table row, read only on the rare >= 2^32 path
__device__ __forceinline__ uint32_t hot_add(uint32_t hist_e, uint32_t st_e, uint32_t mm_e, const RawTab& tab,
                                            RowOf row_of, int j, uint64_t v, bool on, uint32_t mn, uint32_t mx,
                                            uint32_t& a) {
  const bool small = kSmall || (v >> 32) == 0;
  const uint32_t v32 = (uint32_t)v;
  // bin_of(v) = min(bit_length(v), 31)
  const uint32_t b = (small ? 32u - (uint32_t)__clz(min(v32, 0x7FFFFFFFu)) : 31u) + 32u * j;
  const bool son = on && small;
  a = son ? v32 : 0u;
  const uint32_t old = atom_shared_add(st_e + 8u * j, a);
  red_shared_add_if(on, hist_e + 4u * b, 1u);
  red_shared_min_if(son && v32 < mn, mm_e + 8u * j, v32);
  red_shared_max_if(son && v32 > mx, mm_e + 8u * j + 4u, v32);
  if (!kSmall && on && !small) {  // rare: a value >= 2^32 ns
    const uint32_t row = row_of();
    red_add_u64(tab.rows[row].sums + 2 * j + 1, v);
    red_max_u64(tab.rows[row].ext + 2 * j, v);
    red_max_u64(tab.rows[row].ext + 2 * j + 1, ~v);
  }
  return old;
}

__device__ __forceinline__ void cold_add(const RawTab& tab, uint32_t row, int j, uint64_t v) {
  // fire-and-forget L2 reductions (no read-back, no dependent latency)
  red_add_u32(tab.rows[row].hist + 32 * j + bin_of(v), 1u);
  red_add_u64(tab.rows[row].sums + 2 * j + 1, v);
  red_max_u64(tab.rows[row].ext + 2 * j, v);
  red_max_u64(tab.rows[row].ext + 2 * j + 1, ~v);
}

// phase flush of the shared rows: u32 bins and split sums -> table, zeroed
__device__ __forceinline__ void flush_epoch(mk::Smem& S, const RawTab& tab, int ctid) {
  // one warp per slot: 64 u32 bins (two per lane) and the two split sums (lanes 0, 1)
  const uint32_t hn = min(S.hot_n, kHotMax);  // admission may overshoot the counter
  const uint32_t lane = (uint32_t)ctid & 31u;
  for (uint32_t e = (uint32_t)ctid >> 5; e < hn; e += mk::WARPS) {
    const uint32_t row = S.grow[e];
    uint32_t* gh = tab.rows[row].hist;
#pragma unroll
    for (uint32_t w = lane; w < 2u * kBins; w += 32u) {
      const uint32_t x = S.hist[e][w];
      if (x) {
        red_add_u32(gh + w, x);
        S.hist[e][w] = 0;
      }
    }
    if (lane < 2) {
      const uint32_t j = lane;
      const uint64_t sum = (uint64_t)S.st[e][2 * j] | ((uint64_t)S.st[e][2 * j + 1] << 32);
      if (sum) red_add_u64(tab.rows[row].sums + 2 * j + 1, sum);
      S.st[e][2 * j] = 0;
      S.st[e][2 * j + 1] = 0;
    }
  }
}

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(mk::CONSUMERS) : "memory"); }

namespace mk {
__device__ __forceinline__ uint32_t tag_bits(uint32_t h) { return (h & TAG_HB) | 0x80000000u; }
// hash of a hot identity's five compressed words (tq, tq4 below): five multiply-adds and a short
// finaliser (the bucket takes the low 11 bits, the tag bits 11..30); collisions only cost a probe
__device__ __forceinline__ uint32_t hot_hash(uint32_t c0, uint32_t k2, uint32_t k3, uint32_t k4, uint32_t c4) {
  // a sum of odd-constant products (one IMAD each) and a short finaliser
  uint32_t h = c0 * 0x9E3779B1u + k2 * 0x85EBCA77u + k3 * 0xC2B2AE3Du + k4 * 0x27D4EB2Fu + c4 * 0x165667B1u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  return h;
}
// slot + 1 of the first tag of bucket t whose hash bits are hb's, 0 if none (an empty tag never
// matches: hb has bit 31 set)
__device__ __forceinline__ uint32_t bucket_match(const uint4 t, uint32_t hb) {
  uint32_t c = 0;
  if ((t.w ^ hb) < 0x800u) c = t.w;
  if ((t.z ^ hb) < 0x800u) c = t.z;
  if ((t.y ^ hb) < 0x800u) c = t.y;
  if ((t.x ^ hb) < 0x800u) c = t.x;
  return c & 0x7FFu;
}
// publish slot e under hash h (its tup words are written and fenced before)
__device__ __forceinline__ void tag_insert(Smem& S, uint32_t h, uint32_t e) {
  const uint32_t tg = tag_bits(h) | (e + 1);
  for (uint32_t q = h & (TAG_Q - 1);; q = (q + 1) & (TAG_Q - 1))
#pragma unroll
    for (uint32_t i = 0; i < TAG_W; i++)
      if (atomicCAS(&S.tagw[q * TAG_W + i], 0u, tg) == 0u) return;
}
// Dynamic admission without duplicates: reserve a tag word for hash h with slot field 0 ("pending":
// bucket_match reads it as no match, so readers take the exact cold path), then allocate the slot,
// write its identity and row, fence, and publish the slot in the reserved word.  A tag with the same
// hash bits met on the way means the identity is already admitted or being admitted by another
// warp (or, rarely, a 20-bit collision: that identity then stays cold, which is also exact): no
// second slot.  Returns without admitting when the slot pool is full (the reservation stays
// pending: a tag that never verifies).
__device__ __forceinline__ void admit(Smem& S, uint32_t h, uint32_t row, uint4 tq, uint32_t tq4) {
  const uint32_t hb = tag_bits(h);
  for (uint32_t q = h & (TAG_Q - 1);; q = (q + 1) & (TAG_Q - 1))
#pragma unroll
    for (uint32_t i = 0; i < TAG_W; i++) {
      uint32_t* w = &S.tagw[q * TAG_W + i];
      uint32_t old = *(volatile uint32_t*)w;
      if (old == 0u) old = atomicCAS(w, 0u, hb);
      if (old == 0u) {  // reserved
        const uint32_t e = atomicAdd(&S.hot_n, 1u);
        if (e >= kHotMax) return;
        S.grow[e] = row;
        S.tq[e + 1] = tq;
        S.tq4[e + 1] = tq4;
        __threadfence_block();
        atomicExch(w, hb | (e + 1));
        return;
      }
      if ((old ^ hb) < 0x800u) return;  // admitted (or pending) already
    }
}
// bucket q as up to 4 tags (missing ones 0); full: its last tag is taken
__device__ __forceinline__ uint4 ld_bucket(const Smem& S, uint32_t q) {
  if constexpr (TAG_W == 4) return reinterpret_cast<const uint4*>(S.tagw)[q];
  const uint2 t = reinterpret_cast<const uint2*>(S.tagw)[q];
  return make_uint4(t.x, t.y, 0u, 0u);
}
__device__ __forceinline__ bool bucket_full(const uint4 t) { return (TAG_W == 4 ? t.w : t.y) != 0u; }
}  // namespace mk

__global__ void __launch_bounds__(mk::THREADS, 1)
    k_measure(const fikit_record_t* __restrict__ recs, uint64_t n, const fikit_record_t* __restrict__ halo,
              const uint64_t* __restrict__ name_hash, const uint64_t* __restrict__ sig_hash, uint32_t n_names,
              uint32_t n_sigs, IndexEntry* idx, uint32_t slots, Tuple* tidx, uint32_t tslots, fikit_status_t* st,
              RawTab tab, Tuple* row_tuple, const Tuple* __restrict__ hot_all,
              const uint32_t* __restrict__ hot_n_all, uint32_t* cur, uint32_t* act, const uint32_t* __restrict__ bstart,
              const uint32_t* __restrict__ btot, const uint32_t* __restrict__ first,
              const uint32_t* __restrict__ order, const uint8_t* __restrict__ grp_bucket, uint32_t ntiles,
              uint32_t* __restrict__ out_row, uint32_t dict) {
  pdl_entry();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  mk::Smem& S = *reinterpret_cast<mk::Smem*>(smem_raw);
  const uint32_t sbase = smem_u32(smem_raw);
  const uint32_t s_hist = sbase + (uint32_t)offsetof(mk::Smem, hist);
  const uint32_t s_st = sbase + (uint32_t)offsetof(mk::Smem, st);
  const uint32_t s_mm = sbase + (uint32_t)offsetof(mk::Smem, mm);
  const uint32_t s_full = sbase + (uint32_t)offsetof(mk::Smem, full);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    S.overlap = 0;
    for (int i = 0; i < mk::WARPS; i++) mbar_init(&S.full[i], 1);
    fence_mbar_init();
    FK_TR_SET(0, gtime());
  }
  FK_TR(__shared__ unsigned long long tr_first_done; uint32_t tr_tiles = 0; unsigned long long tr_t0 = 0;)
  // load the hot set of a task bucket into the shared dictionary, zero the statistics
  auto load_hot_set = [&](uint32_t bkt) {
    const Tuple* hot = hot_all + (size_t)bkt * kHotMax;
    if (tid == 0) {
      S.hot_n = min(hot_n_all[bkt], kHotMax);
      S.tq[0] = make_uint4(0u, 0u, 0u, 0u);
      S.tq4[0] = 0u;
    }
    for (int i = tid; i < (int)(mk::TAG_Q * mk::TAG_W); i += mk::THREADS) S.tagw[i] = 0u;
    for (int i = tid; i < kHotMax * (2 * kBins + 1); i += mk::THREADS) (&S.hist[0][0])[i] = 0;
    for (int i = tid; i < kHotMax * 5; i += mk::THREADS) (&S.st[0][0])[i] = 0u;
    for (int i = tid; i < kHotMax; i += mk::THREADS) S.mm[i] = make_uint4(0xFFFFFFFFu, 0u, 0xFFFFFFFFu, 0u);
    __syncthreads();
    const uint32_t hn = S.hot_n;
    for (uint32_t e = tid; e < hn; e += mk::THREADS) {
      Tuple t = hot[e];
      S.grow[e] = t.row;
      if (((t.w[0] | t.w[1] | t.w[6]) >> 16) == 0u) {  // compressible: may be hot
        const uint32_t c0 = t.w[0] | (t.w[1] << 16), c4 = t.w[5] | (t.w[6] << 16);
        S.tq[e + 1] = make_uint4(c0, t.w[2], t.w[3], t.w[4]);
        S.tq4[e + 1] = c4;
        mk::tag_insert(S, mk::hot_hash(c0, t.w[2], t.w[3], t.w[4], c4), e);
      }
    }
    __syncthreads();
  };
  // min / max of the shared rows into the table (end of a phase, after flush_epoch)
  auto flush_hot_set_ext = [&]() {
    for (uint32_t e = tid, hn = min(S.hot_n, kHotMax); e < hn; e += mk::CONSUMERS) {
      const uint32_t row = S.grow[e];
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const uint32_t mn = j ? S.mm[e].z : S.mm[e].x, mx = j ? S.mm[e].w : S.mm[e].y;
        if (mn != 0xFFFFFFFFu || mx != 0u) {  // a value < 2^32 was seen
          red_max_u64(tab.rows[row].ext + 2 * j, (uint64_t)mx);
          red_max_u64(tab.rows[row].ext + 2 * j + 1, ~(uint64_t)mn);
        }
      }
    }
  };
  __syncthreads();

  // n < 2^32 (checked by the C-ABI): 32-bit tile bookkeeping.  A warp's tiles are claimed one
  // at a time from its CTA's current bucket (cur[b]: positions of b claimed so far, of len_of(b)),
  // through a three-round pipeline so no latency is exposed: a position is claimed (L2 atomic)
  // in round r, mapped to its tile (order[], task mode) in round r + 1, and the tile's TMA is
  // issued in round r + 2 as soon as the stage has been read.  kk counts the tiles the warp's
  // stage has held in this launch (mbarrier parity kk & 1).
  const uint32_t n32 = (uint32_t)n;
  uint32_t kk = 0;
  uint32_t sfirst = 0;  // (all lanes) first launch of the tile in the stage
  const bool by_task = use_task_buckets(hot_n_all);  // else sorted position = tile
  // tile positions of bucket b: [base_of(b), base_of(b) + len_of(b)).  A bucket's groups keep
  // address order, so the last (partial) group is the last of its bucket: that bucket's length
  // stops at the last tile and every position maps to a real tile.
  // (Read when needed: called once per phase and by the bucket picks, nothing kept in registers.)
  auto len_of = [&](uint32_t b) -> uint32_t {
    if (!by_task) return b == kGlobalSet ? ntiles : 0u;
    const uint32_t nt = b < kBuckets ? btot[b] : 0u;
    if (nt == 0u) return 0u;
    const uint32_t ng = (ntiles + kGroupTiles - 1) / kGroupTiles;  // (a non-empty bucket: ng >= 1)
    const uint32_t miss = (uint32_t)__ldg(grp_bucket + ng - 1) == b ? ng * kGroupTiles - ntiles : 0u;
    return kGroupTiles * nt - miss;
  };
  uint32_t cb = kNoBucket, cb_end = 0, cb_base = 0;  // the CTA's current bucket, its length and base
  if (blockIdx.x == 0 && tid == 0) {
    uint32_t nb = 0;
    for (uint32_t b = 0; b < kBuckets; b++) nb += btot[b] ? 1u : 0u;
    st->schedule = by_task ? 1u : 0u;
    st->n_task_buckets = by_task ? nb : 0u;
  }
  constexpr uint32_t kNone = 0xFFFFFFFFu;
  // Positions are claimed kClaim at a time (one L2 atomic per kClaim tiles: a single counter
  // serves every warp in address-order mode); the next range's atomic is issued when the
  // current range is taken, so its result is needed only kClaim tiles later.
  constexpr uint32_t kClaim = 8;
  // The last kTailTiles positions of a bucket are claimed one at a time: a warp that took 8 tiles
  // at the very end would keep its CTA's other warps waiting at the phase barrier for up to 8
  // tile times (~18 us measured with 8-tile claims throughout).
  constexpr uint32_t kTailTiles = 32 * mk::WARPS;
  uint32_t pc = kNone;   // lane 0: claimed position
  uint32_t tn = kNone;   // lane 0: tile of the previous claim (order[] load in flight)
  uint32_t q_pos = 0, q_end = 0, nx = kNone;  // lane 0: current range, next range's start
  uint32_t nsz = kClaim;                       // lane 0: size of the next range
  auto claim = [&]() {   // lane 0
    pc = kNone;
#ifndef FIKIT_ADDR_DYNAMIC
    if (!by_task) {  // address order: the warp's static share [q_pos, q_end) (no claims, no tail skew)
      if (q_pos < q_end) pc = q_pos++;
      return;
    }
#endif
    if (q_pos >= q_end) {
      if (nx == kNone || nx >= cb_end) return;  // drained (claims are monotone)
      q_pos = nx;
      q_end = min(nx + nsz, cb_end);
      nsz = cb_end - q_end > kTailTiles ? kClaim : 1u;
      nx = atomicAdd(cur + cb, nsz);
    }
    pc = q_pos++;
  };
  auto tile_of_claim = [&]() {  // lane 0: position pc -> tile
    tn = pc;
    if (by_task && pc != kNone) {
      const uint32_t p = cb_base + pc;
      tn = __ldg(order + p / kGroupTiles) * kGroupTiles + p % kGroupTiles;
      FK_CHECK(pc < cb_end && tn < ntiles);
    }
  };
  // 1-D TMA of a tile (+ the next launch) into the warp's stage (lane 0)
  auto issue = [&](uint32_t first) {
    FK_CHECK(first < n32 && (first & (mk::CH - 1)) == 0u);
    const uint32_t cnt = min((uint32_t)mk::CH + 1, n32 - first);
    mbar_arrive_expect_tx(&S.full[warp], cnt * 48);
    bulk_g2s(S.ring[warp], recs + first, cnt * 48, &S.full[warp]);
  };

  // ---------------- consumers ----------------
  uint32_t overlap_cnt = 0;
  // deferred cold launches, compacted into lanes [0, np): key words, d, g, record index
  uint32_t pk0 = 0, pk1 = 0, pk2 = 0, pk3 = 0, pk4 = 0, pk5 = 0, pk6 = 0, pgi = 0;
  uint64_t pd = 0, pg = 0;
  uint32_t np = 0;
  auto flush_cold = [&]() {
    FK_TR(if (lane == 0) FK_TR_ADD(8, 1);)
    const uint32_t pend = __ballot_sync(0xffffffffu, lane < (int)np);
    if (lane < (int)np) {
      const uint32_t key[7] = {pk0, pk1, pk2, pk3, pk4, pk5 & 0xFFFFu, pk6};
      const uint32_t row = tuple_find_or_insert(tidx, tslots, key, [&]() {
        const uint64_t kid =
            kernel_id_from(__ldg(name_hash + pk0), __ldg(sig_hash + pk1), pk2, pk3, pk4, pk5 & 0xFFFFu);
        return index_find_or_insert(idx, slots, kid, pk6, key, st, tab.rows, row_tuple, tab.capacity, dict == 0u);
      });
      if (dict && row >= tab.capacity) {  // not in the dictionary (E_DICT): not counted
        atomicOr(&st->flags, kStatusDict);
        atomicMin((unsigned long long*)&st->first_missing_index, (unsigned long long)pgi);
      }
      if (row < tab.capacity) {
        cold_add(tab, row, 0, pd);
        if (pk5 >> 16) cold_add(tab, row, 1, pg);
      }
      FK_CHECK(pgi < n32);
      if (out_row) out_row[pgi] = row;
      // admit the row to the shared dictionary while it has room (one lane per distinct row):
      // this CTA's later launches of it are hot.  mk::admit reserves the tag first, so two warps
      // admitting the same identity concurrently give one slot (a duplicate slot split the row's
      // reductions and wasted the pool: dedup measured k_measure 1.017 -> 0.975 ms on 100M Zipf); a
      // reader that misses the new tag takes the cold path, which is also correct.
      const uint32_t same = __match_any_sync(pend, row);
      if (row < tab.capacity && (same & ((1u << lane) - 1u)) == 0 && ((key[0] | key[1] | key[6]) >> 16) == 0u &&
          *(volatile uint32_t*)&S.hot_n < kHotMax) {
        const uint32_t c0 = key[0] | (key[1] << 16), c4 = key[5] | (key[6] << 16);
        mk::admit(S, mk::hot_hash(c0, key[2], key[3], key[4], c4), row, make_uint4(c0, key[2], key[3], key[4]), c4);
      }
    }
    np = 0;
  };
  // One warp-tile in registers: identity key, K, G and flags of this lane's launch.
  struct Rec {
    uint32_t key[7];
    uint32_t ck0, ck4;  // compressed identity words 0 and 4 (valid if cmp)
    uint32_t hk, gi;
    uint64_t d, g;
    bool valid, gap, live, cmp;
  };
  // read this lane's launch of half h of the stage's tile and the next launch's start/run/task
  // (lane + 1 by shuffle; lane 31 from the record after the half; the halo after the last
  // launch), validate, and compute K, G and the identity hash
  // kFull: the whole tile and the launch after it exist (sfirst + 64 < n, warp-uniform): every lane
  // is live and has a next launch (no per-lane range checks, no halo)
  auto load_half = [&](int h, Rec& R, auto full_tile) {
    constexpr bool kFull = decltype(full_tile)::value;
    const uint32_t first = sfirst + h * mk::TILE;
    const uint32_t cnt = kFull ? (uint32_t)mk::TILE : n32 > first ? min((uint32_t)mk::TILE, n32 - first) : 0u;
    const uint4* rp = S.ring[warp] + (h * mk::TILE + lane) * 3;
    R.live = kFull || (uint32_t)lane < cnt;
    uint4 r0, r1, r2;
    {
      // one 16-B shared load per quarter record (the compiler splits rp[0] into two 8-B loads,
      // which cost as many wavefronts each at this 48-B stride).  Every lane loads (the stage
      // holds 65 records, so the address is in bounds): a lane past the end reads a stale
      // record and every use of it is masked by R.live.
      const uint32_t a = smem_u32(rp);
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r0.x), "=r"(r0.y), "=r"(r0.z), "=r"(r0.w) : "r"(a));
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r1.x), "=r"(r1.y), "=r"(r1.z), "=r"(r1.w) : "r"(a + 16u));
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r2.x), "=r"(r2.y), "=r"(r2.z), "=r"(r2.w) : "r"(a + 32u));
    }
    uint64_t nstart = __shfl_down_sync(0xffffffffu, (uint64_t)r0.x | ((uint64_t)r0.y << 32), 1);
    uint32_t nrun = __shfl_down_sync(0xffffffffu, r2.z, 1);
    uint32_t ntask = __shfl_down_sync(0xffffffffu, r2.w, 1);
    R.gi = first + lane;
    bool has_next = kFull || R.gi + 1 < n32;
    if (lane == 31 && R.live && has_next) {
      const uint4 x = rp[3], y = rp[5];
      nstart = (uint64_t)x.x | ((uint64_t)x.y << 32);
      nrun = y.z;
      ntask = y.w;
    }
    if (!kFull && !has_next && halo != nullptr && R.live) {
      nstart = halo->start_ns;
      nrun = halo->run_id;
      ntask = halo->task_id;
      has_next = true;
    }
    const uint32_t w[12] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w};
    R.valid = R.live && record_valid(w, n_names, n_sigs);
    const uint64_t start = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    const uint64_t end = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    R.d = end - start;                                       // K = end - start
    R.gap = R.live && has_next && ntask == w[11] && nrun == w[10];  // R5
    const bool ov = R.gap && nstart < end;
    R.g = ov ? 0 : nstart - end;  // G = next start - end, clamped
    overlap_cnt += (R.valid && ov) ? 1u : 0u;
    R.key[0] = w[4]; R.key[1] = w[5]; R.key[2] = w[6]; R.key[3] = w[7]; R.key[4] = w[8];
    R.key[5] = w[9] & 0xFFFFu; R.key[6] = w[11];
    R.ck0 = w[4] | (w[5] << 16);
    R.ck4 = (w[9] & 0xFFFFu) | (w[11] << 16);
    R.cmp = ((w[4] | w[5] | w[11]) >> 16) == 0u;
    R.hk = mk::hot_hash(R.ck0, R.key[2], R.key[3], R.key[4], R.ck4);
    // every loaded word is consumed here, so the shared loads have completed
    asm volatile("" ::"r"(R.hk), "l"(R.d), "l"(R.g), "r"((uint32_t)R.gap), "r"((uint32_t)R.valid), "r"(R.gi));
  };
  auto verify = [&](uint32_t c, const Rec& R) -> bool {  // c = slot + 1; branch-free: both loads in flight
    const uint4 a = S.tq[c];
    const uint32_t b = S.tq4[c];
    return ((a.x ^ R.ck0) | (a.y ^ R.key[2]) | (a.z ^ R.key[3]) | (a.w ^ R.key[4]) | (b ^ R.ck4)) == 0u;
  };
  // full lookup (rare: a full home bucket without the key, or a 20-bit tag collision)
  auto probe_slow = [&](const Rec& R) -> int {
    const uint32_t hb = mk::tag_bits(R.hk);
    for (uint32_t q = R.hk & (mk::TAG_Q - 1);; q = (q + 1) & (mk::TAG_Q - 1)) {
      const uint4 t = mk::ld_bucket(S, q);
      const uint32_t v[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int i = 0; i < (int)mk::TAG_W; i++) {
        if (v[i] == 0u) return -1;  // end of the filled prefix: absent
        if ((v[i] ^ hb) < 0x800u && verify(v[i] & 0x7FFu, R)) return (int)(v[i] & 0x7FFu) - 1;
      }
    }
  };
  auto update = [&](const Rec& R, int slot, auto small_tile) {
    constexpr bool kSmall = decltype(small_tile)::value;
    FK_CHECK(slot >= 0 && (uint32_t)slot < min(S.hot_n, kHotMax));
    // the slot's table row: needed for out_row and the >= 2^32 path only (a random 4-B shared load
    // per launch otherwise spent; loading it here schedules better than on demand)
    const uint32_t rowv = (kSmall && out_row == nullptr) ? 0u : S.grow[slot];
    FK_CHECK((kSmall && out_row == nullptr) || rowv < tab.capacity);
    auto row = [&]() { return rowv; };
    const uint32_t hist_e = s_hist + (uint32_t)slot * ((2 * kBins + 1) * 4);
    const uint32_t st_e = s_st + (uint32_t)slot * 20u;
    const uint32_t mm_e = s_mm + (uint32_t)slot * 16u;
    uint4 mm;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(mm.x), "=r"(mm.y), "=r"(mm.z), "=r"(mm.w) : "r"(mm_e));
    uint32_t ad, ag;
    const uint32_t od = hot_add<kSmall>(hist_e, st_e, mm_e, tab, row, 0, R.d, true, mm.x, mm.y, ad);
    const uint32_t og = hot_add<kSmall>(hist_e, st_e, mm_e, tab, row, 1, R.g, R.gap, mm.z, mm.w, ag);
    if (out_row) out_row[R.gi] = row();
    // carries of the two sums (old + a wrapped past 2^32)
    red_shared_add_if(od + ad < od, st_e + 4u, 1u);
    red_shared_add_if(og + ag < og, st_e + 12u, 1u);
  };
  // compact this tile's cold launches behind the pending ones; resolve when a batch is full
  auto compact = [&](const Rec& R, bool cold) {
    const uint32_t cmask = __ballot_sync(0xffffffffu, cold);
    if (!cmask) return;
    const uint32_t nc = __popc(cmask);
    if (np + nc > 32) flush_cold();
    const int t = lane - (int)np;  // lane np + t takes the t-th cold launch of this tile
    int src = 0;
    if (t >= 0 && t < (int)nc) {  // position of the t-th set bit of cmask
      uint32_t m = cmask, q = (uint32_t)t, c;
      c = __popc(m & 0xFFFFu); if (q >= c) { q -= c; src += 16; m >>= 16; }
      c = __popc(m & 0xFFu);   if (q >= c) { q -= c; src += 8;  m >>= 8; }
      c = __popc(m & 0xFu);    if (q >= c) { q -= c; src += 4;  m >>= 4; }
      c = __popc(m & 0x3u);    if (q >= c) { q -= c; src += 2;  m >>= 2; }
      c = m & 1u;              if (q >= c) { src += 1; }
    }
    const bool take = t >= 0 && t < (int)nc;
    const uint32_t k5 = R.key[5] | (R.gap ? 0x10000u : 0u);
    uint32_t v;
    v = __shfl_sync(0xffffffffu, R.key[0], src); if (take) pk0 = v;
    v = __shfl_sync(0xffffffffu, R.key[1], src); if (take) pk1 = v;
    v = __shfl_sync(0xffffffffu, R.key[2], src); if (take) pk2 = v;
    v = __shfl_sync(0xffffffffu, R.key[3], src); if (take) pk3 = v;
    v = __shfl_sync(0xffffffffu, R.key[4], src); if (take) pk4 = v;
    v = __shfl_sync(0xffffffffu, k5, src);       if (take) pk5 = v;
    v = __shfl_sync(0xffffffffu, R.key[6], src); if (take) pk6 = v;
    v = __shfl_sync(0xffffffffu, R.gi, src);     if (take) pgi = v;
    const uint64_t dv = __shfl_sync(0xffffffffu, R.d, src);
    const uint64_t gv = __shfl_sync(0xffffffffu, R.g, src);
    if (take) {
      pd = dv;
      pg = gv;
    }
    np += nc;
    if (np >= 24) flush_cold();
  };

  uint32_t* s_next = &S.next_bucket;
  // the bucket to move to: the most unclaimed tiles among buckets nobody works on (they must
  // be taken) or with more than two tiles left per warp of the CTAs on it and ours (worth a
  // hot-set reload); CTA-uniform
  auto pick_bucket = [&]() -> uint32_t {
    if (warp == 0) {  // the lanes read the buckets' counters in parallel (one L2 round trip)
      uint32_t best = kNoBucket, most = 0;
      for (uint32_t b = lane; b < kSchedWords; b += 32) {
        const uint32_t e = len_of(b), c = *(volatile uint32_t*)(cur + b), a = *(volatile uint32_t*)(act + b);
        const uint32_t left = e > c ? e - c : 0u;
        if (left > most && (left > 2u * mk::WARPS * (a + 1u) || a == 0u)) {
          most = left;
          best = b;
        }
      }
      // the most unclaimed tiles; ties -> the smallest bucket index
      const uint32_t mx = __reduce_max_sync(0xffffffffu, most);
      const uint32_t bb = __reduce_min_sync(0xffffffffu, (mx != 0u && most == mx) ? best : kNoBucket);
      if (lane == 0) *s_next = mx ? bb : kNoBucket;
    }
    __syncthreads();
    const uint32_t b = *s_next;
    __syncthreads();
    return b;
  };
  cb = by_task ? first[blockIdx.x] : kGlobalSet;
  if (cb == kNoBucket) cb = pick_bucket();
  while (cb != kNoBucket) {
    if (tid == 0) atomicAdd(act + cb, 1u);
    FK_TR(if (tid == 0) { tr_t0 = gtime(); tr_first_done = ~0ull; FK_TR_ADD(3, 1); })
    load_hot_set(cb);
    FK_TR(if (tid == 0) { const unsigned long long t = gtime(); FK_TR_ADD(5, t - tr_t0); if (g_trace[blockIdx.x * 16 + 1] == 0) FK_TR_SET(1, t); })
    cb_end = len_of(cb);
    cb_base = by_task ? kGroupTiles * bstart[cb] : 0u;
    q_pos = q_end = 0;
    nsz = 1u;  // (the first range: one tile, the pipeline then sizes the next from its position)
#ifndef FIKIT_ADDR_DYNAMIC
    if (!by_task) {
      // Address order: every warp of the grid takes a static contiguous share of the tiles (+-1
      // tile).  Claiming from one counter shared by all 3552 warps needed multi-tile claims to keep
      // the atomic rate down, and a warp holding a multi-tile claim at the end kept its CTA ~13 us
      // past the others (ResNet-like 3M: phase tail 13 us of a 48 us kernel).
      const uint64_t gw = (uint64_t)blockIdx.x * mk::WARPS + (uint64_t)warp, W = (uint64_t)gridDim.x * mk::WARPS;
      q_pos = (uint32_t)((uint64_t)ntiles * gw / W);
      q_end = (uint32_t)((uint64_t)ntiles * (gw + 1) / W);
    } else
#endif
    if (lane == 0) nx = atomicAdd(cur + cb, 1u);
    // prime the pipeline: the first tile's TMA, the second tile's order[] load, a third claim
    bool staged = false;  // (all lanes) a tile is in flight to the stage
    if (lane == 0) {
      claim();
      tile_of_claim();
      claim();
    }
    {
      const uint32_t t0 = __shfl_sync(0xffffffffu, tn, 0);
      if (t0 != kNone) {
        staged = true;
        sfirst = t0 * mk::CH;
        if (lane == 0) issue(sfirst);
      }
      if (lane == 0) {
        tile_of_claim();
        claim();
      }
    }
    // one phase: every warp consumes tiles until the bucket's claims run out, then the CTA
    // flushes once (u32 bins and carry counters cannot overflow within a call: n < 2^32)
    {
      while (staged) {
        // Each round reads the warp's tile (both halves, A and B) into registers, refills the
        // stage with the next tile, then processes A and B with their identity probes
        // interleaved (two independent dependency chains per lane).
        Rec A, B;
        mbar_wait_s(s_full + 8u * warp, kk & 1u);
        kk++;
        FK_TR(tr_tiles++;)
        if (sfirst + (uint32_t)mk::CH < n32) {  // (every tile but the trace's last)
          load_half(0, A, std::true_type{});
          load_half(1, B, std::true_type{});
        } else {
          load_half(0, A, std::false_type{});
          load_half(1, B, std::false_type{});
        }
        // order the stage reads (generic proxy) before the TMA overwrite (async proxy), refill early
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        const uint32_t tnext = __shfl_sync(0xffffffffu, tn, 0);
        staged = tnext != kNone;
        if (staged) {
          sfirst = tnext * mk::CH;
          if (lane == 0) issue(sfirst);
        }
        if (lane == 0) {
          tile_of_claim();
          claim();
        }
        // home buckets of both launches together (one 8-B load each), then speculative
        // verification of the slot whose tag matches; a miss is final unless the bucket is full
        const uint4 tA = mk::ld_bucket(S, A.hk & (mk::TAG_Q - 1)), tB = mk::ld_bucket(S, B.hk & (mk::TAG_Q - 1));
        uint32_t cA = mk::bucket_match(tA, mk::tag_bits(A.hk)), cB = mk::bucket_match(tB, mk::tag_bits(B.hk));
        const bool fullA = mk::bucket_full(tA), fullB = mk::bucket_full(tB);
        // speculative verification (both loads in flight before the tag compare resolves): without
        // a matching tag (c = 0) the read goes to identity entry 0, which no admission writes
        const bool vA = verify(cA, A) & (cA != 0u);
        const bool vB = verify(cB, B) & (cB != 0u);
        int sA = -1, sB = -1;
        if (A.valid && A.cmp) sA = vA ? (int)cA - 1 : ((cA != 0u || fullA) ? probe_slow(A) : -1);
        if (B.valid && B.cmp) sB = vB ? (int)cB - 1 : ((cB != 0u || fullB) ? probe_slow(B) : -1);
        // every value the warp adds < 2^32 ns (all but pathological traces): the update without the
        // per-value >= 2^32 checks and path
        const uint64_t big = (sA >= 0 ? (A.d | (A.gap ? A.g : 0ull)) : 0ull) | (sB >= 0 ? (B.d | (B.gap ? B.g : 0ull)) : 0ull);
        if (__all_sync(0xffffffffu, (big >> 32) == 0ull)) {
          if (sA >= 0) update(A, sA, std::true_type{});
          if (sB >= 0) update(B, sB, std::true_type{});
        } else {
          if (sA >= 0) update(A, sA, std::false_type{});
          if (sB >= 0) update(B, sB, std::false_type{});
        }
        if (A.live && !A.valid) flag_record(st, A.gi);
        if (B.live && !B.valid) flag_record(st, B.gi);
        compact(A, A.valid && sA < 0);
        compact(B, B.valid && sB < 0);
      }
      FK_TR(if (lane == 0) atomicMin(&tr_first_done, gtime());)
      __syncthreads();
      FK_TR(if (tid == 0) { tr_t0 = gtime(); FK_TR_ADD(6, tr_t0 - tr_first_done); })
      flush_epoch(S, tab, tid);
      __syncthreads();
    }
    flush_hot_set_ext();
    if (tid == 0) atomicSub(act + cb, 1u);  // every claim of cb is done
#ifndef FIKIT_ADDR_DYNAMIC
    if (!by_task) break;  // (address order: the static shares cover every tile)
#endif
    cb = pick_bucket();  // (its barriers also keep the shared rows until every warp is done)
    FK_TR(if (tid == 0) FK_TR_ADD(7, gtime() - tr_t0);)
  }
  FK_TR(if (lane == 0) FK_TR_ADD(4, tr_tiles);)
  if (np) flush_cold();
  // warp-aggregate the overlap count
  uint32_t ov_w = __reduce_add_sync(0xffffffffu, overlap_cnt);
  if (lane == 0 && ov_w) atomicAdd(&S.overlap, (unsigned long long)ov_w);
  __syncthreads();
  if (tid == 0 && S.overlap) atomicAdd((unsigned long long*)&st->n_overlap_gaps, S.overlap);
  FK_TR(if (tid == 0) FK_TR_SET(2, gtime());)
}

size_t measure_smem_bytes() { return sizeof(mk::Smem); }

#ifdef FIKIT_TRACE
// (diagnosis builds only; not part of the C-ABI)
extern "C" int fikit_debug_trace(void* host, int reset) {
  if (reset) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_trace) != cudaSuccess) return -4;
    if (cudaMemset(p, 0, sizeof(g_trace)) != cudaSuccess) return -4;
    if (cudaGetSymbolAddress(&p, g_trace_pre) != cudaSuccess) return -4;
    return cudaMemset(p, 0, sizeof(g_trace_pre)) == cudaSuccess ? 0 : -4;
  }
  return cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace)) == cudaSuccess ? 0 : -4;
}
// which = 1: the k_prep / k_plan block stamps of the last call (k_plan's overwrite k_prep's blocks
// with the same index: read after a call that launched only one of them, or compare roles)
extern "C" int fikit_debug_trace_pre(void* host) {
  return cudaMemcpyFromSymbol(host, g_trace_pre, sizeof(g_trace_pre)) == cudaSuccess ? 0 : -4;
}
#endif
int measure_threads() { return mk::THREADS; }

}  // namespace fikit
