// Internal device helpers of libfikit.so (sm_100a).  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fikit.h"

// FK_CHECK: device-side invariant checks of the checked diagnosis build (nvcc -DFIKIT_CHECKS,
// tests/test_gpu_checked.py: the parity cases rerun on it; a failed check prints and traps, which
// fails the call).  The product build compiles none of them.
#ifdef FIKIT_CHECKS
#include <cstdio>
#define FK_CHECK(c)                                                                    \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("FIKIT_CHECK failed: %s (%s:%d, block %d thread %d)\n", #c, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                       \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define FK_CHECK(c) ((void)0)
#endif

namespace fikit {

constexpr uint32_t kStatusArg = 1u, kStatusName = 2u, kStatusRecord = 4u, kStatusCapacity = 8u, kStatusDict = 16u;
constexpr int kBins = FIKIT_NBINS;

// ---- workspace layout ------------------------------------------------------
struct IndexEntry {  // global open-addressing index (task, kernel ID) -> row
  unsigned long long kid;
  uint32_t task;
  uint32_t state;  // 0 empty, kBusy being written, else row + 1
};
constexpr uint32_t kBusy = 0xFFFFFFFFu;

struct alignas(16) Tuple {  // a launch identity as raw record words (the hot dictionary key) + slot/row
  uint32_t w[7];  // name_id, sig_id, grid_x, grid_y|grid_z<<16, block_x|block_y<<16, block_z, task_id
  uint32_t row;
};

// A measured row in the workspace (fikit_measure accumulates here; fikit_table_finalize writes
// the caller's table from it in canonical order).  One contiguous 336-B row: the cold path's
// reductions of one launch touch one row.
struct RawRow {
  uint64_t kid;
  uint32_t task, pad;
  uint64_t sums[4];  // [1] duration sum, [3] gap sum (mod 2^64); [0], [2] unused (counts = hist totals)
  uint64_t ext[4];   // duration max, ~min, gap max, ~min (an all-zero row is the identity)
  uint32_t hist[64];           // duration bins 0..31, gap bins 32..63
};
static_assert(sizeof(RawRow) == 336, "RawRow");

// fikit_measure's launch sample (k_prep -> k_plan): distinct raw identities with their sample
// counts, keyed by a 64-bit fingerprint of the identity (open addressing; fp 0 = empty).  The
// sample only chooses the hot rows: a fingerprint collision merely credits one identity's
// samples to another, and k_measure still resolves every launch exactly.
struct SampEntry {
  uint32_t cnt, task;  // (one 8-B load in k_plan's scans)
  unsigned long long fp;
  uint32_t w[6];  // the identity's other raw words (Tuple::w[0..5]; w[6] = task)
};
constexpr uint32_t kSampSlots = 32768;
// the occupied slots are also listed densely (samp_list[0 .. hot header word kSampN)), so k_plan
// scans only the distinct sampled identities

// the workspace's measured rows as k_measure sees them
struct RawTab {
  RawRow* rows;
  uint32_t capacity;
};

struct WsLayout {
  size_t status, misc, name_hash, sig_hash, index, tindex, row_tuple, samp, hot, raw, rank, fin, tiles, total;
  uint32_t slots, tslots;
  uint64_t ntiles;   // warp-tiles of 64 launches the workspace can schedule
  uint64_t ngroups;  // tile groups (kGroupTiles tiles) of the task-partitioned schedule
};

constexpr uint32_t kHotMax = 400;  // hot rows cached in shared memory per CTA (measure kernel; u32 bins)
// Task-partitioned scheduling of fikit_measure: warp-tiles (32 launches) are bucketed by a
// hash of their first launch's task_id; every bucket has its own hot set.
// regions zeroed by k_zero (one launch instead of a memset per region)
constexpr int kZeroRegions = 12;
struct ZeroList {
  void* p[kZeroRegions];
  uint64_t n[kZeroRegions];  // bytes, multiples of 4; p 4-B aligned
  int k;
};
constexpr uint32_t kBuckets = 64;
constexpr uint32_t kMaxCTAs = 1024;
constexpr uint32_t kSortBlocks = 160;  // blocks of the tile-group counting sort (each a contiguous chunk)
constexpr uint32_t kGroupTiles = 4;    // warp-tiles per schedule group (256 launches: one sector read each)
constexpr uint32_t kGlobalSet = kBuckets;  // hot-set index of the global (all-task) hot set
// hot-set header words (u32): hot_n[kBuckets + 1], then the sample coverage counters
constexpr uint32_t kCovTask = kBuckets + 1;  // samples whose row is in its task bucket's hot set
constexpr uint32_t kCovGlobal = kBuckets + 2;  // samples whose row is in the global hot set
constexpr uint32_t kCovTotal = kBuckets + 3;  // samples with a row
constexpr uint32_t kSampN = kBuckets + 4;  // distinct identities in the launch sample
constexpr uint32_t kPlanStamp = kBuckets + 6;  // (u64, words 70-71) dictionary hash the hot sets were built on
constexpr uint32_t kHotHdr = kBuckets + 8;
constexpr uint32_t kTileLaunches = 64;  // launches per warp-tile of the measure kernel (one TMA)
constexpr uint32_t kFinGroup = 2048;    // fikit_table_finalize: keys per sorted group (one 1024-thread block's)
struct FinKey {                          // a sorted key of finalize's groups (workspace)
  unsigned long long kid;
  uint32_t task, pad;
};
constexpr int kResolveThreads = 1024;        // k_resolve block (one per SM)
constexpr uint32_t kResolveSmemKeys = 8192;  // table keys staged in shared memory (96 KB) up to this K
constexpr int kRegThreads = 512;  // k_simulate_reg block (16 warps, one scenario each)
constexpr int kSimThreads = 128;  // k_simulate block (4 warps, shared-memory pools)
constexpr int kStreamThreads = 128;  // k_simulate_stream block (4 warps, staged windows)
// u32 words of the 256-B status region past fikit_status_t, zeroed with it: replay work counters
constexpr uint32_t kSchedWord1 = 32, kSchedWord2 = 33, kSchedWord3 = 34;
// Dynamic tile schedule (k_plan -> k_measure).  Task mode: tile groups are stably counting-sorted
// by bucket into order[]; bucket b owns the tile positions [4 bstart[b], 4 (bstart[b] + btot[b]))
// (position p = tile 4 order[p / 4] + p % 4; positions past the last tile are skipped).
// Address mode: bucket kGlobalSet = tiles [0, ntiles) in order.  cur[b] counts the positions of
// b claimed so far (zeroed by k_zero); warps claim kClaim at a time.  first[c] is the bucket CTA
// c starts on (kNoBucket: none); a CTA whose bucket runs dry moves to the bucket with the most
// unclaimed tiles among those nobody works on or with > 128 left (act[b]: CTAs working on b).
constexpr uint32_t kNoBucket = 0xFFFFFFFFu;
constexpr uint32_t kSchedWords = kBuckets + 8;  // cur[], act[], bstart[], btot[] length

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline uint32_t index_slots(uint32_t cap) {
  uint32_t s = 1024;
  while (s < 2ull * cap) s <<= 1;
  return s;
}

// Regions are ordered by what sizes them, so that every call finds a region at the same offset
// from the arguments it has: capacity-sized regions first (finalize knows only the table), then
// the string hashes (resolve knows the table and the string tables), then the tile schedule
// (sized by the measure call's record count), then the multi-GPU union scratch.
inline WsLayout ws_layout(uint32_t cap, uint32_t n_names, uint32_t n_sigs, uint64_t n_records) {
  WsLayout L;
  size_t o = 0;
  L.status = o;
  o += 256;
  L.misc = o;
  o += 256;
  L.slots = index_slots(2 * cap);  // KID index: load <= 1/4 (short linear-probe chains: k_plan's
                                   // hot-row inserts wait on the longest one)
  L.index = o;
  o = align256(o + sizeof(IndexEntry) * (size_t)L.slots);
  L.tslots = index_slots(2 * cap);
  L.tindex = o;
  o = align256(o + sizeof(Tuple) * (size_t)L.tslots);
  L.row_tuple = o;
  o = align256(o + sizeof(Tuple) * (size_t)cap);
  L.samp = o;  // SampEntry[kSampSlots], then samp_list[kSampSlots] (u32)
  o = align256(o + sizeof(SampEntry) * (size_t)kSampSlots);
  o = align256(o + 4ull * kSampSlots);
  L.hot = o;  // header[kHotHdr] (u32), then hot[kBuckets + 1][kHotMax] (Tuple)
  o = align256(o + 4ull * kHotHdr + sizeof(Tuple) * (size_t)kHotMax * (kBuckets + 1));
  L.raw = o;  // RawRow[cap]
  o = align256(o + sizeof(RawRow) * (size_t)cap);
  L.rank = o;  // rank[cap] (u32), then the sorted key groups FinKey[cap]
  o = align256(o + 4ull * cap);
  o = align256(o + sizeof(FinKey) * (size_t)cap);
  L.name_hash = o;
  o = align256(o + 8ull * (n_names ? n_names : 1));
  L.sig_hash = o;
  o = align256(o + 8ull * (n_sigs ? n_sigs : 1));
  // tiles: cur[kSchedWords], act[kSchedWords], bstart[kSchedWords], btot[kSchedWords],
  //        first[kMaxCTAs] (u32), blkcnt[kSortBlocks][kBuckets] (u32), grp_bucket[ngroups] (u8),
  //        order[ngroups] (u32)
  L.ntiles = (n_records + kTileLaunches - 1) / kTileLaunches;
  L.ngroups = (L.ntiles + kGroupTiles - 1) / kGroupTiles;
  L.tiles = o;
  o = align256(o + 16ull * kSchedWords + 4ull * kMaxCTAs);
  o = align256(o + 4ull * kSortBlocks * kBuckets);
  o = align256(o + L.ngroups);
  o = align256(o + 4ull * L.ngroups);
  L.fin = o;  // last: scratch of the multi-GPU dictionary union (which also uses the caller's `extra` bytes)
  o = align256(o + 1024);
  L.total = o;
  return L;
}

// arguments of the measure call's preamble kernels (measure.cu)
struct PrepArgs {
  const uint4* recs;
  const fikit_record_t* recs_t;
  uint64_t n, stride, n_samples;
  fikit_strtab_t names, sigs;
  uint64_t* name_hash;
  uint64_t* sig_hash;
  fikit_status_t* st;
  SampEntry* samp;
  uint32_t* samp_list;
  uint32_t* samp_n;
  uint8_t* grp_bucket;
  uint32_t* blkcnt;
  uint32_t ngroups, sb;     // tile groups, group-role blocks
  const uint32_t* hot_hdr;  // the hot-set header (a reused plan's schedule mode)
  uint32_t reused_plan;     // FIKIT_MEASURE_REUSE_PLAN
  uint32_t nb_hash, nb_samp;  // block ranges: [0, nb_hash) hash, then nb_samp sample blocks, then sb group blocks
};
constexpr int kPrepThreads = 256;

struct PlanArgs {
  fikit_status_t* st;
  const SampEntry* samp;
  const uint32_t* samp_list;
  // resolving the chosen identities to rows (kernel ID -> KID index; k_prep hashed the strings)
  const uint64_t* name_hash;
  const uint64_t* sig_hash;
  IndexEntry* idx;
  uint32_t slots;
  RawRow* raw;
  Tuple* row_tuple;
  uint32_t cap;
  Tuple* hot_all;
  uint32_t* hot_hdr;
  const uint8_t* grp_bucket;
  const uint32_t* blkcnt;
  uint32_t ngroups, sb;
  uint32_t grid_measure;  // k_measure CTAs (first-bucket assignment)
  uint32_t* order;
  uint32_t* bstart;
  uint32_t* btot;
  uint32_t* first;
  uint32_t dict;  // dictionary mode: rows are never inserted
  uint32_t hot_blocks;  // kBuckets + 1 (choose the hot sets) or 0 (reused: the plan of the previous call)
  const unsigned long long* dict_hash;  // this call's dictionary hash (k_dict_load)
};

// task bucket: xor-fold of the task id's 6-bit digits -- one-to-one for ids < 64 (a node's
// tasks are usually numbered densely), and multiples of 64 still spread
__host__ __device__ __forceinline__ uint32_t bucket_of(uint32_t task) {
  return (task ^ (task >> 6) ^ (task >> 12) ^ (task >> 18) ^ (task >> 24) ^ (task >> 30)) & (kBuckets - 1);
}

// Schedule mode, decided identically by every kernel from the sample coverage counters (hdr =
// hot-set header): task-partitioned when the global hot set misses > 2% of the sampled launches
// and the per-task hot sets cover > 2 points more; else one grid-stride sweep in address order.
__host__ __device__ __forceinline__ bool use_task_buckets(const uint32_t* hdr) {
  const uint64_t tot = hdr[kCovTotal], g = hdr[kCovGlobal], t = hdr[kCovTask];
  return (tot - g) * 50 > tot && t > g && (t - g) * 50 > tot;
}

// misc counters (u32 words at ws + misc)
enum MiscWord { kMiscDict = 0, kMiscDictHash = 2 };  // dictionary mode of the last measure call: dict_n + 1,
                                                     // 0 = none; words 2-3: the dictionary's hash (u64)

// Programmatic dependent launch hooks (first statement of every kernel of a call): with
// cudaLaunchAttributeProgrammaticStreamSerialization a kernel's CTAs could be scheduled while the
// previous kernel finishes, griddepcontrol.wait then blocking until its writes are visible.  The
// C-ABI launches without the attribute (see launch_pdl: it measured slower), so both are no-ops;
// they keep every kernel correct should a caller launch them programmatically.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

// Kernel launch helper.  Programmatic dependent launch (the attribute
// cudaLaunchAttributeProgrammaticStreamSerialization, with griddepcontrol.wait as every kernel's
// first statement) was measured and left off: the early-launched CTAs sat on SM resources while
// the previous kernel finished, and the measure call got 1-7 % slower (interleaved A/B,
// profiles/r02/README.md).  Without the attribute pdl_entry() is a no-op.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  (void)cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);  // (errors surface in launched())
}

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---- hashing (R2) ------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint64_t kernel_id_from(uint64_t h_name, uint64_t h_sig, uint32_t gx, uint32_t gyz,
                                                   uint32_t bxy, uint32_t bz) {
  // w1 = grid_x | grid_y<<32 | grid_z<<48 ; w2 = block_x | block_y<<16 | block_z<<32
  uint64_t w1 = (uint64_t)gx | ((uint64_t)(gyz & 0xFFFFu) << 32) | ((uint64_t)(gyz >> 16) << 48);
  uint64_t w2 = (uint64_t)bxy | ((uint64_t)(bz & 0xFFFFu) << 32);
  uint64_t h = mix64(h_name ^ h_sig);
  h = mix64(h ^ w1);
  h = mix64(h ^ w2);
  return h == 0 ? 1 : h;
}

__device__ __forceinline__ uint32_t key_hash(uint64_t kid, uint32_t task) {
  uint64_t x = kid ^ (0x9e3779b97f4a7c15ULL * (uint64_t)(task + 1));
  x ^= x >> 29;
  x *= 0xbf58476d1ce4e5b9ULL;
  return (uint32_t)(x >> 32);
}

// 32-bit hash of the raw identity words (hot dictionary / tuple index probe);
// murmur3 fmix32 finaliser: grid/block dims are powers of two, so the low bits
// of a plain multiplicative hash would cluster
__device__ __forceinline__ uint32_t tuple_hash(const uint32_t* w) {
  uint32_t h = w[0] * 0x9E3779B1u;
  h = (h ^ w[1]) * 0x85EBCA77u;
  h = (h ^ w[2]) * 0xC2B2AE3Du;
  h = (h ^ w[3]) * 0x27D4EB2Fu;
  h = (h ^ w[4]) * 0x165667B1u;
  h = (h ^ w[5]) * 0x9E3779B1u;
  h = (h ^ w[6]) * 0x85EBCA77u;
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ int bin_of(uint64_t v) {
  int b = 64 - __clzll((long long)v);  // bit_length
  return b < 31 ? b : 31;
}

// ---- records as 12 u32 words --------------------------------------------------
// w0,w1 start; w2,w3 end; w4 name; w5 sig; w6 grid_x; w7 grid_y|grid_z<<16;
// w8 block_x|block_y<<16; w9 block_z|flags<<16; w10 run; w11 task
__device__ __forceinline__ bool record_valid(const uint32_t* w, uint32_t n_names, uint32_t n_sigs) {
  uint64_t s = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  uint64_t e = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
  // grid_y, grid_z, block_x, block_y >= 1: one packed 16-bit 3-way min; 1 <= block_z and flags == 0
  // <=> 1 <= w9 <= 0xFFFF
  const bool dims = __vminu2(__vminu2(w[7], w[8]), 0x00010001u) == 0x00010001u;
  bool ok = (w[6] != 0) & dims & ((w[9] - 1u) < 0xFFFFu) & (w[4] < n_names) & (w[5] < n_sigs) & (e >= s);
  return ok;
}

// ---- status ---------------------------------------------------------------------
__device__ __forceinline__ void flag_record(fikit_status_t* st, uint64_t idx) {
  atomicOr(&st->flags, kStatusRecord);
  atomicMin((unsigned long long*)&st->first_bad_index, (unsigned long long)idx);
}

// ---- global indices -------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// release store at gpu scope: every earlier write of the thread is visible to a reader that
// observes this value (cheaper than __threadfence() + atomicExch)
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// coherent 16-B load at gpu scope; asm volatile so it is never merged with an
// earlier load of the same entry (the CUDA __ldcg is non-volatile asm and can be CSE'd)
__device__ __forceinline__ uint4 ld_relaxed_v4(const void* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// Entries are written once (key words, __threadfence, then the state word) and never
// change after; a reader takes a 16-B / 32-B entry from L2 in one access (__ldcg), so a
// published state implies the key words of the same sector are visible.

// KID index: find-or-insert (task, kid); returns the row (possibly >= capacity: then
// nothing is materialised and E_CAPACITY is flagged) or FIKIT_NO_ROW if the index is
// full.  The inserting thread records the row's key (in the workspace's raw row) and a
// representative raw tuple.  insert = false (dictionary mode: every row was placed by
// k_dict_load): an absent key returns FIKIT_NO_ROW.
__device__ __forceinline__ uint32_t index_find_or_insert(IndexEntry* idx, uint32_t slots, uint64_t kid, uint32_t task,
                                                         const uint32_t* tuple_w, fikit_status_t* st, RawRow* raw,
                                                         Tuple* row_tuple, uint32_t cap, bool insert = true) {
  uint32_t h = key_hash(kid, task) & (slots - 1);
  for (uint32_t probe = 0; probe < slots; probe++) {
    IndexEntry* e = &idx[h];
    uint4 v = ld_relaxed_v4(e);
    uint32_t s = v.w;
    if (s == 0 && !insert) return FIKIT_NO_ROW;
    if (s == 0) {
      uint32_t old = atomicCAS(&e->state, 0u, kBusy);
      if (old == 0) {
        e->kid = kid;
        e->task = task;
        uint32_t row = (uint32_t)atomicAdd((unsigned long long*)&st->n_rows_needed, 1ull);
        if (row < cap) {  // (its statistics were zeroed by k_zero)
          raw[row].kid = kid;
          raw[row].task = task;
          Tuple t;
#pragma unroll
          for (int j = 0; j < 7; j++) t.w[j] = tuple_w[j];
          t.row = row;
          row_tuple[row] = t;
        } else {
          atomicOr(&st->flags, kStatusCapacity);
        }
        st_release_u32(&e->state, row + 1);  // publishes the key words and the row's key
        return row;
      }
      s = old;
    }
    if (s == kBusy) {
      while (s == kBusy) s = ld_acquire_u32(&e->state);
    }
    v = ld_relaxed_v4(e);
    if ((((uint64_t)v.y << 32) | v.x) == kid && v.z == task) return v.w - 1;
    h = (h + 1) & (slots - 1);
  }
  atomicOr(&st->flags, kStatusCapacity);
  return FIKIT_NO_ROW;
}

// tuple index: raw identity words -> row.  Steady state: one 32-B L2 read per
// launch of a cold row (no name-hash gather, no 64-bit ID mixing); a miss computes
// the kernel ID and resolves it through the KID index (two names with identical
// bytes are two tuples of one row).
template <class Slow>
__device__ __forceinline__ uint32_t tuple_find_or_insert(Tuple* tidx, uint32_t tslots, const uint32_t* key,
                                                         Slow slow) {
  uint32_t h = tuple_hash(key) & (tslots - 1);
  for (uint32_t probe = 0; probe < tslots; probe++) {
    Tuple* e = &tidx[h];
    uint4 a = ld_relaxed_v4(e);
    uint4 b = ld_relaxed_v4(reinterpret_cast<const uint4*>(e) + 1);
    uint32_t s = b.w;
    if (s == 0) {
      uint32_t old = atomicCAS(&e->row, 0u, kBusy);
      if (old == 0) {
        uint32_t row = slow();
#pragma unroll
        for (int j = 0; j < 7; j++) e->w[j] = key[j];
        __threadfence();
        atomicExch(&e->row, (row < 0xFFFFFFFDu ? row : 0xFFFFFFFDu) + 1);
        return row;
      }
      s = old;
    }
    if (s == kBusy || b.w == 0) {  // being written, or our CAS lost to a writer: re-read
      while (s == kBusy) s = ld_relaxed_u32(&e->row);
      a = ld_relaxed_v4(e);
      b = ld_relaxed_v4(reinterpret_cast<const uint4*>(e) + 1);
    }
    if (a.x == key[0] && a.y == key[1] && a.z == key[2] && a.w == key[3] && b.x == key[4] && b.y == key[5] &&
        b.z == key[6])
      return b.w - 1;
    h = (h + 1) & (tslots - 1);
  }
  return slow();
}

// ---- mbarrier / bulk copy (sm_90+ PTX) --------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// variants on precomputed 32-bit shared addresses (no generic->shared conversion per call)
__device__ __forceinline__ void mbar_arrive_s(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// 1-D TMA: global -> shared, completion counted on the mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void lds128(const void* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(smem_u32(p)));
}

// shared-memory 64-bit min/max (no native ATOMS.MIN.64: CAS loop; rare after warm-up)
__device__ __forceinline__ void smem_min64(unsigned long long* p, unsigned long long v) {
  unsigned long long cur = *(volatile unsigned long long*)p;
  while (v < cur) {
    unsigned long long prev = atomicCAS(p, cur, v);
    if (prev == cur) break;
    cur = prev;
  }
}
__device__ __forceinline__ void smem_max64(unsigned long long* p, unsigned long long v) {
  unsigned long long cur = *(volatile unsigned long long*)p;
  while (v > cur) {
    unsigned long long prev = atomicCAS(p, cur, v);
    if (prev == cur) break;
    cur = prev;
  }
}

}  // namespace fikit

// launch bookkeeping (host)
void fikit_note_launch(int n = 1);
