// C-ABI entry points of libfikit.so (declared in include/fikit.h).
// Argument checks on the host, then stream-ordered launches; no allocation.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>

#include "fikit_internal.cuh"

namespace fikit {
// kernels (measure.cu, finalize.cu, replay.cu)
__global__ void k_reset_status(fikit_status_t*);
__global__ void k_zero(ZeroList, fikit_status_t*);
__global__ void k_strtab_hash(fikit_strtab_t, uint64_t*, fikit_strtab_t, uint64_t*, fikit_status_t*);
__global__ void k_identify(const uint4*, uint64_t, const uint64_t*, const uint64_t*, uint32_t, uint32_t, uint64_t*,
                           fikit_status_t*);
__global__ void k_prep(PrepArgs);
__global__ void k_plan(PlanArgs);
__global__ void k_measure(const fikit_record_t*, uint64_t, const fikit_record_t*, const uint64_t*, const uint64_t*,
                          uint32_t, uint32_t, IndexEntry*, uint32_t, Tuple*, uint32_t, fikit_status_t*, RawTab, Tuple*,
                          const Tuple*, const uint32_t*, uint32_t*, uint32_t*, const uint32_t*, const uint32_t*,
                          const uint32_t*, const uint32_t*, const uint8_t*, uint32_t, uint32_t*, uint32_t);
size_t measure_smem_bytes();
int measure_threads();
__global__ void k_fin_sort(const fikit_status_t*, const RawRow*, uint32_t, fikit_table_t, FinKey*, const uint32_t*);
__global__ void k_fin_sort256(const fikit_status_t*, const RawRow*, uint32_t, fikit_table_t, FinKey*, const uint32_t*);
__global__ void k_fin_scatter(const fikit_status_t*, const RawRow*, uint32_t, uint32_t, const FinKey*, uint32_t, fikit_table_t,
                              uint32_t*, const uint32_t*);
__global__ void k_dict_load(const uint64_t*, const uint32_t*, uint32_t, IndexEntry*, uint32_t, RawRow*,
                            fikit_status_t*, uint32_t*, uint32_t);
__global__ void k_remap_rows(uint32_t*, uint64_t, const uint32_t*, const uint32_t*);
__global__ void k_means(fikit_table_t);
__global__ void k_predict(fikit_table_t, uint32_t, uint32_t);
__global__ void k_lookup(fikit_table_t, const uint64_t*, const uint32_t*, uint64_t, uint32_t*);
__global__ void k_resolve(const uint4*, uint64_t, const fikit_record_t*, const uint64_t*, const uint64_t*, uint32_t,
                          uint32_t, fikit_table_t, uint32_t*, uint64_t*, uint64_t*, fikit_status_t*);
__global__ void k_union_flags(const uint64_t*, const uint32_t*, const uint32_t*, uint32_t, uint32_t, uint32_t*);
__global__ void k_union_scan(const uint32_t*, uint32_t, uint32_t*);
__global__ void k_union_place(const uint64_t*, const uint32_t*, const uint32_t*, uint32_t, uint32_t, uint32_t,
                              const uint32_t*, const uint32_t*, uint64_t*, uint32_t*, uint32_t, uint32_t*, uint32_t*,
                              fikit_status_t*);
__global__ void k_table_remap(fikit_table_t, const uint32_t*, const uint64_t*, const uint32_t*, const uint32_t*,
                              fikit_table_t);
__global__ void k_table_bias(fikit_table_t);
__global__ void k_fill(fikit_table_t, const uint64_t*, const uint64_t*, const uint32_t*, const uint64_t*,
                       const uint8_t*, const uint32_t*, const uint32_t*, uint32_t, fikit_fill_params_t, uint32_t*,
                       const uint32_t*, uint32_t*, uint64_t*, uint64_t*, fikit_status_t*);
const void* simulate_smem_kernel(bool sched);
void launch_simulate_smem(int, int, cudaStream_t, const fikit_table_t&, const uint32_t*, const uint64_t*,
                          const uint64_t*, const uint32_t*, const uint64_t*, const uint8_t*, const fikit_scenario_t*,
                          uint32_t, fikit_fill_params_t, fikit_result_t*, int32_t*, uint64_t*, const uint64_t*,
                          fikit_status_t*);
const void* simulate_reg_kernel(bool sched);
void launch_simulate_reg(int, int, cudaStream_t, const fikit_table_t&, const uint32_t*, const uint64_t*,
                         const uint64_t*, const uint32_t*, const uint64_t*, const uint8_t*, const fikit_scenario_t*,
                         uint32_t, fikit_fill_params_t, fikit_result_t*, int32_t*, uint64_t*, const uint64_t*,
                         fikit_status_t*);
const void* simulate_stream_kernel(bool sched);
void launch_simulate_stream(int, int, cudaStream_t, const fikit_table_t&, const uint32_t*, const uint64_t*,
                            const uint64_t*, const uint32_t*, const uint64_t*, const uint8_t*, const uint32_t*,
                            const uint64_t*, const uint64_t*, const fikit_scenario_t*, uint32_t, fikit_fill_params_t,
                            fikit_result_t*, int32_t*, uint64_t*, const uint64_t*, fikit_status_t*);
}  // namespace fikit

using namespace fikit;

static std::atomic<uint64_t> g_launches{0};
void fikit_note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

namespace {

// Per-device caches of immutable device / kernel properties (SM count, occupancy, the
// k_measure shared-memory attribute).  Every entry is computed idempotently from the current
// device and published with a relaxed atomic store, so concurrent first calls only repeat the
// same query and a second device gets its own entry (no per-process "first device" state).
constexpr int kMaxDevices = 64;
enum : int { kPropSms, kPropWaveReg, kPropWaveSmem, kPropWaveStream, kPropMeasureAttr, kPropFinAttr, kPropResolveAttr, kNumProps };
std::atomic<int> g_prop[kMaxDevices][kNumProps];  // 0 = not computed yet

int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  return dev;
}

template <class F>
int dev_prop(int which, F compute) {
  const int dev = cur_device();
  if (dev >= kMaxDevices) return compute(dev);
  int v = g_prop[dev][which].load(std::memory_order_relaxed);
  if (v == 0) {
    v = compute(dev);
    if (v > 0) g_prop[dev][which].store(v, std::memory_order_relaxed);
  }
  return v;
}

int num_sms() {
  return dev_prop(kPropSms, [](int dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    return n;
  });
}

inline bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

inline int launched() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "libfikit: launch failed: %s\n", cudaGetErrorString(e));
    return FIKIT_E_CUDA;
  }
  fikit_note_launch();
  return FIKIT_OK;
}

struct Ws {
  unsigned char* base;
  WsLayout L;
  fikit_status_t* st() const { return reinterpret_cast<fikit_status_t*>(base + L.status); }
  uint32_t* misc() const { return reinterpret_cast<uint32_t*>(base + L.misc); }
  uint64_t* name_hash() const { return reinterpret_cast<uint64_t*>(base + L.name_hash); }
  uint64_t* sig_hash() const { return reinterpret_cast<uint64_t*>(base + L.sig_hash); }
  IndexEntry* index() const { return reinterpret_cast<IndexEntry*>(base + L.index); }
  Tuple* row_tuple() const { return reinterpret_cast<Tuple*>(base + L.row_tuple); }
  Tuple* tindex() const { return reinterpret_cast<Tuple*>(base + L.tindex); }
  SampEntry* samp() const { return reinterpret_cast<SampEntry*>(base + L.samp); }
  uint32_t* samp_list() const {
    return reinterpret_cast<uint32_t*>(base + L.samp + align256(sizeof(SampEntry) * (size_t)kSampSlots));
  }
  uint32_t* hot_n() const { return reinterpret_cast<uint32_t*>(base + L.hot); }  // header [kHotHdr]
  Tuple* hot() const { return reinterpret_cast<Tuple*>(base + L.hot + 4ull * kHotHdr); }  // [kBuckets + 1][kHotMax]
  RawRow* raw() const { return reinterpret_cast<RawRow*>(base + L.raw); }
  uint32_t* rank() const { return reinterpret_cast<uint32_t*>(base + L.rank); }  // [cap]
  FinKey* fin_keys(uint32_t cap) const {  // [cap], after rank[]
    return reinterpret_cast<FinKey*>(base + L.rank + align256(4ull * cap));
  }
  uint32_t* cur() const { return reinterpret_cast<uint32_t*>(base + L.tiles); }   // [kSchedWords]
  uint32_t* act() const { return cur() + kSchedWords; }                           // [kSchedWords]
  uint32_t* bstart() const { return act() + kSchedWords; }                        // [kSchedWords]
  uint32_t* btot() const { return bstart() + kSchedWords; }                       // [kSchedWords]
  uint32_t* first() const { return btot() + kSchedWords; }                        // [kMaxCTAs]
  uint32_t* blkcnt() const {  // [kSortBlocks][kBuckets]
    return reinterpret_cast<uint32_t*>(base + L.tiles + align256(16ull * kSchedWords + 4ull * kMaxCTAs));
  }
  uint8_t* grp_bucket() const {
    return reinterpret_cast<uint8_t*>(blkcnt()) + align256(4ull * kSortBlocks * kBuckets);
  }
  uint32_t* order() const { return reinterpret_cast<uint32_t*>(grp_bucket() + align256(L.ngroups)); }
  unsigned char* fin() const { return base + L.fin; }
};

// workspace check for a capacity and string-table sizes
int get_ws(void* ws, size_t ws_bytes, uint32_t cap, uint32_t nn, uint32_t ns, Ws* out, uint64_t n_records = 0) {
  if (!ws || !aligned(ws, 256)) return FIKIT_E_ARG;
  out->base = static_cast<unsigned char*>(ws);
  out->L = ws_layout(cap, nn, ns, n_records);
  if (ws_bytes < out->L.total) return FIKIT_E_ARG;
  return FIKIT_OK;
}

inline int reset_status(const Ws& w, cudaStream_t s) {
  launch_pdl(k_reset_status, 1, 32, 0, s, w.st());  // a kernel, so the call stays graph-capturable
  return launched();
}

inline bool strtab_ok(const fikit_strtab_t& t) { return t.offsets != nullptr && (t.count == 0 || t.bytes != nullptr); }

inline bool table_ok(const fikit_table_t* t) {
  return t && t->kernel_id && t->task_id && t->sums && t->hist && t->ext && t->mean && t->n_rows && t->capacity > 0 &&
         t->capacity <= (1u << 24);
}

int hash_strtabs(const Ws& w, const fikit_strtab_t& names, const fikit_strtab_t& sigs, cudaStream_t s) {
  const uint32_t mx = names.count > sigs.count ? names.count : sigs.count;
  if (mx) {  // one warp per string, names (y = 0) and signatures (y = 1) in one launch
    launch_pdl(k_strtab_hash, dim3((mx + 3) / 4, 2), 128, 0, s, names, w.name_hash(), sigs, w.sig_hash(), w.st());
    if (int r = launched()) return r;
  }
  return FIKIT_OK;
}

unsigned grid_for(uint64_t work, unsigned per_block, unsigned max_blocks) {
  uint64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (unsigned)b;
}

}  // namespace

extern "C" {

size_t fikit_ws_bytes(uint32_t capacity, uint32_t n_names, uint32_t n_sigs, uint64_t n_records) {
  return ws_layout(capacity ? capacity : 1, n_names, n_sigs, n_records).total;
}

size_t fikit_table_bytes(uint32_t cap) {
  size_t o = 0;
  o = align256(o + 8ull * cap);   // kernel_id
  o = align256(o + 4ull * cap);   // task_id
  o = align256(o + 32ull * cap);  // sums
  o = align256(o + 256ull * cap); // hist
  o = align256(o + 32ull * cap);  // ext
  o = align256(o + 16ull * cap);  // mean
  o = align256(o + 4);            // n_rows
  return o;
}

int fikit_table_carve(void* block, uint32_t cap, fikit_table_t* t) {
  if (!block || !t || !aligned(block, 256) || cap == 0) return FIKIT_E_ARG;
  unsigned char* b = static_cast<unsigned char*>(block);
  size_t o = 0;
  t->kernel_id = reinterpret_cast<uint64_t*>(b + o);
  o = align256(o + 8ull * cap);
  t->task_id = reinterpret_cast<uint32_t*>(b + o);
  o = align256(o + 4ull * cap);
  t->sums = reinterpret_cast<uint64_t*>(b + o);
  o = align256(o + 32ull * cap);
  t->hist = reinterpret_cast<uint32_t*>(b + o);
  o = align256(o + 256ull * cap);
  t->ext = reinterpret_cast<uint64_t*>(b + o);
  o = align256(o + 32ull * cap);
  t->mean = reinterpret_cast<uint64_t*>(b + o);
  o = align256(o + 16ull * cap);
  t->n_rows = reinterpret_cast<uint32_t*>(b + o);
  t->capacity = cap;
  return FIKIT_OK;
}

int fikit_identify(const fikit_record_t* recs, uint64_t n, fikit_strtab_t names, fikit_strtab_t sigs, uint64_t* out,
                   void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  if (n >= (1ull << 32) || (n && (!recs || !out || !aligned(recs, 16))) || !strtab_ok(names) || !strtab_ok(sigs))
    return FIKIT_E_ARG;
  if (int r = get_ws(ws, ws_bytes, 1, names.count, sigs.count, &w)) return r;
  if (int r = reset_status(w, s)) return r;
  if (int r = hash_strtabs(w, names, sigs, s)) return r;
  if (n == 0) return FIKIT_OK;
  launch_pdl(k_identify, grid_for((n + 31) / 32, 8, num_sms() * 8), 256, 0, s, 
      reinterpret_cast<const uint4*>(recs), n, w.name_hash(), w.sig_hash(), names.count, sigs.count, out, w.st());
  return launched();
}

// the caller's timing events: inside a stream capture they become external event-record nodes, so
// they still time the kernel on every replay of the graph (a plain record there is only an
// internal dependency)
static bool record_ev(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) return false;
  return (cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                                              : cudaEventRecord(ev, s)) == cudaSuccess;
}

static int measure_impl(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                        fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, void* ws,
                        size_t ws_bytes, void* stream, cudaEvent_t ev0, cudaEvent_t ev1,
                        const uint64_t* dict_kid = nullptr, const uint32_t* dict_task = nullptr,
                        uint32_t dict_n = 0, uint32_t flags = 0) {
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  const bool dict = dict_kid != nullptr;
  const bool reuse = (flags & FIKIT_MEASURE_REUSE_PLAN) != 0;
  if (n >= (1ull << 32) || (n && (!recs || !aligned(recs, 16))) || !strtab_ok(names) || !strtab_ok(sigs) ||
      !table_ok(tab) || (dict && (!dict_task || dict_n == 0 || dict_n > tab->capacity)) ||
      (flags & ~FIKIT_MEASURE_REUSE_PLAN) || (reuse && !dict))
    return FIKIT_E_ARG;
  if (int r = get_ws(ws, ws_bytes, tab->capacity, names.count, sigs.count, &w, n)) return r;
  const uint32_t cap = tab->capacity;
  // 1. reset the status; zero the workspace's measured rows (an all-zero row is the identity of
  //    every statistic), the indexes, the sample counts, the hot-set header, the schedule's
  //    counters and finalize's counters: one launch
  ZeroList z{};
  auto add = [&](void* p, uint64_t bytes) {
    z.p[z.k] = p;
    z.n[z.k++] = bytes;
  };
  add(w.raw(), sizeof(RawRow) * (size_t)cap);
  if (!reuse) add(w.index(), sizeof(IndexEntry) * (size_t)w.L.slots);  // (dictionary rows only: reusable)
  add(w.tindex(), sizeof(Tuple) * (size_t)w.L.tslots);
  if (!reuse) add(w.samp(), sizeof(SampEntry) * (size_t)kSampSlots);  // (a reused plan keeps its
  add(w.misc(), 256);  // (dictionary word: none unless k_dict_load sets it)   hot sets and header)
  if (!reuse) add(w.hot_n(), 4ull * kHotHdr);
  add(w.cur(), 16ull * kSchedWords);  // cur, act, bstart, btot
  launch_pdl(k_zero, 2 * num_sms(), 256, 0, s, z, w.st());
  if (int r = launched()) return r;
  if (dict) {  // rows fixed in advance: dictionary key j -> row j
    launch_pdl(k_dict_load, (dict_n + 255) / 256, 256, 0, s, dict_kid, dict_task, dict_n, w.index(), w.L.slots, w.raw(),
                                                      w.st(), w.misc(), reuse ? 1u : 0u);
    if (int r = launched()) return r;
  }
  if (n == 0) return reuse ? FIKIT_OK : hash_strtabs(w, names, sigs, s);
  // persistent k_measure: one CTA per SM, fewer if there are not enough 64-launch warp-tiles
  const uint32_t ntiles = (uint32_t)((n + kTileLaunches - 1) / kTileLaunches);
  const uint32_t ngroups = (ntiles + kGroupTiles - 1) / kGroupTiles;
  uint64_t ctas = (ntiles + measure_threads() / 32 - 1) / (measure_threads() / 32);
  unsigned grid = (unsigned)(ctas < (uint64_t)num_sms() ? ctas : (uint64_t)num_sms());
  if (grid > kMaxCTAs) grid = kMaxCTAs;
  // 2. k_prep: string hashes | a ~64k-launch sample -> rows + counts | tile-group buckets
  PrepArgs pa{};
  pa.recs = reinterpret_cast<const uint4*>(recs);
  pa.recs_t = recs;
  pa.n = n;
  const uint64_t target = 65536;
  pa.stride = n > target ? n / target : 1;
  pa.n_samples = (n + pa.stride - 1) / pa.stride;
  pa.names = names;
  pa.sigs = sigs;
  pa.name_hash = w.name_hash();
  pa.sig_hash = w.sig_hash();
  pa.st = w.st();
  pa.samp = w.samp();
  pa.samp_list = w.samp_list();
  pa.samp_n = w.hot_n() + kSampN;
  pa.grp_bucket = w.grp_bucket();
  pa.blkcnt = w.blkcnt();
  pa.ngroups = ngroups;
  uint32_t sb = (ngroups + 511) / 512;  // group blocks: <= 512 groups (128k launches) each, <= 160
  sb = sb < 1 ? 1 : sb > kSortBlocks ? kSortBlocks : sb;
  pa.sb = sb;
  const uint64_t nstr = (uint64_t)names.count + sigs.count;
  // (a reused plan: the string hashes and the hot sets of the previous call; only the tile groups)
  pa.hot_hdr = w.hot_n();
  pa.reused_plan = reuse ? 1u : 0u;
  pa.nb_hash = reuse ? 0u : (uint32_t)((nstr + kPrepThreads / 32 - 1) / (kPrepThreads / 32));
  pa.nb_samp = reuse ? 0u : (uint32_t)((pa.n_samples + 2 * kPrepThreads - 1) / (2 * kPrepThreads));  // <= 2 per thread
  launch_pdl(k_prep, pa.nb_hash + pa.nb_samp + pa.sb, kPrepThreads, 0, s, pa);
  if (int r = launched()) return r;
  // 3. k_plan: hot sets + schedule mode | the groups' counting-sort scatter, bucket ranges, first buckets
  PlanArgs pl{};
  pl.st = w.st();
  pl.samp = w.samp();
  pl.samp_list = w.samp_list();
  pl.name_hash = w.name_hash();
  pl.sig_hash = w.sig_hash();
  pl.idx = w.index();
  pl.slots = w.L.slots;
  pl.raw = w.raw();
  pl.row_tuple = w.row_tuple();
  pl.cap = cap;
  pl.dict = dict ? 1u : 0u;
  pl.hot_blocks = reuse ? 0u : kBuckets + 1;
  pl.dict_hash = reinterpret_cast<const unsigned long long*>(w.misc() + kMiscDictHash);
  pl.hot_all = w.hot();
  pl.hot_hdr = w.hot_n();
  pl.grp_bucket = w.grp_bucket();
  pl.blkcnt = w.blkcnt();
  pl.ngroups = ngroups;
  pl.sb = sb;
  pl.grid_measure = grid;
  pl.order = w.order();
  pl.bstart = w.bstart();
  pl.btot = w.btot();
  pl.first = w.first();
  launch_pdl(k_plan, pl.hot_blocks + sb, 1024, 0, s, pl);
  if (int r = launched()) return r;
  // 4. the streaming kernel
  const size_t smem = measure_smem_bytes();
  // the dynamic shared-memory opt-in is a per-device function attribute
  if (dev_prop(kPropMeasureAttr, [&](int) {
        return cudaFuncSetAttribute(k_measure, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                       cudaSuccess
                   ? 1
                   : -1;
      }) < 0)
    return FIKIT_E_CUDA;
  if (ev0 && !record_ev(ev0, s)) return FIKIT_E_CUDA;
  launch_pdl(k_measure, grid, measure_threads(), smem, s, 
      recs, n, halo, w.name_hash(), w.sig_hash(), names.count, sigs.count, w.index(), w.L.slots, w.tindex(),
      w.L.tslots, w.st(), RawTab{w.raw(), cap}, w.row_tuple(), w.hot(), w.hot_n(), w.cur(), w.act(), w.bstart(),
      w.btot(), w.first(), w.order(), w.grp_bucket(), ntiles, out_row, dict ? 1u : 0u);
  if (int r = launched()) return r;
  if (ev1 && !record_ev(ev1, s)) return FIKIT_E_CUDA;
  return FIKIT_OK;
}

int fikit_measure(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                  fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, void* ws, size_t ws_bytes,
                  void* stream) {
  return measure_impl(recs, n, halo, names, sigs, tab, out_row, ws, ws_bytes, stream, nullptr, nullptr);
}

int fikit_measure_timed(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                        fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, void* ws,
                        size_t ws_bytes, void* stream, void* ev_start, void* ev_stop) {
  return measure_impl(recs, n, halo, names, sigs, tab, out_row, ws, ws_bytes, stream, (cudaEvent_t)ev_start,
                      (cudaEvent_t)ev_stop);
}

int fikit_measure_dict(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                       fikit_strtab_t sigs, const uint64_t* dict_kid, const uint32_t* dict_task, uint32_t dict_n,
                       const fikit_table_t* tab, uint32_t* out_row, void* ws, size_t ws_bytes, void* stream) {
  if (!dict_kid) return FIKIT_E_ARG;
  return measure_impl(recs, n, halo, names, sigs, tab, out_row, ws, ws_bytes, stream, nullptr, nullptr, dict_kid,
                      dict_task, dict_n);
}

int fikit_measure_dict_ex(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                          fikit_strtab_t sigs, const uint64_t* dict_kid, const uint32_t* dict_task, uint32_t dict_n,
                          uint32_t flags, const fikit_table_t* tab, uint32_t* out_row, void* ws, size_t ws_bytes,
                          void* stream, void* ev_start, void* ev_stop) {
  if (!dict_kid) return FIKIT_E_ARG;
  return measure_impl(recs, n, halo, names, sigs, tab, out_row, ws, ws_bytes, stream, (cudaEvent_t)ev_start,
                      (cudaEvent_t)ev_stop, dict_kid, dict_task, dict_n, flags);
}

int fikit_measure_dict_timed(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo,
                             fikit_strtab_t names, fikit_strtab_t sigs, const uint64_t* dict_kid,
                             const uint32_t* dict_task, uint32_t dict_n, const fikit_table_t* tab, uint32_t* out_row,
                             void* ws, size_t ws_bytes, void* stream, void* ev_start, void* ev_stop) {
  if (!dict_kid) return FIKIT_E_ARG;
  return measure_impl(recs, n, halo, names, sigs, tab, out_row, ws, ws_bytes, stream, (cudaEvent_t)ev_start,
                      (cudaEvent_t)ev_stop, dict_kid, dict_task, dict_n);
}

int fikit_table_finalize(const fikit_table_t* tab, uint32_t* out_row, uint64_t n, void* ws, size_t ws_bytes,
                         void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!table_ok(tab) || (n && !out_row) || n >= (1ull << 32)) return FIKIT_E_ARG;
  Ws w;
  if (int r = get_ws(ws, ws_bytes, tab->capacity, 0, 0, &w)) return r;  // (the capacity-sized regions)
  const uint32_t cap = tab->capacity;
  uint32_t* rank = w.rank();
  // sorted groups of G keys (one block each: G / 2 threads, one compare-exchange per stage): 256-key
  // groups up to 8192 rows (a 2048-key block sort costs ~20 us more there), 2048-key groups above
  // (every row's rank searches 8x fewer groups: Z64k's 65,536-row finalize 0.335 -> 0.151 ms)
  const uint32_t G = cap <= 8192 ? 256u : kFinGroup;
  if (G == 256)
    launch_pdl(k_fin_sort256, (cap + 255) / 256, 128, 0, s, w.st(), w.raw(), cap, *tab, w.fin_keys(cap), w.misc());
  else
    launch_pdl(k_fin_sort, (cap + kFinGroup - 1) / kFinGroup, kFinGroup / 2, 0, s, w.st(), w.raw(), cap, *tab,
               w.fin_keys(cap), w.misc());
  if (int r = launched()) return r;
  // rows per scatter block: at most R (the shared-memory size, >= cap / num_sms), on the device
  // min(R, max(16, K / num_sms)) -- so a table far below its capacity (ResNet-like: 96 rows of 4096)
  // still spreads its rows over several blocks (finalize 18.6 -> 14.4 us there); one block per SM
  uint32_t R = (cap + num_sms() - 1) / num_sms();
  R = R < 64 ? 64 : R > 4096 ? 4096 : (R + 31) / 32 * 32;
  const size_t fsm = (sizeof(FinKey) + 4) * (size_t)R;  // row keys + ranks
  if (dev_prop(kPropFinAttr, [&](int) {
        return cudaFuncSetAttribute(k_fin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)((sizeof(FinKey) + 4) * 4096)) == cudaSuccess
                   ? 1
                   : -1;
      }) < 0)
    return FIKIT_E_CUDA;
  launch_pdl(k_fin_scatter, (unsigned)num_sms(), 256, fsm, s, w.st(), w.raw(), cap, R, w.fin_keys(cap), G, *tab, rank,
                                                    w.misc());
  if (int r = launched()) return r;
  if (out_row && n) {
    launch_pdl(k_remap_rows, grid_for(n, 256, num_sms() * 8), 256, 0, s, out_row, n, rank, tab->n_rows);
    if (int r = launched()) return r;
  }
  return FIKIT_OK;
}

int fikit_table_means(const fikit_table_t* tab, void* stream) {
  if (!table_ok(tab)) return FIKIT_E_ARG;
  k_means<<<(tab->capacity + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*tab);
  return launched();
}

int fikit_table_predict(const fikit_table_t* tab, uint32_t mode, uint32_t pct, void* stream) {
  if (!table_ok(tab) || mode > FIKIT_PREDICT_EXTREMES ||
      (mode == FIKIT_PREDICT_PERCENTILE && (pct < 1 || pct > 99)))
    return FIKIT_E_ARG;
  k_predict<<<(tab->capacity + 7) / 8, 256, 0, (cudaStream_t)stream>>>(*tab, mode, pct);  // a warp per row
  return launched();
}

static int resolve_impl(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                        fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, uint64_t* out_dur,
                        uint64_t* out_gap, void* ws, size_t ws_bytes, void* stream, uint32_t flags) {
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  if (n >= (1ull << 32) || (n && (!recs || !aligned(recs, 16) || !out_row || !out_dur || !out_gap)) ||
      !strtab_ok(names) || !strtab_ok(sigs) || !table_ok(tab) || (flags & ~FIKIT_RESOLVE_REUSE_HASHES))
    return FIKIT_E_ARG;
  // the measure call's layout (its string hashes) when the workspace holds a table of this capacity
  const bool measure_layout =
      ws && ws_bytes >= ws_layout(tab->capacity, names.count, sigs.count, 0).total;
  if ((flags & FIKIT_RESOLVE_REUSE_HASHES) && !measure_layout) return FIKIT_E_ARG;
  if (int r = get_ws(ws, ws_bytes, measure_layout ? tab->capacity : 1, names.count, sigs.count, &w)) return r;
  if (int r = reset_status(w, s)) return r;
  if (!(flags & FIKIT_RESOLVE_REUSE_HASHES))
    if (int r = hash_strtabs(w, names, sigs, s)) return r;
  if (n == 0) return FIKIT_OK;
  const size_t smem = sizeof(uint4) * (kResolveThreads / 32) * 99 + 12ull * kResolveSmemKeys;
  if (dev_prop(kPropResolveAttr, [&](int) {
        return cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess
                   ? 1
                   : -1;
      }) < 0)
    return FIKIT_E_CUDA;
  const uint64_t nchunks = (n + 31) / 32;
  const uint64_t blocks = (nchunks + kResolveThreads / 32 - 1) / (kResolveThreads / 32);
  launch_pdl(k_resolve, (unsigned)(blocks < (uint64_t)num_sms() ? blocks : (uint64_t)num_sms()), kResolveThreads,
             smem, s, reinterpret_cast<const uint4*>(recs), n, halo, w.name_hash(), w.sig_hash(), names.count,
             sigs.count, *tab, out_row, out_dur, out_gap, w.st());
  return launched();
}

int fikit_resolve(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                  fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, uint64_t* out_dur,
                  uint64_t* out_gap, void* ws, size_t ws_bytes, void* stream) {
  return resolve_impl(recs, n, halo, names, sigs, tab, out_row, out_dur, out_gap, ws, ws_bytes, stream, 0u);
}

int fikit_resolve_ex(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo, fikit_strtab_t names,
                     fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, uint64_t* out_dur,
                     uint64_t* out_gap, uint32_t flags, void* ws, size_t ws_bytes, void* stream) {
  return resolve_impl(recs, n, halo, names, sigs, tab, out_row, out_dur, out_gap, ws, ws_bytes, stream, flags);
}

int fikit_lookup(const fikit_table_t* tab, const uint64_t* kid, const uint32_t* task, uint64_t n, uint32_t* out_row,
                 void* stream) {
  if (!table_ok(tab) || (n && (!kid || !task || !out_row))) return FIKIT_E_ARG;
  if (n == 0) return FIKIT_OK;
  k_lookup<<<grid_for(n, 256, num_sms() * 8), 256, 0, (cudaStream_t)stream>>>(*tab, kid, task, n, out_row);
  return launched();
}

int fikit_fill(const fikit_table_t* tab, const uint64_t* R0, const uint64_t* deadline, const uint32_t* pool_row,
               const uint64_t* pool_dur, const uint8_t* pool_level, const uint32_t* pool_off,
               const uint32_t* pool_len, uint32_t G, fikit_fill_params_t prm, uint32_t* picks,
               const uint32_t* picks_off, uint32_t* n_picks, uint64_t* R_left, uint64_t* t_used, void* ws,
               size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  if (!table_ok(tab) || (G && (!R0 || !deadline || !pool_off || !pool_len || !picks_off || !n_picks || !R_left ||
                               !t_used)))
    return FIKIT_E_ARG;
  if (int r = get_ws(ws, ws_bytes, 1, 0, 0, &w)) return r;
  if (int r = reset_status(w, s)) return r;
  if (G == 0) return FIKIT_OK;
  launch_pdl(k_fill, grid_for(G, 4, num_sms() * 16), 128, 0, s, *tab, R0, deadline, pool_row, pool_dur, pool_level, pool_off,
                                                         pool_len, G, prm, picks, picks_off, n_picks, R_left, t_used,
                                                         w.st());
  return launched();
}

// persistent grid: blocks of one full wave of the kernel at its occupancy (per device)
static int one_wave(int which, const void* kernel, int threads) {
  return dev_prop(which, [&](int) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0) != cudaSuccess || occ < 1) occ = 1;
    return occ * num_sms();
  });
}

int fikit_simulate_batch(const fikit_table_t* tab, const uint32_t* hp_row, const uint64_t* hp_dur,
                         const uint64_t* hp_gap, const uint32_t* lp_row, const uint64_t* lp_dur,
                         const uint8_t* lp_level, const fikit_scenario_t* sc, uint32_t S, fikit_fill_params_t prm,
                         fikit_result_t* out, int32_t* fill_gap, uint64_t* lp_start, const uint64_t* sched_off,
                         void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  if (!table_ok(tab) || (S && (!sc || !out))) return FIKIT_E_ARG;
  if (int r = get_ws(ws, ws_bytes, 1, 0, 0, &w)) return r;
  if (int r = reset_status(w, s)) return r;
  if (S == 0) return FIKIT_OK;
  // pass 1: register-pool scenarios (m <= 64); pass 2: the ones it deferred (shared-memory pool).
  // Both persistent: one wave of the kernel's occupancy.
  const int g1 = one_wave(kPropWaveReg, simulate_reg_kernel(false), kRegThreads);
  const int g2 = one_wave(kPropWaveSmem, simulate_smem_kernel(false), kSimThreads);
  const uint64_t n1 = ((uint64_t)S + kRegThreads / 32 - 1) / (kRegThreads / 32);
  const uint64_t n2 = ((uint64_t)S + kSimThreads / 32 - 1) / (kSimThreads / 32);
  const int b1 = (int)(n1 < (uint64_t)g1 ? n1 : (uint64_t)g1);
  const int b2 = (int)(n2 < (uint64_t)g2 ? n2 : (uint64_t)g2);
  launch_simulate_reg(b1, kRegThreads, s, *tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, S, prm, out,
                      fill_gap, lp_start, sched_off, w.st());
  if (int r = launched()) return r;
  launch_simulate_smem(b2, kSimThreads, s, *tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, S, prm, out,
                       fill_gap, lp_start, sched_off, w.st());
  return launched();
}

int fikit_simulate_stream_batch(const fikit_table_t* tab, const uint32_t* hp_row, const uint64_t* hp_dur,
                                const uint64_t* hp_gap, const uint32_t* lp_row, const uint64_t* lp_dur,
                                const uint8_t* lp_level, const uint32_t* lp_stream, const uint64_t* lp_think,
                                const uint64_t* hp_arrival, const fikit_scenario_t* sc, uint32_t S,
                                fikit_fill_params_t prm, fikit_result_t* out,
                                int32_t* fill_gap, uint64_t* lp_start, const uint64_t* sched_off, void* ws,
                                size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Ws w;
  if (!table_ok(tab) || (S && (!sc || !out))) return FIKIT_E_ARG;
  if (int r = get_ws(ws, ws_bytes, 1, 0, 0, &w)) return r;
  if (int r = reset_status(w, s)) return r;
  if (S == 0) return FIKIT_OK;
  // persistent, one wave; warps claim scenarios from a counter
  const int g = one_wave(kPropWaveStream, simulate_stream_kernel(false), kStreamThreads);
  const uint64_t need = ((uint64_t)S + kStreamThreads / 32 - 1) / (kStreamThreads / 32);
  const int b = (int)(need < (uint64_t)g ? need : (uint64_t)g);
  launch_simulate_stream(b, kStreamThreads, s, *tab, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, lp_stream,
                         lp_think, hp_arrival, sc, S, prm, out, fill_gap, lp_start, sched_off, w.st());
  return launched();
}

int fikit_dict_union(const uint64_t* all_kid, const uint32_t* all_task, const uint32_t* n_list, uint32_t P,
                     uint32_t Kmax, uint32_t self_rank, uint64_t* out_kid, uint32_t* out_task, uint32_t cap_out,
                     uint32_t* out_n, uint32_t* local_to_union, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!all_kid || !all_task || !n_list || P == 0 || P > 1024 || Kmax == 0 || self_rank >= P || !out_kid ||
      !out_task || !out_n || !local_to_union || cap_out == 0)
    return FIKIT_E_ARG;
  Ws w;
  if (int r = get_ws(ws, ws_bytes, 1, 0, 0, &w)) return r;
  // scratch: canon [P][Kmax] + cpre [P][Kmax+1]
  size_t need = w.L.fin + 4ull * P * Kmax + 4ull * P * (Kmax + 1);
  if (ws_bytes < need) return FIKIT_E_ARG;
  uint32_t* canon = reinterpret_cast<uint32_t*>(w.fin());
  uint32_t* cpre = canon + (size_t)P * Kmax;
  if (int r = reset_status(w, s)) return r;
  dim3 g((Kmax + 255) / 256, P);
  k_union_flags<<<g, 256, 0, s>>>(all_kid, all_task, n_list, P, Kmax, canon);
  if (int r = launched()) return r;
  k_union_scan<<<P, 1024, 0, s>>>(canon, Kmax, cpre);
  if (int r = launched()) return r;
  k_union_place<<<g, 256, 0, s>>>(all_kid, all_task, n_list, P, Kmax, self_rank, canon, cpre, out_kid, out_task,
                                  cap_out, out_n, local_to_union, w.st());
  return launched();
}

int fikit_table_remap(const fikit_table_t* local, const uint32_t* l2u, const uint64_t* ukid, const uint32_t* utask,
                      const uint32_t* un, const fikit_table_t* dense, void* stream) {
  if (!table_ok(local) || !table_ok(dense) || !l2u || !ukid || !utask || !un) return FIKIT_E_ARG;
  uint32_t m = local->capacity > dense->capacity ? local->capacity : dense->capacity;
  k_table_remap<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*local, l2u, ukid, utask, un, *dense);
  return launched();
}

int fikit_table_bias(const fikit_table_t* tab, void* stream) {
  if (!table_ok(tab)) return FIKIT_E_ARG;
  k_table_bias<<<grid_for(4ull * tab->capacity, 256, num_sms() * 4), 256, 0, (cudaStream_t)stream>>>(*tab);
  return launched();
}

static_assert(sizeof(fikit_status_t) <= 64, "status lives in the first 64 workspace bytes");

int fikit_get_status(const void* ws, fikit_status_t* out, void* stream) {
  if (!ws || !out) return FIKIT_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(out, ws, sizeof(fikit_status_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return FIKIT_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return FIKIT_E_CUDA;
  uint32_t f = out->flags;
  out->code = (f & kStatusArg)        ? FIKIT_E_ARG
              : (f & kStatusName)     ? FIKIT_E_NAME
              : (f & kStatusRecord)   ? FIKIT_E_RECORD
              : (f & kStatusDict)     ? FIKIT_E_DICT
              : (f & kStatusCapacity) ? FIKIT_E_CAPACITY
                                      : FIKIT_OK;
  return out->code;
}

const char* fikit_strerror(int code) {
  switch (code) {
    case FIKIT_OK: return "ok";
    case FIKIT_E_ARG: return "invalid argument";
    case FIKIT_E_RECORD: return "invalid launch record";
    case FIKIT_E_CAPACITY: return "statistic table capacity exceeded";
    case FIKIT_E_CUDA: return "CUDA launch failure";
    case FIKIT_E_NAME: return "empty kernel name";
    case FIKIT_E_DICT: return "launch identity not in the supplied dictionary";
    default: return "unknown";
  }
}

uint64_t fikit_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
