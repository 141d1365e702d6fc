/*
 * fikit.h -- C-ABI of libfikit.so, the B200 (sm_100a) hot path of FIKIT
 * (arXiv 2311.10359, "FIKIT: Priority-Based Real-time GPU Multi-tasking
 * Scheduling with Kernel Identification").  PAPER.md line numbers = P:<n>.
 *
 * The library computes, over traces of kernel launches with integer
 * nanosecond timestamps:
 *   identify  -- the kernel ID of every launch
 *   measure   -- per-ID duration and following-gap statistics
 *   finalize  -- S_UID in canonical order, SK_j and SG_j
 *   resolve   -- profile lookup of fresh launches              (Alg.1 lines 3-5)
 *   fill      -- Algorithm 1 (FIKIT) + Algorithm 2 (BestPrioFit) on independent gaps
 *   simulate  -- batch replay of HP/LP scenarios with runtime feedback
 *   dict/remap-- multi-GPU merge of per-rank tables (the NCCL collectives are the caller's)
 *
 * Conventions (all entry points):
 *  - Every array pointer is a DEVICE pointer owned by the caller, unless the
 *    argument says "host".  The library never allocates persistent memory;
 *    scratch lives in the caller's workspace `ws` of `ws_bytes` bytes
 *    (fikit_ws_bytes), which must be 256-byte aligned.
 *  - Every call is stream-ordered and asynchronous on `stream` (a
 *    cudaStream_t passed as void*) and runs on the calling thread's current
 *    device.  The only process-wide state is (a) per-device caches of
 *    immutable properties (SM count, occupancy, the k_measure shared-memory
 *    opt-in), computed idempotently and published atomically, and (b) the
 *    launch counter (fikit_launch_count).  Calls on different streams (or
 *    devices, or host threads) with distinct workspaces may run concurrently.
 *    No call allocates, and none but fikit_get_status (which copies the
 *    status back and synchronises the stream) synchronises the host, so a
 *    sequence of the other calls can be captured into a CUDA graph
 *    (cudaStreamBeginCapture) and replayed; the launch counter counts
 *    launches at capture, not at replay.
 *  - The return value is a HOST status checked before any launch:
 *    FIKIT_OK, FIKIT_E_ARG (null / misaligned pointer, n >= 2^32, workspace
 *    too small) or FIKIT_E_CUDA (launch failure).
 *  - Data errors are detected on the device and accumulated in the
 *    workspace status (fikit_status_t), reset by every call that validates
 *    records (identify, measure, resolve, fill, simulate) and read with
 *    fikit_get_status().  Precedence: E_ARG > E_NAME > E_RECORD > E_DICT > E_CAPACITY.
 *    Outputs of a call whose status is not FIKIT_OK are unspecified.
 *  - All times are unsigned 64-bit nanoseconds; sums wrap mod 2^64 (R10).
 *  - "R<k>" = reading k of a silent/garbled passage, DESIGN.md §Readings.
 */
#ifndef FIKIT_H
#define FIKIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FIKIT_OK = 0,
  FIKIT_E_ARG = -1,      /* bad argument (host check) or malformed string table (device) */
  FIKIT_E_RECORD = -2,   /* invalid record / LP level; first_bad_index = smallest such index */
  FIKIT_E_CAPACITY = -3, /* more distinct (task, kernel) rows than table capacity; n_rows_needed */
  FIKIT_E_CUDA = -4,     /* kernel launch failed */
  FIKIT_E_NAME = -5,     /* empty kernel name in the names table (SPEC) */
  FIKIT_E_DICT = -6      /* fikit_measure_dict: a launch identity is not in the supplied dictionary;
                            first_missing_index = smallest such launch index */
};

#define FIKIT_NBINS 32         /* log2 histogram bins per statistic (R9) */
#define FIKIT_NO_ROW 0xFFFFFFFFu

/* One kernel launch (D2 of SURVEY: ID_{t,i}, K, G), 48 bytes, 16-byte aligned
 * arrays.  Valid iff all six dims >= 1, name_id < names.count,
 * sig_id < sigs.count, flags == 0 and end_ns >= start_ns (R4). */
typedef struct {
  uint64_t start_ns, end_ns; /* device timestamps of the launch ("cuda event") */
  uint32_t name_id;          /* index into the names table (kernel function name) */
  uint32_t sig_id;           /* index into the signatures table (argument types; "" = paper's ID, R1) */
  uint32_t grid_x;
  uint16_t grid_y, grid_z;
  uint16_t block_x, block_y, block_z;
  uint16_t flags;   /* reserved, must be 0 */
  uint32_t run_id;  /* t: the run (inference) index */
  uint32_t task_id; /* caller-interned Task Key */
} fikit_record_t;

/* count strings; string j = bytes[offsets[j] .. offsets[j+1]) (device arrays).
 * The kernels read `bytes` in whole aligned 16-byte blocks (any block holding a
 * string byte), which device allocations (>= 256-byte granularity) always allow. */
typedef struct {
  const uint8_t* bytes;
  const uint32_t* offsets; /* count + 1 entries, non-decreasing */
  uint32_t count;
} fikit_strtab_t;

/* Per-(task, kernel ID) statistic table, SoA over `capacity` rows, caller-owned
 * device memory.  Blocks are grouped by their multi-GPU reduction operator:
 *   sums[cap][4]  u64 SUM : dur_cnt, dur_sum, gap_cnt, gap_sum  (SK/SG numerators and denominators,
 *                           P:249; counts are written by finalize)
 *   hist[cap][64] u32 SUM : duration bins 0..31, gap bins 32..63; bin(v) = min(31, bit_length(v)) (R9)
 *   ext[cap][4]   u64 MAX : dur_max, dur_nmin, gap_max, gap_nmin with nmin = ~min, so an all-zero row is
 *                           the identity of every reduction (empty min = 2^64-1, max = 0)
 *   mean[cap][2]  u64     : SK_j (dur_mean), SG_j (gap_mean), round half up (R8); written by finalize
 * fikit_measure zeroes the table first.  Rows are in racy order until
 * fikit_table_finalize sorts them by (task_id, kernel_id) (R11). */
typedef struct {
  uint64_t* kernel_id; /* [cap] */
  uint32_t* task_id;   /* [cap] */
  uint64_t* sums;      /* [cap*4] */
  uint32_t* hist;      /* [cap*64] */
  uint64_t* ext;       /* [cap*4] */
  uint64_t* mean;      /* [cap*2] */
  uint32_t* n_rows;    /* [1] device */
  uint32_t capacity;
} fikit_table_t;

/* device-side status in the workspace (first 64 bytes) */
typedef struct {
  int32_t code;             /* derived by fikit_get_status from the flag word */
  uint32_t flags;           /* bit0 ARG, bit1 NAME, bit2 RECORD, bit3 CAPACITY */
  uint64_t first_bad_index; /* E_RECORD: smallest invalid index (deterministic: atomicMin) */
  uint64_t n_rows_needed;   /* measure: number of distinct (task, kernel ID) rows seen */
  uint64_t n_overlap_gaps;  /* measure/resolve: gaps clamped from negative to 0 (R5) */
  uint32_t schedule;        /* measure: 0 = address-order sweep with one global hot set,
                               1 = warp-tiles sorted by task bucket, per-bucket hot sets */
  uint32_t n_task_buckets;  /* measure, schedule 1: non-empty task buckets */
  uint64_t first_missing_index; /* fikit_measure_dict: smallest launch index whose (task, kernel ID)
                                   is not in the dictionary (E_DICT); ~0 if none */
} fikit_status_t;

/* Scenario of the batch replay: HP template kernels [hp_off, hp_off+hp_len) and
 * LP requests [lp_off, lp_off+lp_len) of the SoA kernel arrays, gap scale Q16 (R24). */
typedef struct {
  uint32_t hp_off, hp_len, lp_off, lp_len, gap_scale_q16, pad;
} fikit_scenario_t;

typedef struct {
  uint64_t threshold_ns; /* Alg.1 lines 6-8: skip predicted gaps < 0.1 ms; default 100000 */
  uint32_t feedback;     /* runtime feedback / early stop; default 1 */
  uint32_t flags;        /* reserved, 0 */
} fikit_fill_params_t;

typedef struct {
  uint64_t hp_jct;    /* end of the last HP kernel (JCT; R23) */
  uint64_t lp_jct;    /* max end over LP requests (all arrive at 0; R22); 0 if m = 0 */
  uint64_t hp_delay;  /* sum over gaps of max(0, fill end - HP arrival): "overhead 2" of P:362 */
  uint64_t fill_work; /* sum of actual e over fills */
  uint64_t digest;    /* sum_k MIX(k ^ (fill_gap[k]+1)<<32 ^ MIX(lp_start[k])) mod 2^64 (checksum) */
  uint32_t n_fills, n_tail;
} fikit_result_t;

/* ---- sizes ---------------------------------------------------------------- */
/* Workspace bytes for tables of `capacity` rows (<= 2^24), string tables of up to
 * n_names / n_sigs entries, and fikit_measure calls of up to n_records launches
 * (its task-partitioned tile schedule: ~5 bytes per 32 launches); the same workspace
 * serves every call. */
size_t fikit_ws_bytes(uint32_t capacity, uint32_t n_names, uint32_t n_sigs, uint64_t n_records);
/* Device bytes of a table of `capacity` rows when allocated as one block
 * (layout of fikit_table_carve). */
size_t fikit_table_bytes(uint32_t capacity);
/* Point a table's arrays into one 256-byte aligned device block of
 * fikit_table_bytes(capacity) bytes: sums, hist and ext each contiguous, so a
 * collective can reduce each block in one call.  Host-only, no launch. */
int fikit_table_carve(void* block, uint32_t capacity, fikit_table_t* out /* host */);

/* ---- identify --------------------------------------------------
 * out_kernel_id[i] = KID(name bytes, signature bytes, grid, block) of record i:
 *   KID = MIX(MIX(MIX(FNV1a64(name) ^ FNV1a64(sig)) ^ w1) ^ w2), 0 -> 1   (R2)
 *   w1 = grid_x | grid_y<<32 | grid_z<<48,  w2 = block_x | block_y<<16 | block_z<<32,
 *   MIX = splitmix64 finaliser.  The ID is independent of the launch's position
 * and run.  recs: n records (16-B aligned).  Errors: E_NAME, E_RECORD. */
int fikit_identify(const fikit_record_t* recs, uint64_t n, fikit_strtab_t names, fikit_strtab_t sigs,
                   uint64_t* out_kernel_id, void* ws, size_t ws_bytes, void* stream);

/* ---- measure ---------------------------------------------------
 * Zeroes *tab, then for every record i accumulates into row (task_id, KID_i):
 * duration K = end - start and, iff the next launch (record i+1, or
 * *halo_next after the last record; nullable) has the same (task_id, run_id),
 * the following gap G = max(0, start_{i+1} - end_i) (R5).  Per statistic:
 * sum, min, max, 32-bin histogram (counts = histogram totals, set by finalize).
 * out_row (nullable) receives each record's row; it becomes the canonical row
 * after fikit_table_finalize(tab, out_row, n).  Errors: E_NAME, E_RECORD,
 * E_CAPACITY (n_rows_needed = distinct rows).  The halo record is not validated. */
int fikit_measure(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next, fikit_strtab_t names,
                  fikit_strtab_t sigs, const fikit_table_t* tab /* host struct, device arrays */,
                  uint32_t* out_row, void* ws, size_t ws_bytes, void* stream);

/* ---- measure against a supplied dictionary (SURVEY §8e "B200-native upgrade": repeated
 * services keep their kernel IDs from run to run) ------------------------------------
 * As fikit_measure, but the table's rows are fixed in advance: row j is the j-th key
 * (dict_task[j], dict_kid[j]) of the dictionary, dict_n keys (host value, 1 <= dict_n <=
 * tab->capacity) in strictly increasing canonical order (task_id, then kernel_id; R11) --
 * e.g. the kernel_id / task_id columns of an earlier finalized or merged table.  No row is
 * created: a launch whose (task, KID) is absent sets FIKIT_E_DICT (first_missing_index) and is
 * not counted.  The following fikit_table_finalize keeps the dictionary order (no sort; n_rows =
 * dict_n, rows without launches have count 0, mean 0, min 2^64-1, max 0), so tables measured
 * against one dictionary on several ranks merge by two all-reduces alone (fikit_table_bias,
 * SUM over sums + hist, MAX over ext, fikit_table_bias, fikit_table_means): no key exchange, no
 * union, no remap.  A dictionary that is not strictly increasing sets FIKIT_E_ARG. */
int fikit_measure_dict(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next, fikit_strtab_t names,
                       fikit_strtab_t sigs, const uint64_t* dict_kid, const uint32_t* dict_task, uint32_t dict_n,
                       const fikit_table_t* tab, uint32_t* out_row, void* ws, size_t ws_bytes, void* stream);
/* fikit_measure_dict with flags and (nullable) fikit_measure_timed events.
 * FIKIT_MEASURE_REUSE_PLAN: keep the string hashes and the hot sets (the most-sampled launch
 * identities per task bucket, with their dictionary rows) of the previous fikit_measure_dict
 * call on this workspace -- repeated services keep their kernels, so a step skips the
 * launch sample, the hot-set choice and the string hashing; only the tile schedule is rebuilt
 * from the new records.  Requires: that previous call used the same dictionary (checked: a
 * different dictionary sets FIKIT_E_ARG in the status), the same string tables (same device
 * bytes, unchanged) and a table of the same capacity.  The statistics are exact either way; a
 * stale plan only makes more launches take the cold path. */
#define FIKIT_MEASURE_REUSE_PLAN 1u
int fikit_measure_dict_ex(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next,
                          fikit_strtab_t names, fikit_strtab_t sigs, const uint64_t* dict_kid,
                          const uint32_t* dict_task, uint32_t dict_n, uint32_t flags, const fikit_table_t* tab,
                          uint32_t* out_row, void* ws, size_t ws_bytes, void* stream, void* ev_start, void* ev_stop);
/* fikit_measure_dict with fikit_measure_timed's events around the streaming kernel. */
int fikit_measure_dict_timed(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next,
                             fikit_strtab_t names, fikit_strtab_t sigs, const uint64_t* dict_kid,
                             const uint32_t* dict_task, uint32_t dict_n, const fikit_table_t* tab, uint32_t* out_row,
                             void* ws, size_t ws_bytes, void* stream, void* ev_start, void* ev_stop);

/* ---- finalize --------------------------------------------------
 * Sorts the rows of a measured table by (task_id asc, kernel_id asc) (R11),
 * sets n_rows, dur_cnt/gap_cnt (histogram totals) and SK_j / SG_j =
 * floor(sum/cnt) + [2(sum mod cnt) >= cnt] (R8; cnt = 0 -> 0).  If out_row is
 * non-null its n entries are remapped to canonical rows.  Must follow the
 * fikit_measure (or fikit_measure_dict: dictionary order kept) that filled `tab` with the same
 * workspace. */
int fikit_table_finalize(const fikit_table_t* tab, uint32_t* out_row, uint64_t n, void* ws, size_t ws_bytes,
                         void* stream);

/* fikit_measure, instrumented: ev_start / ev_stop (cudaEvent_t, created by the caller, may
 * be null) are recorded on `stream` just before and after the fused streaming kernel
 * (k_measure), so a benchmark can time the dominant kernel alone inside a live step.  Inside a
 * stream capture they are recorded as external event nodes (cudaEventRecordExternal), so they
 * time the kernel on every replay of the captured graph. */
int fikit_measure_timed(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next,
                        fikit_strtab_t names, fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row,
                        void* ws, size_t ws_bytes, void* stream, void* ev_start, void* ev_stop);

/* Recompute counts and means of an already canonical table (after a multi-GPU merge). */
int fikit_table_means(const fikit_table_t* tab, void* stream);

/* ---- predictor variants ("dynamic duration and idling
 * prediction", readings R26-R28) -------------------------------------------------
 * Rewrites the predictions a finalized table gives the replay (mean[r*2] = the
 * predicted duration q of Alg.1 line 4, mean[r*2+1] = the predicted gap p of
 * line 3) for every row r < n_rows, from the row's counts, histogram and extremes:
 *   FIKIT_PREDICT_MEAN        SK, SG (what finalize / table_means write; R8)
 *   FIKIT_PREDICT_PERCENTILE  b_P = the smallest bin with 100*cum(b) >= P*count:
 *                             duration = min(upper edge of b_P, max), gap =
 *                             max(lower edge of b_(100-P), min); 1 <= pct <= 99
 *   FIKIT_PREDICT_EXTREMES    duration = max, gap = min
 * A row without samples predicts 0.  Device arrays of `tab` are read and written
 * in place; stream-ordered.  Errors: FIKIT_E_ARG (bad table, mode or pct). */
#define FIKIT_PREDICT_MEAN 0u
#define FIKIT_PREDICT_PERCENTILE 1u
#define FIKIT_PREDICT_EXTREMES 2u
int fikit_table_predict(const fikit_table_t* tab, uint32_t mode, uint32_t pct, void* stream);

/* ---- resolve (Alg. 1 lines 3-5) ------------------------------------
 * For fresh launches (HP template runs, LP requests): out_row[i] = canonical
 * row of (task_id, KID_i) in the finalized table or FIKIT_NO_ROW;
 * out_dur[i] = end - start; out_gap[i] = following gap as in measure (0 if
 * none).  Errors: E_NAME, E_RECORD. */
int fikit_resolve(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next, fikit_strtab_t names,
                  fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, uint64_t* out_dur,
                  uint64_t* out_gap, void* ws, size_t ws_bytes, void* stream);

/* fikit_resolve with flags.  FIKIT_RESOLVE_REUSE_HASHES: skip hashing the string tables --
 * the workspace already holds their hashes because the previous fikit_measure /
 * fikit_measure_dict / fikit_resolve on this workspace hashed the SAME tables (same device
 * bytes, unchanged) with a table of tab->capacity rows; requires a workspace sized for that
 * capacity (FIKIT_E_ARG otherwise).  One measure + two resolves of a step hash the strings once. */
#define FIKIT_RESOLVE_REUSE_HASHES 1u
int fikit_resolve_ex(const fikit_record_t* recs, uint64_t n, const fikit_record_t* halo_next, fikit_strtab_t names,
                     fikit_strtab_t sigs, const fikit_table_t* tab, uint32_t* out_row, uint64_t* out_dur,
                     uint64_t* out_gap, uint32_t flags, void* ws, size_t ws_bytes, void* stream);

/* out_row[i] = canonical row of (task[i], kid[i]) or FIKIT_NO_ROW (binary search). */
int fikit_lookup(const fikit_table_t* tab, const uint64_t* kid, const uint32_t* task, uint64_t n, uint32_t* out_row,
                 void* stream);

/* ---- fill: Algorithm 1 + 2 on G independent gaps ----
 * Gap g: predicted idle R0[g]; requests pool_*[pool_off[g] .. +pool_len[g])
 * with predicted duration q = SK of pool_row (absent row -> never a fill,
 * R16), actual duration pool_dur, level pool_level in [1,9].  Time t starts
 * at 0 (the HP kernel's end).  If R0 >= threshold: repeat { if feedback and
 * t >= deadline[g]: stop;  k = BestPrioFit(R) = argmin over alive eligible
 * q <= R of (level, -q, pool index);  none: stop;  t += e_k; R -= q_k }.
 * picks[picks_off[g] ..] = pool-local indices in dispatch order; n_picks[g],
 * R_left[g], t_used[g] = t.  Errors: E_RECORD (level outside [1,9]).
 * Limit: pool_len[g] <= 1024 (a warp's shared-memory pool); a longer pool sets
 * FIKIT_E_ARG in the status and gap g's outputs are left unwritten. */
int fikit_fill(const fikit_table_t* tab, const uint64_t* R0, const uint64_t* deadline, const uint32_t* pool_row,
               const uint64_t* pool_dur, const uint8_t* pool_level, const uint32_t* pool_off,
               const uint32_t* pool_len, uint32_t G, fikit_fill_params_t params, uint32_t* picks,
               const uint32_t* picks_off, uint32_t* n_picks, uint64_t* R_left, uint64_t* t_used, void* ws,
               size_t ws_bytes, void* stream);

/* ---- simulate: batch replay of S scenarios (Case B) ----
 * HP kernels (hp_row, hp_dur = d_i, hp_gap = a_i: the HP client's think time
 * after kernel i), LP requests (lp_row, lp_dur = e_k, lp_level).  Scenario s
 * replays, with scale s_q16: t = 0; for each HP kernel i: start = max(t, r_i),
 * t = end_i = start + d_i; then (i < n_h-1) r_{i+1} = end_i + (a_i*s>>16),
 * p_i = (SG(row_i)*s>>16), and Alg. 1 fills the gap from t with deadline
 * r_{i+1}; remaining requests run after the HP job in (level, index) order.
 * Writes out[s]; if fill_gap/lp_start are non-null, scenario s's m entries go
 * to [sched_off[s], sched_off[s]+m): gap index i of the fill or -1 (tail), and
 * start time.  Errors: E_RECORD (level outside [1,9]).
 * Limit: lp_len <= 1024 per scenario (a warp's shared-memory pool); a longer
 * window sets FIKIT_E_ARG in the status and that scenario's out[s] is left
 * unwritten (the other scenarios are replayed). */
int fikit_simulate_batch(const fikit_table_t* tab, const uint32_t* hp_row, const uint64_t* hp_dur,
                         const uint64_t* hp_gap, const uint32_t* lp_row, const uint64_t* lp_dur,
                         const uint8_t* lp_level, const fikit_scenario_t* sc, uint32_t S, fikit_fill_params_t params,
                         fikit_result_t* out, int32_t* fill_gap, uint64_t* lp_start, const uint64_t* sched_off,
                         void* ws, size_t ws_bytes, void* stream);

/* ---- STREAM-model replay (readings R29-R32) ----------------
 * As fikit_simulate_batch, but the LP requests of a scenario are kernel streams
 * (a hooked client has one launch in flight): a stream
 * is a maximal run of equal consecutive lp_stream[] ids in the scenario's window
 * (device u32 per LP request); only each stream's first undispatched request is
 * queued.  Streams' first requests arrive at t = 0; request k+1 arrives
 * lp_think[k] ns (device u64 per LP request, e.g. fikit_resolve's out_gap of
 * the LP launches) after request k ends.  In a gap, BestPrioFit runs over the
 * arrived heads; when none fits the scheduler waits for the next arrival A if
 * A - t <= R (and, with feedback, A < r_{i+1}), consuming R by the wait.  After
 * the HP job the rest runs in (level, index) order among arrived heads.
 * Case A (§8f row 2; R33-R34): hp_arrival (device u64 per
 * scenario, nullable = 0) is when the HP job arrives; before it the LP streams
 * hold the GPU (arrived heads in (level, index) order), an LP kernel launches
 * only before hp_arrival and the running one is not preempted: HP kernel 0
 * starts at max(hp_arrival, its end).  hp_jct stays absolute; LP kernels run
 * before the HP job count in neither n_fills nor n_tail.
 * Results, schedule and digest as fikit_simulate_batch.  Limits: m <= 1024 and
 * <= 64 streams per scenario (else FIKIT_E_ARG in the status and that
 * scenario's out[s] is left unwritten; singleton streams are the POOL model:
 * use fikit_simulate_batch).  One warp per scenario. */
int fikit_simulate_stream_batch(const fikit_table_t* tab, const uint32_t* hp_row, const uint64_t* hp_dur,
                                const uint64_t* hp_gap, const uint32_t* lp_row, const uint64_t* lp_dur,
                                const uint8_t* lp_level, const uint32_t* lp_stream, const uint64_t* lp_think,
                                const uint64_t* hp_arrival, const fikit_scenario_t* sc, uint32_t S,
                                fikit_fill_params_t params,
                                fikit_result_t* out, int32_t* fill_gap, uint64_t* lp_start,
                                const uint64_t* sched_off, void* ws, size_t ws_bytes, void* stream);

/* ---- multi-GPU merge ------------------------------------------
 * Each rank finalizes its local table, all-gathers the sorted keys
 * (P lists of n_list[r] keys, padded to stride Kmax), then:
 * fikit_dict_union builds the sorted union (identical on every rank) into
 * out_kid/out_task (capacity cap_out) and *out_n (device), and for list
 * `self_rank` the map local row -> union row into local_to_union;
 * fikit_table_remap scatters the local rows into the zero-initialised dense
 * table `dense` (kernel_id/task_id of every union row set); the caller then
 * all-reduces dense.sums (SUM u64), dense.hist (SUM u32), dense.ext (MAX u64)
 * and calls fikit_table_means.  E_CAPACITY if the union exceeds cap_out. */
int fikit_dict_union(const uint64_t* all_kid, const uint32_t* all_task, const uint32_t* n_list /* device [P] */,
                     uint32_t P, uint32_t Kmax, uint32_t self_rank, uint64_t* out_kid, uint32_t* out_task,
                     uint32_t cap_out, uint32_t* out_n, uint32_t* local_to_union, void* ws, size_t ws_bytes,
                     void* stream);
int fikit_table_remap(const fikit_table_t* local, const uint32_t* local_to_union, const uint64_t* union_kid,
                      const uint32_t* union_task, const uint32_t* union_n, const fikit_table_t* dense,
                      void* stream);

/* XOR 2^63 into every ext word of rows [0, capacity): maps the unsigned order of
 * the MAX block onto the signed order, so a signed 64-bit MAX all-reduce
 * (what NCCL / gloo offer through torch) reduces it correctly; an all-zero row
 * becomes INT64_MIN, the identity of signed MAX.  An involution: apply it
 * before and after the reduction. */
int fikit_table_bias(const fikit_table_t* tab, void* stream);

/* ---- status --------------------------------------------------------------- */
/* Synchronises `stream`, copies the workspace status to *out (host) and
 * derives out->code from the flags by precedence.  Returns out->code. */
int fikit_get_status(const void* ws, fikit_status_t* out, void* stream);
const char* fikit_strerror(int code);
/* Number of kernels the library launched since load (host counter; evidence for bench.py). */
uint64_t fikit_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FIKIT_H */
