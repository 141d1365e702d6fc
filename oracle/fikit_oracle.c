/*
 * FIKIT CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2311_10359_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path:
 * every layout below is re-declared here from DESIGN.md / PAPER.md.
 *
 * Plain, single-threaded, slow on purpose.  Each function cites the passage
 * it follows.  PAPER.md = P:<line>; readings of silent/garbled passages are
 * DESIGN.md "Readings" R1..R25 (= SURVEY.md §8c-4 C1..C25).
 *
 *   or_identify   kernel ID of every launch           P:188-201 (fig:kernelID), R1-R2
 *   or_measure    S_UID, SK, SG (+count/min/max/hist) P:233-257, R3-R11
 *   or_resolve    profile lookup per launch           P:278, P:330 (Alg.1 lines 3-5)
 *   or_best_prio_fit   Algorithm 2                    P:332-334, R14-R16
 *   or_fikit_fill      Algorithm 1 (one gap)          P:328-330, R13, R17-R19
 *   or_simulate        replay of one HP/LP scenario   P:286-313, R20-R24
 *   or_table_merge     union of per-shard tables      P:246-256, SURVEY §8e (all-core driver)
 *
 * Parity pins (tests/test_oracle_*.py) -- none of them re-types these
 * formulas: published FNV-1a / splitmix64 vectors, the paper's worked
 * examples, SPEC fixtures, closed
 * forms, a numpy group-by, brute-force optimal fills.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- byte layouts (re-declared independently) ---- */
typedef struct {
  uint64_t start_ns, end_ns;
  uint32_t name_id, sig_id;
  uint32_t grid_x;
  uint16_t grid_y, grid_z;
  uint16_t block_x, block_y, block_z, flags;
  uint32_t run_id, task_id;
} orec_t;
_Static_assert(sizeof(orec_t) == 48, "record is 48 bytes");

typedef struct {
  const uint8_t* bytes;
  const uint32_t* offsets; /* count+1 */
  uint32_t count;
} ostrtab_t;

enum {
  OR_OK = 0,
  OR_E_ARG = -1,
  OR_E_RECORD = -2,
  OR_E_CAPACITY = -3,
  OR_E_NAME = -5,
  OR_E_COLLISION = -99 /* two distinct identities hashed to one ID: a test failure (R2) */
};

typedef struct {
  int32_t code;
  uint32_t pad;
  uint64_t first_bad_index;
  uint64_t n_rows_needed;
  uint64_t n_overlap_gaps;
} ostatus_t;

/* Output statistic table, already in canonical (task_id, kernel_id) order. */
typedef struct {
  uint64_t* kernel_id;
  uint32_t* task_id;
  uint64_t *dur_cnt, *dur_sum, *dur_min, *dur_max;
  uint64_t *gap_cnt, *gap_sum, *gap_min, *gap_max;
  uint32_t *dur_hist, *gap_hist; /* [capacity][32] */
  uint64_t *dur_mean, *gap_mean;
  uint32_t capacity;
  uint32_t n_rows; /* out */
} otable_t;

typedef struct {
  uint64_t hp_jct, lp_jct, hp_delay, fill_work, digest;
  uint32_t n_fills, n_tail;
} oresult_t;
_Static_assert(sizeof(oresult_t) == 48, "result is 48 bytes");

#define NBINS 32

/* ------------------------------------------------------------------------- */
/* R2: the kernel ID is a 64-bit content hash of the paper's tuple            */
/* (name, block dims, grid dims) plus the argument-type signature    */
/* (north_star; R1).  FNV-1a-64 over bytes, splitmix64 finaliser to mix.      */
/* ------------------------------------------------------------------------- */
uint64_t or_fnv1a64(const uint8_t* b, uint64_t len) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < len; i++) {
    h ^= (uint64_t)b[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

uint64_t or_mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

uint64_t or_kernel_id(const uint8_t* name, uint64_t name_len, const uint8_t* sig, uint64_t sig_len,
                      uint32_t grid_x, uint32_t grid_y, uint32_t grid_z, uint32_t block_x, uint32_t block_y,
                      uint32_t block_z) {
  uint64_t w1 = (uint64_t)grid_x | ((uint64_t)grid_y << 32) | ((uint64_t)grid_z << 48);
  uint64_t w2 = (uint64_t)block_x | ((uint64_t)block_y << 16) | ((uint64_t)block_z << 32);
  uint64_t h = or_mix64(or_fnv1a64(name, name_len) ^ or_fnv1a64(sig, sig_len));
  h = or_mix64(h ^ w1);
  h = or_mix64(h ^ w2);
  return h == 0 ? 1 : h; /* ID 0 reserved (R2) */
}

static uint64_t rec_kid(const orec_t* r, const ostrtab_t* names, const ostrtab_t* sigs) {
  const uint8_t* nm = names->bytes + names->offsets[r->name_id];
  uint64_t nl = names->offsets[r->name_id + 1] - names->offsets[r->name_id];
  const uint8_t* sg = sigs->bytes + sigs->offsets[r->sig_id];
  uint64_t sl = sigs->offsets[r->sig_id + 1] - sigs->offsets[r->sig_id];
  return or_kernel_id(nm, nl, sg, sl, r->grid_x, r->grid_y, r->grid_z, r->block_x, r->block_y, r->block_z);
}

/* a1: a launch record is valid iff all dims >= 1,
 * name_id/sig_id index their tables, flags == 0 (reserved), and
 * (for a duration) end >= start (R4). */
static int rec_ok(const orec_t* r, uint32_t n_names, uint32_t n_sigs) {
  if (r->grid_x < 1 || r->grid_y < 1 || r->grid_z < 1) return 0;
  if (r->block_x < 1 || r->block_y < 1 || r->block_z < 1) return 0;
  if (r->name_id >= n_names || r->sig_id >= n_sigs) return 0;
  if (r->flags != 0) return 0;
  if (r->end_ns < r->start_ns) return 0;
  return 1;
}

static int strtabs_check(const ostrtab_t* names, const ostrtab_t* sigs) {
  for (uint32_t j = 0; j < names->count; j++) {
    if (names->offsets[j + 1] < names->offsets[j]) return OR_E_ARG;
    if (names->offsets[j + 1] == names->offsets[j]) return OR_E_NAME; /* empty name */
  }
  for (uint32_t j = 0; j < sigs->count; j++)
    if (sigs->offsets[j + 1] < sigs->offsets[j]) return OR_E_ARG;
  return OR_OK;
}

static void status_init(ostatus_t* st) {
  memset(st, 0, sizeof(*st));
  st->first_bad_index = UINT64_MAX;
}

/* first invalid record (E_RECORD) -- error precedence: NAME > RECORD > CAPACITY */
static int validate_all(const orec_t* rec, uint64_t n, const ostrtab_t* names, const ostrtab_t* sigs,
                        ostatus_t* st) {
  int c = strtabs_check(names, sigs);
  if (c != OR_OK) {
    st->code = c;
    return c;
  }
  for (uint64_t i = 0; i < n; i++)
    if (!rec_ok(&rec[i], names->count, sigs->count)) {
      st->code = OR_E_RECORD;
      st->first_bad_index = i;
      return OR_E_RECORD;
    }
  return OR_OK;
}

/* ---- identify: one ID per launch, independent of position ---- */
int or_identify(const orec_t* rec, uint64_t n, ostrtab_t names, ostrtab_t sigs, uint64_t* out_kid, ostatus_t* st) {
  status_init(st);
  if (validate_all(rec, n, &names, &sigs, st) != OR_OK) return st->code;
  for (uint64_t i = 0; i < n; i++) out_kid[i] = rec_kid(&rec[i], &names, &sigs);
  return OR_OK;
}

/* ---- measure ------------------------------------------------- */
static int bin_of(uint64_t v) { /* R9: bin(v) = min(31, bit_length(v)) */
  int b = 0;
  while (v) {
    b++;
    v >>= 1;
  }
  return b < 31 ? b : 31;
}

/* R8: integer mean, round half up; cnt = 0 -> 0 */
static uint64_t mean_of(uint64_t sum, uint64_t cnt) {
  if (cnt == 0) return 0;
  uint64_t q = sum / cnt, r = sum % cnt;
  return q + (2 * r >= cnt ? 1 : 0);
}

typedef struct {
  uint32_t task;
  uint64_t kid;
  uint64_t idx;
} okey_t;

static int cmp_key(const void* a, const void* b) {
  const okey_t* x = (const okey_t*)a;
  const okey_t* y = (const okey_t*)b;
  if (x->task != y->task) return x->task < y->task ? -1 : 1;
  if (x->kid != y->kid) return x->kid < y->kid ? -1 : 1;
  if (x->idx != y->idx) return x->idx < y->idx ? -1 : 1;
  return 0;
}

static int same_identity(const orec_t* a, const orec_t* b, const ostrtab_t* names, const ostrtab_t* sigs) {
  uint32_t la = names->offsets[a->name_id + 1] - names->offsets[a->name_id];
  uint32_t lb = names->offsets[b->name_id + 1] - names->offsets[b->name_id];
  if (la != lb || memcmp(names->bytes + names->offsets[a->name_id], names->bytes + names->offsets[b->name_id], la))
    return 0;
  la = sigs->offsets[a->sig_id + 1] - sigs->offsets[a->sig_id];
  lb = sigs->offsets[b->sig_id + 1] - sigs->offsets[b->sig_id];
  if (la != lb || memcmp(sigs->bytes + sigs->offsets[a->sig_id], sigs->bytes + sigs->offsets[b->sig_id], la))
    return 0;
  return a->grid_x == b->grid_x && a->grid_y == b->grid_y && a->grid_z == b->grid_z && a->block_x == b->block_x &&
         a->block_y == b->block_y && a->block_z == b->block_z;
}

/* The following gap of launch i ("from each kernel ends to the next
 * kernel starts", N_t - 1 gaps per run).  R5: a gap exists iff the next
 * launch (record i+1, or the halo record after the last one) has the same
 * (task_id, run_id); a negative gap (overlap) is clamped to 0 and counted. */
static int gap_of(const orec_t* rec, uint64_t n, const orec_t* halo, uint64_t i, uint64_t* g, int* clamped) {
  const orec_t* nx = (i + 1 < n) ? &rec[i + 1] : halo;
  *clamped = 0;
  if (!nx || nx->task_id != rec[i].task_id || nx->run_id != rec[i].run_id) return 0;
  if (nx->start_ns >= rec[i].end_ns)
    *g = nx->start_ns - rec[i].end_ns;
  else {
    *g = 0;
    *clamped = 1;
  }
  return 1;
}

int or_measure(const orec_t* rec, uint64_t n, const orec_t* halo, ostrtab_t names, ostrtab_t sigs, otable_t* tab,
               uint32_t* out_row /* nullable */, ostatus_t* st) {
  status_init(st);
  tab->n_rows = 0;
  if (validate_all(rec, n, &names, &sigs, st) != OR_OK) return st->code;

  /* ID_{t,i} for every launch, hashed from the strings each time */
  okey_t* keys = (okey_t*)malloc((n ? n : 1) * sizeof(okey_t));
  for (uint64_t i = 0; i < n; i++) {
    keys[i].task = rec[i].task_id;
    keys[i].kid = rec_kid(&rec[i], &names, &sigs);
    keys[i].idx = i;
  }
  /* S_UID: the distinct IDs, here per Task Key (R3), canonical order (R11) */
  qsort(keys, n, sizeof(okey_t), cmp_key);

  /* collision check (R2): equal kernel_id must mean an identical tuple */
  {
    okey_t* byk = (okey_t*)malloc((n ? n : 1) * sizeof(okey_t));
    for (uint64_t i = 0; i < n; i++) {
      byk[i] = keys[i];
      byk[i].task = 0;
    }
    qsort(byk, n, sizeof(okey_t), cmp_key);
    for (uint64_t i = 1; i < n; i++)
      if (byk[i].kid == byk[i - 1].kid && !same_identity(&rec[byk[i].idx], &rec[byk[i - 1].idx], &names, &sigs)) {
        st->code = OR_E_COLLISION;
        st->first_bad_index = byk[i].idx;
        free(byk);
        free(keys);
        return OR_E_COLLISION;
      }
    free(byk);
  }

  uint64_t distinct = 0;
  for (uint64_t i = 0; i < n; i++)
    if (i == 0 || keys[i].task != keys[i - 1].task || keys[i].kid != keys[i - 1].kid) distinct++;
  if (distinct > tab->capacity) {
    free(keys);
    st->code = OR_E_CAPACITY;
    st->n_rows_needed = distinct;
    return OR_E_CAPACITY;
  }

  /* SK_j and SG_j as exact (count, sum), plus min/max/hist (R9):
   * walk each group of launches with the same ID j -- the Kronecker delta. */
  uint32_t row = 0;
  for (uint64_t a = 0; a < n;) {
    uint64_t b = a;
    while (b < n && keys[b].task == keys[a].task && keys[b].kid == keys[a].kid) b++;
    uint64_t dc = 0, ds = 0, dmin = UINT64_MAX, dmax = 0, gc = 0, gs = 0, gmin = UINT64_MAX, gmax = 0;
    uint32_t* dh = tab->dur_hist + (uint64_t)row * NBINS;
    uint32_t* gh = tab->gap_hist + (uint64_t)row * NBINS;
    memset(dh, 0, NBINS * sizeof(uint32_t));
    memset(gh, 0, NBINS * sizeof(uint32_t));
    for (uint64_t j = a; j < b; j++) {
      uint64_t i = keys[j].idx;
      uint64_t d = rec[i].end_ns - rec[i].start_ns; /* K_{ID_{t,i}} = end - start */
      dc += 1;
      ds += d;
      if (d < dmin) dmin = d;
      if (d > dmax) dmax = d;
      dh[bin_of(d)]++;
      uint64_t g;
      int cl;
      if (gap_of(rec, n, halo, i, &g, &cl)) { /* G_{ID_{t,i}}, i <= N_t - 1 */
        gc += 1;
        gs += g;
        if (g < gmin) gmin = g;
        if (g > gmax) gmax = g;
        gh[bin_of(g)]++;
        st->n_overlap_gaps += (uint64_t)cl;
      }
      if (out_row) out_row[i] = row;
    }
    tab->kernel_id[row] = keys[a].kid;
    tab->task_id[row] = keys[a].task;
    tab->dur_cnt[row] = dc;
    tab->dur_sum[row] = ds;
    tab->dur_min[row] = dmin;
    tab->dur_max[row] = dmax;
    tab->gap_cnt[row] = gc;
    tab->gap_sum[row] = gs;
    tab->gap_min[row] = gmin;
    tab->gap_max[row] = gmax;
    tab->dur_mean[row] = mean_of(ds, dc); /* SK_j */
    tab->gap_mean[row] = mean_of(gs, gc); /* SG_j; no samples -> 0 -> no fill (R12) */
    row++;
    a = b;
  }
  tab->n_rows = row;
  free(keys);
  return OR_OK;
}

/* ---- profile lookup ("filter out the profiling data matching the
 * Task Key"; Alg.1 lines 3-5) + per-launch duration and following
 * gap.  Absent IDs get row 0xFFFFFFFF. ----------------------------------- */
int or_resolve(const orec_t* rec, uint64_t n, const orec_t* halo, ostrtab_t names, ostrtab_t sigs,
               const uint64_t* tab_kid, const uint32_t* tab_task, uint32_t n_rows, uint32_t* out_row,
               uint64_t* out_dur, uint64_t* out_gap, ostatus_t* st) {
  status_init(st);
  if (validate_all(rec, n, &names, &sigs, st) != OR_OK) return st->code;
  for (uint64_t i = 0; i < n; i++) {
    uint64_t kid = rec_kid(&rec[i], &names, &sigs);
    uint32_t row = 0xFFFFFFFFu;
    for (uint32_t r = 0; r < n_rows; r++) /* linear search: slow and obvious */
      if (tab_task[r] == rec[i].task_id && tab_kid[r] == kid) {
        row = r;
        break;
      }
    out_row[i] = row;
    out_dur[i] = rec[i].end_ns - rec[i].start_ns;
    uint64_t g = 0;
    int cl;
    if (!gap_of(rec, n, halo, i, &g, &cl)) g = 0;
    st->n_overlap_gaps += (uint64_t)cl;
    out_gap[i] = g;
  }
  return OR_OK;
}

/* ---- Algorithm 2, BestPrioFit ---------------------------------
 * Iterate the priority levels from highest (1; level 0 is the gap holder,
 * R16) to lowest (9) (line 5); at each level examine every waiting request
 * (line 7), keeping the one whose duration is the longest so far and fits
 * the remaining idle gap (lines 13-18; fit is q <= R, R14; ties keep the
 * earliest request, R15).  The first level with a fit wins; the request is
 * dequeued and returned with its duration (lines 25-29).  Requests without
 * an SK profile are never fills (R16).  Returns -1 if nothing fits. */
int64_t or_best_prio_fit(uint32_t m, const uint64_t* q, const uint8_t* elig, const uint8_t* level, uint8_t* alive,
                         uint64_t R) {
  for (uint32_t L = 1; L <= 9; L++) {
    int64_t best = -1;
    for (uint32_t k = 0; k < m; k++) {
      if (!alive[k] || !elig[k] || level[k] != L) continue;
      if (q[k] > R) continue;
      if (best < 0 || q[k] > q[best]) best = (int64_t)k;
    }
    if (best >= 0) {
      alive[best] = 0; /* dequeue */
      return best;
    }
  }
  return -1;
}

/* ---- Algorithm 1, the FIKIT procedure for one gap ------------
 * R0: predicted idle time of the running HP kernel (lines 3-5, looked up by
 * the caller).  Gaps below the threshold are skipped (lines 6-8, R13).
 * Otherwise BestPrioFit is called repeatedly (lines 9-16); each fill is
 * launched (line 14) and the idle duration is revised by the returned
 * duration (line 15, R17: the predicted q).  Runtime feedback (P:354-362,
 * R19): fills are dispatched one at a time at device time t; with feedback
 * on, dispatch stops as soon as the HP client's next launch has arrived
 * (t >= deadline; tie -> HP).  Times are absolute; t starts at t0.
 * picks[] receives the pool indices in dispatch order, start[] their start. */
uint32_t or_fikit_fill(uint64_t R0, uint64_t t0, uint64_t deadline, uint64_t threshold, uint32_t feedback,
                       uint32_t m, const uint64_t* q, const uint64_t* e, const uint8_t* elig, const uint8_t* level,
                       uint8_t* alive, uint32_t* picks, uint64_t* start, uint64_t* R_left, uint64_t* t_end) {
  uint32_t np = 0;
  uint64_t R = R0, t = t0;
  if (R0 >= threshold) {
    for (;;) {
      if (feedback && t >= deadline) break; /* early stop */
      int64_t k = or_best_prio_fit(m, q, elig, level, alive, R);
      if (k < 0) break; /* no more suitable requests */
      picks[np] = (uint32_t)k;
      start[np] = t;
      np++;
      t += e[k];
      R -= q[k];
    }
  }
  *R_left = R;
  *t_end = t;
  return np;
}

/* Batch form of Alg. 1 over G independent gaps (building block of the
 * replay); times relative to the gap start (t0 = 0). */
int or_fill_batch(const uint64_t* R0, const uint64_t* deadline, const uint32_t* pool_row, const uint64_t* pool_dur,
                  const uint8_t* pool_level, const uint32_t* pool_off, const uint32_t* pool_len, uint32_t G,
                  const uint64_t* dur_mean, const uint64_t* dur_cnt, uint32_t n_rows, uint64_t threshold,
                  uint32_t feedback, uint32_t* picks, const uint32_t* picks_off, uint32_t* n_picks, uint64_t* R_left,
                  uint64_t* t_used, ostatus_t* st) {
  status_init(st);
  for (uint32_t g = 0; g < G; g++) {
    uint32_t m = pool_len[g], off = pool_off[g];
    for (uint32_t k = 0; k < m; k++)
      if (pool_level[off + k] < 1 || pool_level[off + k] > 9) {
        st->code = OR_E_RECORD;
        st->first_bad_index = (uint64_t)off + k;
        return OR_E_RECORD;
      }
  }
  for (uint32_t g = 0; g < G; g++) {
    uint32_t m = pool_len[g], off = pool_off[g];
    uint64_t* q = (uint64_t*)malloc((m ? m : 1) * 8);
    uint8_t* el = (uint8_t*)malloc(m ? m : 1);
    uint8_t* al = (uint8_t*)malloc(m ? m : 1);
    uint64_t* stt = (uint64_t*)malloc((m ? m : 1) * 8);
    for (uint32_t k = 0; k < m; k++) {
      uint32_t r = pool_row[off + k];
      el[k] = (r < n_rows && dur_cnt[r] > 0);
      q[k] = el[k] ? dur_mean[r] : 0;
      al[k] = 1;
    }
    uint64_t te;
    n_picks[g] = or_fikit_fill(R0[g], 0, deadline[g], threshold, feedback, m, q, pool_dur + off, el,
                               pool_level + off, al, picks + picks_off[g], stt, &R_left[g], &te);
    t_used[g] = te;
    free(q);
    free(el);
    free(al);
    free(stt);
  }
  return OR_OK;
}

/* ---- replay of one scenario (Case B) ----------------
 * HP task (level 0) holds the GPU and launches its kernels in order; kernel
 * i runs d_i; its client launches kernel i+1 a'_i after observing kernel i's
 * end (R20).  After HP kernel i the FIKIT procedure fills the predicted gap
 * p_i = SG of its ID (Alg.1 lines 3-5, R12), scaled by s (R24).  The next HP
 * kernel starts at max(t, r_{i+1}): fills already queued cannot be revoked
 * ("overhead 2").  After the HP job, the remaining LP requests run
 * back to back in Q1..Q9 order, FIFO within a queue (R22). */
static uint64_t digest_term(uint32_t k, int32_t fill_gap, uint64_t lp_start) {
  return or_mix64((uint64_t)k ^ ((uint64_t)(uint32_t)(fill_gap + 1) << 32) ^ or_mix64(lp_start));
}

int or_simulate(const uint32_t* hp_row, const uint64_t* hp_dur, const uint64_t* hp_gap, uint32_t n_h,
                const uint32_t* lp_row, const uint64_t* lp_dur, const uint8_t* lp_level, uint32_t m,
                uint32_t gap_scale_q16, const uint64_t* dur_mean, const uint64_t* dur_cnt, const uint64_t* gap_mean,
                uint32_t n_rows, uint64_t threshold, uint32_t feedback, oresult_t* out, int32_t* fill_gap,
                uint64_t* lp_start) {
  uint64_t* q = (uint64_t*)malloc((m ? m : 1) * 8);
  uint8_t* el = (uint8_t*)malloc(m ? m : 1);
  uint8_t* al = (uint8_t*)malloc(m ? m : 1);
  uint32_t* picks = (uint32_t*)malloc((m ? m : 1) * 4);
  uint64_t* pst = (uint64_t*)malloc((m ? m : 1) * 8);
  for (uint32_t k = 0; k < m; k++) {
    uint32_t r = lp_row[k];
    el[k] = (r < n_rows && dur_cnt[r] > 0); /* R16 */
    q[k] = el[k] ? dur_mean[r] : 0;         /* SK of the request's ID */
    al[k] = 1;
    fill_gap[k] = -1;
    lp_start[k] = 0;
  }
  uint64_t s = gap_scale_q16;
  uint64_t t = 0, hp_delay = 0, fill_work = 0;
  uint32_t n_fills = 0;
  for (uint32_t i = 0; i < n_h; i++) {
    uint64_t start = t; /* next HP kernel: t >= r_{i} already folded in below */
    uint64_t end = start + hp_dur[i];
    t = end;
    if (i == n_h - 1) break;
    uint64_t r = end + ((hp_gap[i] * s) >> 16); /* HP client's next launch arrives (R20, R24) */
    uint32_t hr = hp_row[i];
    uint64_t p = (hr < n_rows) ? ((gap_mean[hr] * s) >> 16) : 0; /* predicted gap (R12, R24) */
    uint64_t Rl;
    uint32_t np = or_fikit_fill(p, t, r, threshold, feedback, m, q, lp_dur, el, lp_level, al, picks, pst, &Rl, &t);
    for (uint32_t j = 0; j < np; j++) {
      fill_gap[picks[j]] = (int32_t)i;
      lp_start[picks[j]] = pst[j];
      fill_work += lp_dur[picks[j]];
    }
    n_fills += np;
    if (t > r) hp_delay += t - r; /* overhead the fills imposed on HP kernel i+1 */
    t = (t > r) ? t : r;          /* kernel i+1 starts at max(t, r_{i+1}) */
  }
  uint64_t hp_jct = t; /* end of the last HP kernel (R23) */
  uint32_t n_tail = 0;
  for (uint32_t L = 1; L <= 9; L++) /* tail: Q1..Q9, FIFO within a queue */
    for (uint32_t k = 0; k < m; k++)
      if (al[k] && lp_level[k] == L) {
        al[k] = 0;
        fill_gap[k] = -1;
        lp_start[k] = t;
        t += lp_dur[k];
        n_tail++;
      }
  uint64_t lp_jct = 0, digest = 0;
  for (uint32_t k = 0; k < m; k++) {
    uint64_t e = lp_start[k] + lp_dur[k];
    if (e > lp_jct) lp_jct = e;
    digest += digest_term(k, fill_gap[k], lp_start[k]);
  }
  out->hp_jct = hp_jct;
  out->lp_jct = lp_jct;
  out->hp_delay = hp_delay;
  out->fill_work = fill_work;
  out->digest = digest;
  out->n_fills = n_fills;
  out->n_tail = n_tail;
  free(q);
  free(el);
  free(al);
  free(picks);
  free(pst);
  return OR_OK;
}

typedef struct {
  uint32_t hp_off, hp_len, lp_off, lp_len, gap_scale_q16, pad;
} oscen_t;

int or_simulate_batch(const uint32_t* hp_row, const uint64_t* hp_dur, const uint64_t* hp_gap, const uint32_t* lp_row,
                      const uint64_t* lp_dur, const uint8_t* lp_level, const oscen_t* sc, uint32_t S,
                      const uint64_t* dur_mean, const uint64_t* dur_cnt, const uint64_t* gap_mean, uint32_t n_rows,
                      uint64_t threshold, uint32_t feedback, oresult_t* out, int32_t* fill_gap /* nullable */,
                      uint64_t* lp_start /* nullable */, const uint64_t* sched_off /* nullable */, ostatus_t* st) {
  status_init(st);
  for (uint32_t s = 0; s < S; s++)
    for (uint32_t k = 0; k < sc[s].lp_len; k++) {
      uint8_t L = lp_level[(uint64_t)sc[s].lp_off + k];
      if (L < 1 || L > 9) {
        st->code = OR_E_RECORD;
        st->first_bad_index = (uint64_t)sc[s].lp_off + k;
        return OR_E_RECORD;
      }
    }
  uint32_t mmax = 1;
  for (uint32_t s = 0; s < S; s++)
    if (sc[s].lp_len > mmax) mmax = sc[s].lp_len;
  int32_t* fg = (int32_t*)malloc(mmax * 4);
  uint64_t* ls = (uint64_t*)malloc(mmax * 8);
  for (uint32_t s = 0; s < S; s++) {
    const oscen_t* c = &sc[s];
    or_simulate(hp_row + c->hp_off, hp_dur + c->hp_off, hp_gap + c->hp_off, c->hp_len, lp_row + c->lp_off,
                lp_dur + c->lp_off, lp_level + c->lp_off, c->lp_len, c->gap_scale_q16, dur_mean, dur_cnt, gap_mean,
                n_rows, threshold, feedback, &out[s], fg, ls);
    if (fill_gap && sched_off)
      for (uint32_t k = 0; k < c->lp_len; k++) {
        fill_gap[sched_off[s] + k] = fg[k];
        lp_start[sched_off[s] + k] = ls[k];
      }
  }
  free(fg);
  free(ls);
  return OR_OK;
}

/* ---- predictor variants ("dynamic duration and idling
 * prediction", the "same ID, different duration" weakness).  The replay reads a
 * row's predicted duration q (Alg.1 line 4) from dur_mean and its predicted gap p
 * (line 3) from gap_mean; this rewrites those two columns (readings R26-R28):
 *   mode 0 (the paper): the integer means SK, SG (R8).
 *   mode 1 (histogram percentile, conservative): with cum(b) the count of bins
 *     0..b and c the row's count, b_P = the smallest b with 100*cum(b) >= P*c (and
 *     cum(b) >= 1).  Duration: the upper edge of bin b_P (2^b - 1; bin 31 is
 *     unbounded: the row's max), capped at the row's max.  Gap: the lower edge of
 *     bin b_(100-P) (2^(b-1); bin 0: 0), raised to the row's min.  1 <= P <= 99.
 *   mode 2 (extremes): duration = max, gap = min.
 * A row without samples predicts 0 in every mode. */
static uint32_t pct_bin(const uint32_t* h, uint64_t c, uint32_t P) {
  uint64_t cum = 0;
  for (uint32_t b = 0; b < 32; b++) {
    cum += h[b];
    if (cum >= 1 && 100 * cum >= (uint64_t)P * c) return b;
  }
  return 31;
}

int or_predict(otable_t* tab, uint32_t mode, uint32_t pct) {
  if (mode > 2 || (mode == 1 && (pct < 1 || pct > 99))) return OR_E_ARG;
  for (uint32_t r = 0; r < tab->n_rows; r++) {
    const uint64_t dc = tab->dur_cnt[r], gc = tab->gap_cnt[r];
    uint64_t d = 0, g = 0;
    if (mode == 0) {
      d = mean_of(tab->dur_sum[r], dc);
      g = mean_of(tab->gap_sum[r], gc);
    } else if (mode == 1) {
      if (dc) {
        const uint32_t b = pct_bin(tab->dur_hist + (size_t)r * 32, dc, pct);
        const uint64_t up = b == 0 ? 0 : (b < 31 ? (1ull << b) - 1 : tab->dur_max[r]);
        d = up < tab->dur_max[r] ? up : tab->dur_max[r];
      }
      if (gc) {
        const uint32_t b = pct_bin(tab->gap_hist + (size_t)r * 32, gc, 100 - pct);
        const uint64_t lo = b == 0 ? 0 : (1ull << (b - 1));
        g = lo > tab->gap_min[r] ? lo : tab->gap_min[r];
      }
    } else {
      d = dc ? tab->dur_max[r] : 0;
      g = gc ? tab->gap_min[r] : 0;
    }
    tab->dur_mean[r] = d;
    tab->gap_mean[r] = g;
  }
  return OR_OK;
}

/* ---- STREAM-model replay (readings R29-R32) ----------------
 * The LP requests of a scenario are kernel streams (LP tasks whose hook client
 * blocks each launch): a stream is a maximal run of equal consecutive
 * lp_stream values; only its first undispatched request (the head) is queued
 * (P:297-299).  Heads arrive at time 0; request k+1 of a stream arrives
 * lp_think[k] after request k ends (the LP trace's own gap, R5) (R29).  In gap i
 * BestPrioFit (Alg. 2) runs over the arrived heads; when none fits, the
 * scheduler waits for the next head arrival A -- an arrival triggers a scan
 * -- if A - t <= R and, with feedback, A < r_{i+1}; waiting consumes
 * predicted idle (R -= A - t) (R30).  After the HP job the remaining requests run
 * in (level, index) order among the arrived heads, time jumping to the earliest
 * arrival when none has arrived (R31).  HP side, gate, R and feedback as
 * or_simulate (R13, R17-R20, R24).  Singleton streams are the POOL model. */
/* Case A (§8f row 2; "the scheduler withholds the next launching kernel of A to let the
 * later arriving high-priority B's kernel run"): with t_arrive > 0 the LP streams hold
 * the GPU from t = 0 -- heads in (level, index) order among the arrived ones, time jumping to
 * the next arrival -- and an LP kernel may start only before the HP job arrives at t_arrive;
 * the one running then is not preempted, so the HP's first kernel starts at
 * max(t_arrive, its end) (R33).  hp_jct stays absolute: the HP response time is
 * hp_jct - t_arrive (R34).  LP kernels run before the HP job count in neither n_fills nor
 * n_tail (fill_gap -1, R31's tail counter excludes them). */
int or_simulate_stream(const uint32_t* hp_row, const uint64_t* hp_dur, const uint64_t* hp_gap, uint32_t n_h,
                       const uint32_t* lp_row, const uint64_t* lp_dur, const uint8_t* lp_level,
                       const uint32_t* lp_stream, const uint64_t* lp_think, uint32_t m, uint32_t gap_scale_q16,
                       const uint64_t* dur_mean, const uint64_t* dur_cnt, const uint64_t* gap_mean, uint32_t n_rows,
                       uint64_t threshold, uint32_t feedback, uint64_t t_arrive, oresult_t* out, int32_t* fill_gap,
                       uint64_t* lp_start) {
  uint32_t M = m ? m : 1;
  uint64_t* q = (uint64_t*)malloc(M * 8);
  uint8_t* el = (uint8_t*)malloc(M);
  uint32_t* head = (uint32_t*)malloc(M * 4); /* per stream: next request, one past its last */
  uint32_t* send = (uint32_t*)malloc(M * 4);
  uint64_t* arr = (uint64_t*)malloc(M * 8);
  uint32_t ns = 0;
  for (uint32_t k = 0; k < m; k++) {
    uint32_t r = lp_row[k];
    el[k] = (r < n_rows && dur_cnt[r] > 0); /* R16 */
    q[k] = el[k] ? dur_mean[r] : 0;
    fill_gap[k] = -1;
    lp_start[k] = 0;
    if (k == 0 || lp_stream[k] != lp_stream[k - 1]) {
      head[ns] = k;
      arr[ns] = 0;
      ns++;
    }
    send[ns - 1] = k + 1;
  }
  uint64_t s = gap_scale_q16;
  uint64_t t = 0, hp_delay = 0, fill_work = 0;
  uint32_t n_fills = 0;
  for (;;) { /* before the HP job arrives (R33) */
    if (t >= t_arrive) break;
    int64_t bs = -1;
    uint64_t A = UINT64_MAX;
    for (uint32_t j = 0; j < ns; j++) {
      if (head[j] >= send[j]) continue;
      if (arr[j] > t) {
        if (arr[j] < A) A = arr[j];
        continue;
      }
      uint32_t k = head[j];
      if (bs < 0 || lp_level[k] < lp_level[head[bs]] || (lp_level[k] == lp_level[head[bs]] && k < head[bs]))
        bs = j;
    }
    if (bs < 0) {
      if (A >= t_arrive) break;
      t = A;
      continue;
    }
    uint32_t k = head[bs];
    lp_start[k] = t;
    t += lp_dur[k];
    head[bs]++;
    arr[bs] = t + lp_think[k];
  }
  if (t < t_arrive) t = t_arrive; /* HP kernel 0 starts at max(t_arrive, the running LP kernel's end) */
  for (uint32_t i = 0; i < n_h; i++) {
    uint64_t end = t + hp_dur[i];
    t = end;
    if (i == n_h - 1) break;
    uint64_t r = end + ((hp_gap[i] * s) >> 16); /* R20, R24 */
    uint32_t hr = hp_row[i];
    uint64_t p = (hr < n_rows) ? ((gap_mean[hr] * s) >> 16) : 0;
    uint64_t R = p;
    if (p >= threshold) { /* R13 */
      for (;;) {
        if (feedback && t >= r) break; /* R19 */
        /* BestPrioFit (Alg. 2) over the arrived heads: the first level with a fit, the longest
           q there, ties to the earliest request (R14-R16) */
        int64_t bs = -1;
        for (uint32_t L = 1; L <= 9 && bs < 0; L++)
          for (uint32_t j = 0; j < ns; j++) {
            if (head[j] >= send[j] || arr[j] > t) continue;
            uint32_t k = head[j];
            if (!el[k] || lp_level[k] != L || q[k] > R) continue;
            if (bs < 0 || q[k] > q[head[bs]] || (q[k] == q[head[bs]] && k < head[bs])) bs = j;
          }
        if (bs >= 0) {
          uint32_t k = head[bs];
          fill_gap[k] = (int32_t)i;
          lp_start[k] = t;
          t += lp_dur[k];
          R -= q[k];
          fill_work += lp_dur[k];
          n_fills++;
          head[bs]++;
          arr[bs] = t + lp_think[k];
          continue;
        }
        /* no arrived head fits: wait for the next arrival within the predicted idle (R30) */
        uint64_t A = UINT64_MAX;
        for (uint32_t j = 0; j < ns; j++)
          if (head[j] < send[j] && arr[j] > t && arr[j] < A) A = arr[j];
        if (A == UINT64_MAX || A - t > R || (feedback && A >= r)) break;
        R -= A - t;
        t = A;
      }
    }
    if (t > r) hp_delay += t - r;
    t = (t > r) ? t : r;
  }
  uint64_t hp_jct = t; /* R23 */
  uint32_t n_tail = 0;
  for (;;) { /* tail (R31) */
    int64_t bs = -1;
    uint64_t A = UINT64_MAX;
    for (uint32_t j = 0; j < ns; j++) {
      if (head[j] >= send[j]) continue;
      if (arr[j] > t) {
        if (arr[j] < A) A = arr[j];
        continue;
      }
      uint32_t k = head[j];
      if (bs < 0 || lp_level[k] < lp_level[head[bs]] || (lp_level[k] == lp_level[head[bs]] && k < head[bs]))
        bs = j;
    }
    if (bs < 0) {
      if (A == UINT64_MAX) break;
      t = A;
      continue;
    }
    uint32_t k = head[bs];
    lp_start[k] = t;
    t += lp_dur[k];
    head[bs]++;
    arr[bs] = t + lp_think[k];
    n_tail++;
  }
  uint64_t lp_jct = 0, digest = 0;
  for (uint32_t k = 0; k < m; k++) {
    uint64_t e = lp_start[k] + lp_dur[k];
    if (e > lp_jct) lp_jct = e;
    digest += digest_term(k, fill_gap[k], lp_start[k]);
  }
  out->hp_jct = hp_jct;
  out->lp_jct = m ? lp_jct : 0;
  out->hp_delay = hp_delay;
  out->fill_work = fill_work;
  out->digest = digest;
  out->n_fills = n_fills;
  out->n_tail = n_tail;
  free(q);
  free(el);
  free(head);
  free(send);
  free(arr);
  return OR_OK;
}

int or_simulate_stream_batch(const uint32_t* hp_row, const uint64_t* hp_dur, const uint64_t* hp_gap,
                             const uint32_t* lp_row, const uint64_t* lp_dur, const uint8_t* lp_level,
                             const uint32_t* lp_stream, const uint64_t* lp_think, const oscen_t* sc, uint32_t S,
                             const uint64_t* dur_mean, const uint64_t* dur_cnt, const uint64_t* gap_mean,
                             uint32_t n_rows, uint64_t threshold, uint32_t feedback,
                             const uint64_t* hp_arrival /* nullable: 0 */, oresult_t* out, int32_t* fill_gap,
                             uint64_t* lp_start, const uint64_t* sched_off) {
  for (uint32_t i = 0; i < S; i++) {
    const oscen_t* c = sc + i;
    for (uint32_t k = 0; k < c->lp_len; k++) {
      uint8_t L = lp_level[c->lp_off + k];
      if (L < 1 || L > 9) return OR_E_RECORD;
    }
    int rc = or_simulate_stream(hp_row + c->hp_off, hp_dur + c->hp_off, hp_gap + c->hp_off, c->hp_len,
                                lp_row + c->lp_off, lp_dur + c->lp_off, lp_level + c->lp_off, lp_stream + c->lp_off,
                                lp_think + c->lp_off, c->lp_len, c->gap_scale_q16, dur_mean, dur_cnt, gap_mean,
                                n_rows, threshold, feedback, hp_arrival ? hp_arrival[i] : 0, out + i,
                                fill_gap + sched_off[i], lp_start + sched_off[i]);
    if (rc) return rc;
  }
  return OR_OK;
}

/* ---- merge of per-shard tables (the all-core CPU baseline's
 * sharded driver, oracle/sharded.py).  Each part is the or_measure table of
 * one contiguous record shard whose last gap used the next shard's first
 * record as its halo (R5), so every launch and every gap was counted by
 * exactly one part.  S_UID of the whole trace is the union of the
 * parts' rows, and the statistics of a row j are sums / minima / maxima over
 * the parts that saw j: SK_j = (sum of K over all occurrences) / (count of all
 * occurrences), likewise SG_j; the integer mean is R8.
 * Plain form: collect every (task, kernel_id, part, row) key, sort it in the
 * canonical order (R11), walk runs of equal (task, kernel_id). ------------ */
typedef struct {
  uint32_t task;
  uint64_t kid;
  uint32_t part, row;
} opkey_t;

static int cmp_pkey(const void* a, const void* b) {
  const opkey_t* x = (const opkey_t*)a;
  const opkey_t* y = (const opkey_t*)b;
  if (x->task != y->task) return x->task < y->task ? -1 : 1;
  if (x->kid != y->kid) return x->kid < y->kid ? -1 : 1;
  if (x->part != y->part) return x->part < y->part ? -1 : 1;
  return 0;
}

int or_table_merge(const otable_t* parts, uint32_t P, otable_t* out, ostatus_t* st) {
  status_init(st);
  out->n_rows = 0;
  uint64_t total = 0;
  for (uint32_t p = 0; p < P; p++) total += parts[p].n_rows;
  opkey_t* keys = (opkey_t*)malloc((total ? total : 1) * sizeof(opkey_t));
  uint64_t k = 0;
  for (uint32_t p = 0; p < P; p++)
    for (uint32_t r = 0; r < parts[p].n_rows; r++) {
      keys[k].task = parts[p].task_id[r];
      keys[k].kid = parts[p].kernel_id[r];
      keys[k].part = p;
      keys[k].row = r;
      k++;
    }
  qsort(keys, total, sizeof(opkey_t), cmp_pkey);
  uint64_t distinct = 0;
  for (uint64_t i = 0; i < total; i++)
    if (i == 0 || keys[i].task != keys[i - 1].task || keys[i].kid != keys[i - 1].kid) distinct++;
  if (distinct > out->capacity) {
    free(keys);
    st->code = OR_E_CAPACITY;
    st->n_rows_needed = distinct;
    return OR_E_CAPACITY;
  }
  uint32_t row = 0;
  for (uint64_t a = 0; a < total;) {
    uint64_t b = a;
    while (b < total && keys[b].task == keys[a].task && keys[b].kid == keys[a].kid) b++;
    uint64_t dc = 0, ds = 0, dmin = UINT64_MAX, dmax = 0, gc = 0, gs = 0, gmin = UINT64_MAX, gmax = 0;
    uint32_t* dh = out->dur_hist + (uint64_t)row * NBINS;
    uint32_t* gh = out->gap_hist + (uint64_t)row * NBINS;
    memset(dh, 0, NBINS * sizeof(uint32_t));
    memset(gh, 0, NBINS * sizeof(uint32_t));
    for (uint64_t j = a; j < b; j++) {
      const otable_t* t = &parts[keys[j].part];
      uint32_t r = keys[j].row;
      dc += t->dur_cnt[r];
      ds += t->dur_sum[r];
      if (t->dur_min[r] < dmin) dmin = t->dur_min[r];
      if (t->dur_max[r] > dmax) dmax = t->dur_max[r];
      gc += t->gap_cnt[r];
      gs += t->gap_sum[r];
      if (t->gap_min[r] < gmin) gmin = t->gap_min[r];
      if (t->gap_max[r] > gmax) gmax = t->gap_max[r];
      for (int x = 0; x < NBINS; x++) {
        dh[x] += t->dur_hist[(uint64_t)r * NBINS + x];
        gh[x] += t->gap_hist[(uint64_t)r * NBINS + x];
      }
    }
    out->kernel_id[row] = keys[a].kid;
    out->task_id[row] = keys[a].task;
    out->dur_cnt[row] = dc;
    out->dur_sum[row] = ds;
    out->dur_min[row] = dmin;
    out->dur_max[row] = dmax;
    out->gap_cnt[row] = gc;
    out->gap_sum[row] = gs;
    out->gap_min[row] = gmin;
    out->gap_max[row] = gmax;
    out->dur_mean[row] = mean_of(ds, dc); /* SK_j over all parts */
    out->gap_mean[row] = mean_of(gs, gc); /* SG_j over all parts */
    row++;
    a = b;
  }
  out->n_rows = row;
  free(keys);
  return OR_OK;
}
