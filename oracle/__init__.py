"""ctypes binding of the FIKIT CPU oracle (oracle/fikit_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only callers.  The product
package (paper_2311_10359_b200) never imports this module.

Marshalling only -- every computation happens in the C file, which cites
the PAPER.md passages it follows.  Functions return numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fikit_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_ARG, E_RECORD, E_CAPACITY, E_NAME, E_COLLISION = 0, -1, -2, -3, -5, -99
NBINS = 32
NO_ROW = 0xFFFFFFFF


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


class _StrTab(C.Structure):
    _fields_ = [("bytes", C.c_void_p), ("offsets", C.c_void_p), ("count", C.c_uint32)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("pad", C.c_uint32), ("first_bad_index", C.c_uint64),
                ("n_rows_needed", C.c_uint64), ("n_overlap_gaps", C.c_uint64)]

    def as_dict(self):
        return {"code": self.code, "first_bad_index": self.first_bad_index, "n_rows_needed": self.n_rows_needed,
                "n_overlap_gaps": self.n_overlap_gaps}


class _Table(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("kernel_id", "task_id", "dur_cnt", "dur_sum", "dur_min", "dur_max",
                                          "gap_cnt", "gap_sum", "gap_min", "gap_max", "dur_hist", "gap_hist",
                                          "dur_mean", "gap_mean")] + [("capacity", C.c_uint32), ("n_rows", C.c_uint32)]


RESULT_DTYPE = np.dtype([("hp_jct", "<u8"), ("lp_jct", "<u8"), ("hp_delay", "<u8"), ("fill_work", "<u8"),
                         ("digest", "<u8"), ("n_fills", "<u4"), ("n_tail", "<u4")])
assert RESULT_DTYPE.itemsize == 48

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        u64, u32, p = C.c_uint64, C.c_uint32, C.c_void_p
        _lib.or_fnv1a64.restype = u64
        _lib.or_fnv1a64.argtypes = [p, u64]
        _lib.or_mix64.restype = u64
        _lib.or_mix64.argtypes = [u64]
        _lib.or_kernel_id.restype = u64
        _lib.or_kernel_id.argtypes = [p, u64, p, u64] + [u32] * 6
        _lib.or_identify.argtypes = [p, u64, _StrTab, _StrTab, p, C.POINTER(Status)]
        _lib.or_measure.argtypes = [p, u64, p, _StrTab, _StrTab, C.POINTER(_Table), p, C.POINTER(Status)]
        _lib.or_resolve.argtypes = [p, u64, p, _StrTab, _StrTab, p, p, u32, p, p, p, C.POINTER(Status)]
        _lib.or_best_prio_fit.restype = C.c_int64
        _lib.or_best_prio_fit.argtypes = [u32, p, p, p, p, u64]
        _lib.or_fikit_fill.restype = u32
        _lib.or_fikit_fill.argtypes = [u64, u64, u64, u64, u32, u32, p, p, p, p, p, p, p, p, p]
        _lib.or_fill_batch.argtypes = [p, p, p, p, p, p, p, u32, p, p, u32, u64, u32, p, p, p, p, p,
                                       C.POINTER(Status)]
        _lib.or_simulate.argtypes = [p, p, p, u32, p, p, p, u32, u32, p, p, p, u32, u64, u32, p, p, p]
        _lib.or_simulate_stream.argtypes = [p, p, p, u32, p, p, p, p, p, u32, u32, p, p, p, u32, u64, u32, u64, p, p,
                                            p]
        _lib.or_simulate_stream_batch.restype = C.c_int
        _lib.or_simulate_stream_batch.argtypes = [p, p, p, p, p, p, p, p, p, u32, p, p, p, u32, u64, u32, p, p, p, p,
                                                  p]
        _lib.or_predict.restype = C.c_int
        _lib.or_predict.argtypes = [C.POINTER(_Table), u32, u32]
        _lib.or_simulate_batch.argtypes = [p, p, p, p, p, p, p, u32, p, p, p, u32, u64, u32, p, p, p, p,
                                           C.POINTER(Status)]
        _lib.or_table_merge.argtypes = [C.POINTER(_Table), u32, C.POINTER(_Table), C.POINTER(Status)]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _st(tab) -> _StrTab:
    return _StrTab(_ptr(tab.data), _ptr(tab.offsets), tab.count)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------------------
def fnv1a64(b: bytes) -> int:
    buf = np.frombuffer(b or b"\0", dtype=np.uint8)
    return int(lib().or_fnv1a64(_ptr(buf), len(b)))


def mix64(x: int) -> int:
    return int(lib().or_mix64(x & 0xFFFFFFFFFFFFFFFF))


def kernel_id(name: bytes, sig: bytes, grid=(1, 1, 1), block=(1, 1, 1)) -> int:
    nb = np.frombuffer(name or b"\0", dtype=np.uint8)
    sb = np.frombuffer(sig or b"\0", dtype=np.uint8)
    return int(lib().or_kernel_id(_ptr(nb), len(name), _ptr(sb), len(sig), *grid, *block))


def identify(records: np.ndarray, names, sigs):
    st = Status()
    out = np.zeros(records.shape[0], dtype=np.uint64)
    lib().or_identify(_ptr(records), records.shape[0], _st(names), _st(sigs), _ptr(out), C.byref(st))
    return out, st.as_dict()


@dataclass
class Table:
    n_rows: int
    kernel_id: np.ndarray
    task_id: np.ndarray
    dur_cnt: np.ndarray
    dur_sum: np.ndarray
    dur_min: np.ndarray
    dur_max: np.ndarray
    gap_cnt: np.ndarray
    gap_sum: np.ndarray
    gap_min: np.ndarray
    gap_max: np.ndarray
    dur_hist: np.ndarray
    gap_hist: np.ndarray
    dur_mean: np.ndarray
    gap_mean: np.ndarray

    def head(self):
        """Arrays cut to n_rows."""
        n = self.n_rows
        return {k: (getattr(self, k)[:n]) for k in self.__dataclass_fields__ if k != "n_rows"}


def _table_arrays(cap: int) -> dict:
    arrs = {k: np.zeros(cap, dtype=np.uint64) for k in ("kernel_id", "dur_cnt", "dur_sum", "dur_min", "dur_max",
                                                       "gap_cnt", "gap_sum", "gap_min", "gap_max", "dur_mean",
                                                       "gap_mean")}
    arrs["task_id"] = np.zeros(cap, dtype=np.uint32)
    arrs["dur_hist"] = np.zeros((cap, NBINS), dtype=np.uint32)
    arrs["gap_hist"] = np.zeros((cap, NBINS), dtype=np.uint32)
    return arrs


def _ctable(tab: "Table") -> _Table:
    arrs = {k: getattr(tab, k) for k in tab.__dataclass_fields__ if k != "n_rows"}
    return _Table(**{k: _ptr(v) for k, v in arrs.items()}, capacity=arrs["kernel_id"].shape[0], n_rows=tab.n_rows)


def measure(records: np.ndarray, names, sigs, capacity: int | None = None, halo: np.ndarray | None = None,
            want_rows: bool = False):
    n = records.shape[0]
    cap = max(1, capacity if capacity is not None else n)
    arrs = _table_arrays(cap)
    t = _Table(**{k: _ptr(v) for k, v in arrs.items()}, capacity=cap, n_rows=0)
    rows = np.zeros(n, dtype=np.uint32) if want_rows else None
    st = Status()
    rec = np.ascontiguousarray(records)
    h = None if halo is None else np.ascontiguousarray(halo.reshape(1))
    lib().or_measure(_ptr(rec), n, _ptr(h), _st(names), _st(sigs), C.byref(t), _ptr(rows), C.byref(st))
    tab = Table(n_rows=t.n_rows, **arrs)
    return tab, st.as_dict(), rows


def table_merge(parts: list, capacity: int):
    """Union of per-shard tables (or_table_merge): returns (Table, status)."""
    arrs = _table_arrays(max(1, capacity))
    out = _Table(**{k: _ptr(v) for k, v in arrs.items()}, capacity=max(1, capacity), n_rows=0)
    cparts = (_Table * max(1, len(parts)))(*[_ctable(t) for t in parts])
    st = Status()
    lib().or_table_merge(cparts, len(parts), C.byref(out), C.byref(st))
    return Table(n_rows=out.n_rows, **arrs), st.as_dict()


def resolve(records: np.ndarray, names, sigs, tab: Table, halo: np.ndarray | None = None):
    n = records.shape[0]
    row = np.zeros(n, dtype=np.uint32)
    dur = np.zeros(n, dtype=np.uint64)
    gap = np.zeros(n, dtype=np.uint64)
    st = Status()
    rec = np.ascontiguousarray(records)
    h = None if halo is None else np.ascontiguousarray(halo.reshape(1))
    lib().or_resolve(_ptr(rec), n, _ptr(h), _st(names), _st(sigs), _ptr(tab.kernel_id), _ptr(tab.task_id),
                     tab.n_rows, _ptr(row), _ptr(dur), _ptr(gap), C.byref(st))
    return row, dur, gap, st.as_dict()


def best_prio_fit(q, elig, level, alive, R: int) -> tuple[int, np.ndarray]:
    q = _c(q, np.uint64)
    el = _c(elig, np.uint8)
    lv = _c(level, np.uint8)
    al = np.array(alive, dtype=np.uint8)
    k = int(lib().or_best_prio_fit(q.shape[0], _ptr(q), _ptr(el), _ptr(lv), _ptr(al), R))
    return k, al


def fikit_fill(R0: int, q, e, level, elig=None, t0: int = 0, deadline: int = 2**64 - 1, threshold: int = 100_000,
               feedback: int = 1, alive=None):
    """Alg. 1 on one gap.  Returns (picks, starts, R_left, t_end, alive)."""
    m = len(q)
    q = _c(q, np.uint64)
    e = _c(e, np.uint64)
    lv = _c(level, np.uint8)
    el = _c(np.ones(m) if elig is None else elig, np.uint8)
    al = _c(np.ones(m) if alive is None else alive, np.uint8)
    picks = np.zeros(max(m, 1), dtype=np.uint32)
    starts = np.zeros(max(m, 1), dtype=np.uint64)
    Rl = C.c_uint64()
    te = C.c_uint64()
    npk = lib().or_fikit_fill(R0, t0, deadline, threshold, feedback, m, _ptr(q), _ptr(e), _ptr(el), _ptr(lv),
                              _ptr(al), _ptr(picks), _ptr(starts), C.byref(Rl), C.byref(te))
    return picks[:npk].copy(), starts[:npk].copy(), Rl.value, te.value, al


def fill_batch(R0, deadline, pool_row, pool_dur, pool_level, pool_off, pool_len, tab: Table, threshold=100_000,
               feedback=1):
    G = len(R0)
    R0 = _c(R0, np.uint64)
    dl = _c(deadline, np.uint64)
    pr, pd, pl = _c(pool_row, np.uint32), _c(pool_dur, np.uint64), _c(pool_level, np.uint8)
    po, pn = _c(pool_off, np.uint32), _c(pool_len, np.uint32)
    poff = np.zeros(G, dtype=np.uint32)
    if G:
        poff[1:] = np.cumsum(pn[:-1])
    picks = np.zeros(max(1, int(pn.sum())), dtype=np.uint32)
    npk = np.zeros(G, dtype=np.uint32)
    Rl = np.zeros(G, dtype=np.uint64)
    tu = np.zeros(G, dtype=np.uint64)
    st = Status()
    lib().or_fill_batch(_ptr(R0), _ptr(dl), _ptr(pr), _ptr(pd), _ptr(pl), _ptr(po), _ptr(pn), G,
                        _ptr(tab.dur_mean), _ptr(tab.dur_cnt), tab.n_rows, threshold, feedback, _ptr(picks),
                        _ptr(poff), _ptr(npk), _ptr(Rl), _ptr(tu), C.byref(st))
    return picks, poff, npk, Rl, tu, st.as_dict()


def simulate(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, tab: Table, gap_scale_q16=1 << 16,
             threshold=100_000, feedback=1):
    """One scenario; returns (result record, fill_gap[m], lp_start[m])."""
    hr, hd, hg = _c(hp_row, np.uint32), _c(hp_dur, np.uint64), _c(hp_gap, np.uint64)
    lr, ld, ll = _c(lp_row, np.uint32), _c(lp_dur, np.uint64), _c(lp_level, np.uint8)
    m = lr.shape[0]
    out = np.zeros(1, dtype=RESULT_DTYPE)
    fg = np.zeros(max(m, 1), dtype=np.int32)
    ls = np.zeros(max(m, 1), dtype=np.uint64)
    lib().or_simulate(_ptr(hr), _ptr(hd), _ptr(hg), hr.shape[0], _ptr(lr), _ptr(ld), _ptr(ll), m, gap_scale_q16,
                      _ptr(tab.dur_mean), _ptr(tab.dur_cnt), _ptr(tab.gap_mean), tab.n_rows, threshold, feedback,
                      _ptr(out), _ptr(fg), _ptr(ls))
    return out[0], fg[:m].copy(), ls[:m].copy()


def simulate_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, scenarios, tab: Table, threshold=100_000,
                   feedback=1, want_schedule=False):
    hr, hd, hg = _c(hp_row, np.uint32), _c(hp_dur, np.uint64), _c(hp_gap, np.uint64)
    lr, ld, ll = _c(lp_row, np.uint32), _c(lp_dur, np.uint64), _c(lp_level, np.uint8)
    sc = np.ascontiguousarray(scenarios)
    S = sc.shape[0]
    out = np.zeros(S, dtype=RESULT_DTYPE)
    fg = ls = so = None
    if want_schedule:
        m = sc["lp_len"].astype(np.uint64)
        so = np.zeros(S, dtype=np.uint64)
        if S:
            so[1:] = np.cumsum(m[:-1])
        tot = max(1, int(m.sum()))
        fg = np.zeros(tot, dtype=np.int32)
        ls = np.zeros(tot, dtype=np.uint64)
    st = Status()
    lib().or_simulate_batch(_ptr(hr), _ptr(hd), _ptr(hg), _ptr(lr), _ptr(ld), _ptr(ll), _ptr(sc), S,
                            _ptr(tab.dur_mean), _ptr(tab.dur_cnt), _ptr(tab.gap_mean), tab.n_rows, threshold,
                            feedback, _ptr(out), _ptr(fg), _ptr(ls), _ptr(so), C.byref(st))
    return out, fg, ls, so, st.as_dict()


def simulate_stream_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, lp_stream, lp_think, scenarios,
                          tab: Table, threshold=100_000, feedback=1, hp_arrival=None):
    """STREAM-model replay (or_simulate_stream, R29-R32; hp_arrival per scenario: Case A, R33-R34);
    returns (results, fill_gap, lp_start, sched_off) with the schedule of every scenario at sched_off
    (cumulative lp_len)."""
    ha = None if hp_arrival is None else _c(hp_arrival, np.uint64)
    hr, hd, hg = _c(hp_row, np.uint32), _c(hp_dur, np.uint64), _c(hp_gap, np.uint64)
    lr, ld, ll = _c(lp_row, np.uint32), _c(lp_dur, np.uint64), _c(lp_level, np.uint8)
    ls_, lt = _c(lp_stream, np.uint32), _c(lp_think, np.uint64)
    sc = np.ascontiguousarray(scenarios)
    S = sc.shape[0]
    out = np.zeros(S, dtype=RESULT_DTYPE)
    m = sc["lp_len"].astype(np.uint64)
    so = np.zeros(S, dtype=np.uint64)
    if S:
        so[1:] = np.cumsum(m[:-1])
    tot = max(1, int(m.sum()))
    fg = np.zeros(tot, dtype=np.int32)
    ls = np.zeros(tot, dtype=np.uint64)
    rc = lib().or_simulate_stream_batch(_ptr(hr), _ptr(hd), _ptr(hg), _ptr(lr), _ptr(ld), _ptr(ll), _ptr(ls_),
                                        _ptr(lt), _ptr(sc), S, _ptr(tab.dur_mean), _ptr(tab.dur_cnt),
                                        _ptr(tab.gap_mean), tab.n_rows, threshold, feedback, _ptr(ha), _ptr(out),
                                        _ptr(fg), _ptr(ls), _ptr(so))
    if rc != 0:
        raise ValueError(f"or_simulate_stream_batch -> {rc}")
    return out, fg, ls, so


PREDICT_MEAN, PREDICT_PERCENTILE, PREDICT_EXTREMES = 0, 1, 2


def predict(tab: Table, mode: int, pct: int = 90) -> Table:
    """A copy of tab whose dur_mean / gap_mean columns hold the chosen predictor (or_predict:
    0 = the paper's means, 1 = conservative histogram percentile pct, 2 = max / min)."""
    arrs = {k: np.array(v, copy=True) for k, v in tab.__dict__.items() if k != "n_rows"}
    t = _Table(**{k: _ptr(v) for k, v in arrs.items()}, capacity=max(1, arrs["kernel_id"].shape[0]),
               n_rows=tab.n_rows)
    rc = lib().or_predict(C.byref(t), mode, pct)
    if rc != 0:
        raise ValueError(f"or_predict: mode {mode} pct {pct} -> {rc}")
    return Table(n_rows=tab.n_rows, **arrs)


def pipeline(cfg, capacity=None, predictor=None):
    """measure the config's trace, resolve its replay inputs, replay them; predictor =
    (mode, pct) rewrites the table's predictions first (predict())."""
    tr = cfg.trace
    tab, st, _ = measure(tr.records, tr.names, tr.sigs, capacity)
    if predictor is not None:
        tab = predict(tab, *predictor)
    res = {"table": tab, "status": st}
    if cfg.replay is not None:
        rp = cfg.replay
        hr, hd, hg, s1 = resolve(rp.hp_records, tr.names, tr.sigs, tab)
        lr, ld, _, s2 = resolve(rp.lp_records, tr.names, tr.sigs, tab)
        out, fg, ls, so, s3 = simulate_batch(hr, hd, hg, lr, ld, rp.lp_level, rp.scenarios, tab, rp.threshold_ns,
                                             rp.feedback, want_schedule=True)
        res.update(hp=(hr, hd, hg), lp=(lr, ld), results=out, fill_gap=fg, lp_start=ls, sched_off=so)
    return res
