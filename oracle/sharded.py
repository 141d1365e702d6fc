"""All-core driver of the CPU oracle (SURVEY §8d "Oracle timing (ii) All host cores: the sharded
driver") -- TEST INFRASTRUCTURE ONLY, like the rest of oracle/.

The oracle's functions stay single-threaded and plain (oracle/fikit_oracle.c); this module only
splits one job over host threads and puts the pieces back together:

  measure   contiguous record shards, each with the next shard's first record as its halo (R5:
            every boundary gap counted exactly once), one or_measure per shard, then
            or_table_merge (the union of the parts' rows, statistics summed / min'd / max'd,
            means recomputed: SURVEY §8e)
  resolve   contiguous record shards with a halo, results concatenated
  replay    contiguous scenario slices, results concatenated

ctypes releases the GIL for the duration of each C call, so the shards run in parallel on a
thread pool.  Known limit: the oracle's collision check (R2) runs within a shard, not across
shards -- the single-threaded oracle is the checker for parity; this driver is the all-core
baseline.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import OK, RESULT_DTYPE, Table, measure as _measure, resolve as _resolve, simulate_batch as _simulate_batch
from . import simulate_stream_batch as _simulate_stream_batch
from . import table_merge


def host_threads() -> int:
    """The threads this process may run on (the CPU set, not the machine's core count)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _ranges(n: int, parts: int):
    parts = max(1, min(parts, n)) if n else 1
    return [(n * i // parts, n * (i + 1) // parts) for i in range(parts)]


def measure(records: np.ndarray, names, sigs, capacity: int, threads: int | None = None):
    """(Table, status) of the whole trace; equals oracle.measure(records, ...) bit for bit."""
    threads = threads or host_threads()
    n = records.shape[0]
    rg = _ranges(n, threads)

    def one(lo_hi):
        lo, hi = lo_hi
        halo = records[hi] if hi < n else None
        return _measure(records[lo:hi], names, sigs, capacity=capacity, halo=halo)

    with ThreadPoolExecutor(len(rg)) as ex:
        parts = list(ex.map(one, rg))
    for (lo, _), (_, st, _) in zip(rg, parts):  # the first shard with an error decides (lowest index)
        if st["code"] != OK:
            st = dict(st)
            if st["code"] != -3:
                st["first_bad_index"] += lo
            return None, st
    tab, st = table_merge([p[0] for p in parts], capacity)
    st["n_overlap_gaps"] = sum(p[1]["n_overlap_gaps"] for p in parts)
    return tab, st


def resolve(records: np.ndarray, names, sigs, tab: Table, threads: int | None = None):
    threads = threads or host_threads()
    n = records.shape[0]
    rg = _ranges(n, threads)

    def one(lo_hi):
        lo, hi = lo_hi
        return _resolve(records[lo:hi], names, sigs, tab, halo=records[hi] if hi < n else None)

    with ThreadPoolExecutor(len(rg)) as ex:
        parts = list(ex.map(one, rg))
    cat = lambda i: np.concatenate([p[i] for p in parts]) if parts else np.zeros(0)
    return cat(0), cat(1), cat(2)


def simulate_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, scenarios, tab: Table, threshold=100_000,
                   feedback=1, threads: int | None = None):
    """Results of every scenario (no schedule); equals oracle.simulate_batch's results."""
    threads = threads or host_threads()
    S = scenarios.shape[0]
    rg = _ranges(S, threads)

    def one(lo_hi):
        lo, hi = lo_hi
        out, _, _, _, st = _simulate_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level,
                                           np.ascontiguousarray(scenarios[lo:hi]), tab, threshold, feedback)
        return out

    with ThreadPoolExecutor(len(rg)) as ex:
        parts = list(ex.map(one, rg))
    return np.concatenate(parts) if parts else np.zeros(0, dtype=RESULT_DTYPE)


def simulate_stream_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, lp_stream, lp_think, scenarios,
                          tab: Table, threshold=100_000, feedback=1, hp_arrival=None, threads: int | None = None):
    threads = threads or host_threads()
    S = scenarios.shape[0]
    rg = _ranges(S, threads)

    def one(lo_hi):
        lo, hi = lo_hi
        ha = None if hp_arrival is None else hp_arrival[lo:hi]
        out, _, _, _ = _simulate_stream_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, lp_stream,
                                              lp_think, np.ascontiguousarray(scenarios[lo:hi]), tab, threshold,
                                              feedback, hp_arrival=ha)
        return out

    with ThreadPoolExecutor(len(rg)) as ex:
        parts = list(ex.map(one, rg))
    return np.concatenate(parts) if parts else np.zeros(0, dtype=RESULT_DTYPE)
