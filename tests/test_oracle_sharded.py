"""Pins for the all-core oracle driver (oracle/sharded.py, SURVEY §8d "Oracle timing (ii)") and
its table merge (or_table_merge).

The single-threaded oracle is pinned by the other test_oracle_* files; the sharded driver must
reproduce it exactly on every split (integer sum / min / max are associative and commutative, and
the halo gives each boundary gap to exactly one shard), including splits that cut runs, shards of
one record, more threads than records, and error reports at global indices."""
import numpy as np
import pytest

import fikit_synth as F


@pytest.fixture(scope="module")
def sh(orc):
    import oracle.sharded as S

    return S


@pytest.mark.parametrize("threads", [1, 2, 3, 7, 16])
@pytest.mark.parametrize("kind", ["plain", "overlap", "zeros_big"])
def test_sharded_measure_equals_oracle(orc, sh, threads, kind):
    kw = {"plain": {}, "overlap": {"overlap_frac": 0.2}, "zeros_big": {"zero_frac": 0.1, "big_frac": 0.05}}[kind]
    tr = F.random_trace(100 + threads, 3001, n_tasks=4, n_ids=60, run_len_max=50, **kw)
    ref, st_ref, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=512)
    got, st = sh.measure(tr.records, tr.names, tr.sigs, capacity=512, threads=threads)
    assert st["code"] == 0 and st_ref["code"] == 0
    assert st["n_overlap_gaps"] == st_ref["n_overlap_gaps"]
    assert got.n_rows == ref.n_rows
    for k, v in ref.head().items():
        assert np.array_equal(got.head()[k], v), k


def test_sharded_measure_tiny_and_empty(orc, sh):
    tr = F.random_trace(7, 5, run_len_max=3)
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=16)
    got, st = sh.measure(tr.records, tr.names, tr.sigs, capacity=16, threads=64)  # more threads than records
    assert st["code"] == 0
    for k, v in ref.head().items():
        assert np.array_equal(got.head()[k], v), k
    empty, st = sh.measure(tr.records[:0], tr.names, tr.sigs, capacity=16, threads=4)
    assert st["code"] == 0 and empty.n_rows == 0


def test_sharded_measure_errors_at_global_index(orc, sh):
    tr = F.random_trace(8, 2000, run_len_max=20)
    rec = tr.records.copy()
    rec["end_ns"][1500] = rec["start_ns"][1500] - 1  # R4: end < start
    rec["flags"][1700] = 1
    _, st_ref, _ = orc.measure(rec, tr.names, tr.sigs, capacity=512)
    _, st = sh.measure(rec, tr.names, tr.sigs, capacity=512, threads=5)
    assert st["code"] == st_ref["code"] == -2
    assert st["first_bad_index"] == st_ref["first_bad_index"] == 1500


def test_table_merge_capacity(orc, sh):
    # every shard fits its capacity, the union does not: the merge reports the rows it needs
    tr = F.random_trace(9, 4000, n_tasks=1, n_ids=80, run_len_max=30)
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=4096)
    cap = ref.n_rows - 1
    parts = [orc.measure(tr.records[lo:hi], tr.names, tr.sigs, capacity=4096)[0]
             for lo, hi in ((0, 2000), (2000, 4000))]
    assert all(p.n_rows <= 4096 for p in parts)
    _, st = orc.table_merge(parts, cap)
    assert st["code"] == -3 and st["n_rows_needed"] == ref.n_rows


def test_table_merge_is_union_by_hand(orc):
    # two hand-made parts: one shared row, one row each -> sums add, min/max combine, means recomputed
    from helpers import hand_table

    a = hand_table(orc, [0, 0], [0, 0])
    b = hand_table(orc, [0, 0], [0, 0])
    a.task_id[:2], a.kernel_id[:2] = [0, 0], [5, 9]
    b.task_id[:2], b.kernel_id[:2] = [0, 1], [9, 5]
    a.dur_cnt[:2], a.dur_sum[:2], a.dur_min[:2], a.dur_max[:2] = [1, 2], [10, 7], [10, 3], [10, 4]
    b.dur_cnt[:2], b.dur_sum[:2], b.dur_min[:2], b.dur_max[:2] = [2, 1], [2, 4], [1, 4], [1, 4]
    a.dur_hist[1, 2] = 2
    b.dur_hist[0, 1] = 2
    out, st = orc.table_merge([a, b], 8)
    assert st["code"] == 0 and out.n_rows == 3
    # canonical order (task, kid): (0,5), (0,9), (1,5)
    assert list(out.task_id[:3]) == [0, 0, 1] and list(out.kernel_id[:3]) == [5, 9, 5]
    assert list(out.dur_cnt[:3]) == [1, 4, 1] and list(out.dur_sum[:3]) == [10, 9, 4]
    assert list(out.dur_min[:3]) == [10, 1, 4] and list(out.dur_max[:3]) == [10, 4, 4]
    assert list(out.dur_mean[:3]) == [10, 2, 4]  # 9 / 4 = 2.25 -> 2 (R8)
    assert out.dur_hist[1, 1] == 2 and out.dur_hist[1, 2] == 2


def test_sharded_resolve_and_replay_equal_oracle(orc, sh):
    tr = F.random_trace(21, 2500, n_tasks=3, n_ids=40, run_len_max=30)
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    rp = F.random_replay(22, tr, 120, m_max=50, n_h_max=40, levels=9)
    ref_r = orc.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    got_r = sh.resolve(rp.hp_records, tr.names, tr.sigs, tab, threads=6)
    for a, b in zip(ref_r[:3], got_r):
        assert np.array_equal(a, b)
    hr, hd, hg, _ = ref_r
    lr, ld, _, _ = orc.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    ref, _, _, _, _ = orc.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level, rp.scenarios, tab, rp.threshold_ns,
                                         rp.feedback)
    got = sh.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level, rp.scenarios, tab, rp.threshold_ns, rp.feedback,
                            threads=7)
    assert got.tobytes() == ref.tobytes()
