"""Parity at the sizes bench.py runs (configs[3] in full, its replay leg, and the Z64k
stress variant), GPU (C-ABI) against the oracle, bit for bit.

  - configs[3]: 100,000,000 launches, 8,192 rows.  The whole table (every row, every
    field) and every launch's row (out_row) are compared with or_measure run once on the
    same records (about a minute on one host core).  The table is measured in the
    launch configuration bench.py times (no out_row) and again with out_row.
  - The bench's replay leg over that table (fikit_synth.zipf_replay: 100,000 scenarios,
    m = 64, HP runs of 256 kernels, gap scales 1..8) in the no-schedule instantiation
    bench.py times: results of 2,500 sampled scenarios replayed one by one by the
    oracle, then the schedule (fill_gap, lp_start) of the same sample from a second run
    with schedule outputs.
  - Z64k (SURVEY §8d config Z stress variant): 32 tasks x 2,048-kernel vocabularies
    (up to 65,536 rows), 2,048,000 launches, the whole table."""
import os

import numpy as np
import pytest

import fikit_synth as F
from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

TABLE_FIELDS = ("kernel_id", "task_id", "dur_cnt", "dur_sum", "dur_min", "dur_max", "gap_cnt", "gap_sum", "gap_min",
                "gap_max", "dur_hist", "gap_hist", "dur_mean", "gap_mean")


@pytest.fixture(scope="module")
def fk():
    import paper_2311_10359_b200 as fk
    from paper_2311_10359_b200 import _build

    _build.build()
    return fk


def assert_tables_equal(got: dict, ref_tab, ctx=""):
    ref = ref_tab.head()
    assert got["kernel_id"].shape[0] == ref_tab.n_rows, f"{ctx}: n_rows {got['kernel_id'].shape[0]} vs {ref_tab.n_rows}"
    for k in TABLE_FIELDS:
        a, b = np.asarray(got[k]), np.asarray(ref[k])
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)[:5]
            raise AssertionError(f"{ctx}: field {k} differs at {bad.tolist()}: gpu {a[tuple(bad[0])]} "
                                 f"oracle {b[tuple(bad[0])]}")


@pytest.fixture(scope="module")
def z100m(orc):
    cfg = F.zipf_trace(threads=min(16, os.cpu_count() or 8))
    assert cfg.trace.records.shape[0] == 100_000_000
    ref, rst, rrows = orc.measure(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=8192, want_rows=True)
    assert rst["code"] == 0
    return cfg, ref, rst, rrows


def test_zipf_100m_full_table_and_rows(fk, orc, z100m):
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg, ref, rst, rrows = z100m
    tr = cfg.trace
    # bench.py's configuration: fikit_measure without out_row, then finalize
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=8192)
    p.run_measure()
    st = p.check("zipf 100M")
    assert 8000 < ref.n_rows <= 8192
    assert st["n_rows_needed"] == ref.n_rows and st["schedule"] == 1
    assert st["n_overlap_gaps"] == rst["n_overlap_gaps"]
    assert_tables_equal(p.table.to_numpy(), ref, "zipf-100M")
    # every launch's canonical row (fikit_measure out_row + fikit_table_finalize remap)
    del p
    q = Pipeline(tr.records, tr.names, tr.sigs, capacity=8192, want_rows=True)
    q.run_measure()
    q.check("zipf 100M rows")
    assert_tables_equal(q.table.to_numpy(), ref, "zipf-100M (out_row run)")
    rows = q.rows()
    if not np.array_equal(rows, rrows):
        bad = np.flatnonzero(rows != rrows)[:5]
        raise AssertionError(f"out_row differs at {bad.tolist()}: gpu {rows[bad]} oracle {rrows[bad]}")


def test_zipf_replay_leg_sampled(fk, orc, z100m):
    """the bench's replay leg over the 100M table, 2,500 sampled scenarios (results + schedule)"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg, ref, _, _ = z100m
    tr = cfg.trace
    rp = F.zipf_replay(cfg, S=100_000)
    S = rp.scenarios.shape[0]
    pick = np.sort(np.random.default_rng(12).choice(S, 2500, replace=False))
    sc = rp.scenarios[pick].copy()
    hp_idx = np.concatenate([np.arange(c["hp_off"], c["hp_off"] + c["hp_len"]) for c in sc])
    lp_idx = np.concatenate([np.arange(c["lp_off"], c["lp_off"] + c["lp_len"]) for c in sc])
    hr, hd, hg, s1 = orc.resolve(rp.hp_records[hp_idx], tr.names, tr.sigs, ref)
    lr, ld, _, s2 = orc.resolve(rp.lp_records[lp_idx], tr.names, tr.sigs, ref)
    assert s1["code"] == 0 and s2["code"] == 0
    sc["hp_off"] = np.concatenate([[0], np.cumsum(sc["hp_len"][:-1])])
    sc["lp_off"] = np.concatenate([[0], np.cumsum(sc["lp_len"][:-1])])
    out, fg, ls, rso, st = orc.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level[lp_idx], sc, ref, rp.threshold_ns,
                                              rp.feedback, want_schedule=True)
    assert st["code"] == 0 and out["n_fills"].sum() > 0
    for want_schedule in (False, True):  # bench.py's instantiation first
        p = Pipeline(tr.records, tr.names, tr.sigs, capacity=8192, replay=rp, want_schedule=want_schedule,
                     checked=True)
        p.step()
        got = p.results()
        if got[pick].tobytes() != out.tobytes():
            bad = np.flatnonzero(got[pick] != out)[:5]
            raise AssertionError(f"scenarios {pick[bad].tolist()} differ: {got[pick][bad]} vs {out[bad]}")
        assert (got["n_tail"] != 0xFFFFFFFF).all()  # every scenario replayed (none left deferred)
        if want_schedule:
            gfg, gls = p.schedule()
            m = rp.scenarios["lp_len"].astype(np.int64)
            so = np.concatenate([[0], np.cumsum(m[:-1])])
            for j, s in enumerate(pick):
                a, b, n = int(so[s]), int(rso[j]), int(m[s])
                assert np.array_equal(gfg[a:a + n], fg[b:b + n]) and np.array_equal(gls[a:a + n], ls[b:b + n]), s
        del p


def test_z64k_full_table(fk, orc):
    """2,048-kernel vocabularies per task -> up to 65,536 rows, most launches
    outside any CTA's hot set (the cold path, dynamic admission)"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.zipf_trace(n_runs=8000, vocab_per_task=2048, threads=min(16, os.cpu_count() or 8))
    tr = cfg.trace
    ref, rst, rrows = orc.measure(tr.records, tr.names, tr.sigs, capacity=65536, want_rows=True)
    assert rst["code"] == 0 and ref.n_rows > 30_000
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=65536, want_rows=True)
    p.run_measure()
    st = p.check("z64k")
    assert st["n_rows_needed"] == ref.n_rows and st["n_overlap_gaps"] == rst["n_overlap_gaps"]
    assert_tables_equal(p.table.to_numpy(), ref, "z64k")
    assert np.array_equal(p.rows(), rrows)
    # too small a table: E_CAPACITY with the exact number of rows needed
    q = Pipeline(tr.records, tr.names, tr.sigs, capacity=ref.n_rows - 1)
    q.run_measure()
    st = fk.get_status(q.ws)
    assert st["code"] == fk.E_CAPACITY and st["n_rows_needed"] == ref.n_rows
