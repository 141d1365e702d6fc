"""Host-side logic of bench.py's N > 1 path (CPU): a rank keeps only the HP / LP launches its
scenario shard references (compact_replay); the shard's replay results must not change."""
import importlib.util
import os

import numpy as np
import pytest

import fikit_synth as F
import oracle as O
from paper_2311_10359_b200.dist import scenario_shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("world", [2, 3])
def test_compact_replay_pool(bench, world):
    cfg = F.bert_vgg(S=2000)
    tr, rp = cfg.trace, cfg.replay
    ref = O.pipeline(cfg, capacity=1024)["results"]
    for r in range(world):
        sel = scenario_shard(2000, r, world)
        sub = F.Replay(rp.hp_records, rp.lp_records, rp.lp_level, rp.scenarios[sel], rp.threshold_ns, rp.feedback)
        c, _ = bench.compact_replay(sub)
        assert c.lp_records.shape[0] < rp.lp_records.shape[0]
        out = O.pipeline(F.Config("shard", tr, c), capacity=1024)["results"]
        assert out.tobytes() == ref[sel].tobytes()


def test_compact_replay_stream_and_empty_windows(bench):
    cfg, sr = F.bert_vgg_stream(S=600, n_lp_runs=200)
    tr, rp = cfg.trace, cfg.replay
    tab, _, _ = O.measure(tr.records, tr.names, tr.sigs, capacity=1024)

    def run(r, ls):
        hr, hd, hg, _ = O.resolve(r.hp_records, tr.names, tr.sigs, tab)
        lr, ld, lg, _ = O.resolve(r.lp_records, tr.names, tr.sigs, tab)
        return O.simulate_stream_batch(hr, hd, hg, lr, ld, r.lp_level, ls, lg, r.scenarios, tab, r.threshold_ns,
                                       r.feedback)[0]

    sc = rp.scenarios.copy()
    sc["lp_len"][::7] = 0  # empty windows keep offset 0 after compaction
    rp = F.Replay(rp.hp_records, rp.lp_records, rp.lp_level, sc, rp.threshold_ns, rp.feedback)
    full = run(rp, sr.lp_stream)
    sel = scenario_shard(600, 1, 4)
    sub = F.Replay(rp.hp_records, rp.lp_records, rp.lp_level, sc[sel], rp.threshold_ns, rp.feedback)
    c, ls = bench.compact_replay(sub, sr.lp_stream)
    assert run(c, ls).tobytes() == full[sel].tobytes()


def test_cpu_baseline_leg(bench):
    # the all-core oracle leg of the bench line (SURVEY §8d oracle timing (i) + (ii)) on a small workload
    cfg = F.bert_vgg(S=3000)
    wl = dict(records=cfg.trace.records, names=cfg.trace.names, sigs=cfg.trace.sigs, replay=cfg.replay,
              N=cfg.trace.records.shape[0], cap=1024, lp_stream=None, hp_arrival=None, ratio=None)
    cb = bench.cpu_baseline(wl, 4.0)
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["single_core"]["cores"] == 1 and cb["single_core"]["value"] > 0
    assert cb["full_pass"]  # this small workload fits the budget: no extrapolation
    t, n1, s1 = bench.oracle_pass(wl, 0.25, 2)
    assert n1 == round(0.25 * wl["N"]) and s1 == 750 and t > 0
