"""Oracle pins for the measurement statistics (readings R3-R11).

Pins: the paper's SK/SG worked example, the run magnitudes of
P:240-241, SPEC S:140 (single-kernel run), rounding cases, a numpy group-by
(np.unique / np.add.at / np.minimum.at / np.maximum.at) over random traces,
permutation invariance over run order, error cases."""
import numpy as np
import pytest

import fikit_synth as F
from helpers import MS, US, Labeled, golden_lines


def test_paper_worked_example_sk_sg(orc):
    lines = list(golden_lines("paper_sk_sg.txt"))
    runs = {}
    for ln in lines:
        tok = ln.split()
        if tok[0] == "expect":
            exp = dict(zip(tok[2::2], map(int, tok[3::2])))
            continue
        run, pos, k, d, g = int(tok[0]), int(tok[1]), tok[2], float(tok[3]), tok[4]
        runs.setdefault(run, []).append((k, int(d * MS), None if g == "-" else int(float(g) * MS)))
    L = Labeled()
    rec = L.records([runs[1], runs[2]])
    names, sigs = L.strtabs()
    tab, st, rows = orc.measure(rec, names, sigs, want_rows=True)
    assert st["code"] == 0
    j = rows[0]
    assert tab.dur_cnt[j] == exp["dur_cnt"] and tab.dur_mean[j] == exp["dur_mean_ms"] * MS
    assert tab.gap_cnt[j] == exp["gap_cnt"] and tab.gap_mean[j] == exp["gap_mean_ms"] * MS
    assert tab.n_rows == 5  # S_UID = {j, x1, x2, x3, x4}
    x4 = rows[5]
    assert tab.gap_cnt[x4] == 0 and tab.gap_mean[x4] == 0  # last kernel of every run: no SG sample


def test_paper_run_magnitudes(orc):
    g = {ln.split()[0]: [int(x) for x in ln.split()[1:] if x.isdigit()] for ln in golden_lines("paper_run_magnitudes.txt")}
    n_rows, n_gaps, solo_ms = g["expect"]
    d, gp = g["dur_ms"], g["gap_ms"]
    L = Labeled()
    run = [(f"k{i}", d[i] * MS, gp[i] * MS if i < len(gp) else None) for i in range(len(d))]
    rec = L.records([run])
    names, sigs = L.strtabs()
    tab, st, rows = orc.measure(rec, names, sigs, want_rows=True)
    assert st["code"] == 0 and tab.n_rows == n_rows
    assert int(tab.gap_cnt[:4].sum()) == n_gaps  # N_t - 1 idling times
    for i in range(4):
        assert tab.dur_mean[rows[i]] == d[i] * MS and tab.dur_cnt[rows[i]] == 1
    for i in range(3):
        assert tab.gap_mean[rows[i]] == gp[i] * MS
    assert tab.gap_cnt[rows[3]] == 0
    # solo replay (no LP): JCT = sum exec + sum gaps = 44 ms
    hr, hd, hg, _ = orc.resolve(rec, names, sigs, tab)
    res, _, _ = orc.simulate(hr, hd, hg, [], [], [], tab)
    assert res["hp_jct"] == solo_ms * MS and res["hp_delay"] == 0


def test_single_kernel_run_has_no_gap(orc):
    # single run, single kernel, 5000 us -> SK = 5000 us, no SG entry
    L = Labeled()
    rec = L.records([[("a", 5000 * US, None)]])
    tab, st, _ = orc.measure(rec, *L.strtabs())
    assert tab.n_rows == 1 and tab.dur_mean[0] == 5000 * US and tab.gap_cnt[0] == 0 and tab.gap_mean[0] == 0
    assert tab.gap_min[0] == 2**64 - 1 and tab.gap_max[0] == 0  # empty min/max (R9)


@pytest.mark.parametrize("durs,mean", [((2, 2, 3, 3), 3), ((2, 2, 2, 3), 2), ((1, 2), 2), ((0, 1, 1), 1),
                                       ((5,), 5), ((0,), 0)])
def test_mean_rounding_half_up(orc, durs, mean):
    # reading R8: integer ns mean, round half up (sum 10 / cnt 4 -> 3; sum 9 / 4 -> 2)
    L = Labeled()
    rec = L.records([[("a", d, None)] for d in durs])
    tab, st, _ = orc.measure(rec, *L.strtabs())
    assert tab.dur_sum[0] == sum(durs) and tab.dur_cnt[0] == len(durs) and tab.dur_mean[0] == mean


def _bit_length(v):
    return np.array([int(x).bit_length() for x in v], dtype=np.int64)


def numpy_groupby(orc, rec, names, sigs, halo=None):
    """The statistics via numpy group-by (library routines), independent of
    the oracle's sort-and-walk; kernel IDs come from orc.identify (pinned by
    test_oracle_hash)."""
    kid, st = orc.identify(rec, names, sigs)
    n = rec.shape[0]
    key = np.stack([rec["task_id"].astype(np.uint64), kid], axis=1)
    uk, inv = np.unique(key, axis=0, return_inverse=True)
    inv = inv.ravel()
    K = uk.shape[0]
    d = rec["end_ns"] - rec["start_ns"]
    nxt = np.concatenate([rec[1:], halo.reshape(1)]) if halo is not None else rec[1:]
    has = np.zeros(n, bool)
    m = nxt.shape[0]
    has[:m] = (nxt["task_id"] == rec["task_id"][:m]) & (nxt["run_id"] == rec["run_id"][:m])
    raw = np.zeros(n, dtype=np.int64)
    raw[:m] = nxt["start_ns"].astype(np.int64) - rec["end_ns"][:m].astype(np.int64)
    g = np.where(raw > 0, raw, 0).astype(np.uint64)
    out = {"kernel_id": uk[:, 1], "task_id": uk[:, 0].astype(np.uint32)}
    for nm, v, sel in (("dur", d, np.ones(n, bool)), ("gap", g, has)):
        cnt = np.zeros(K, np.uint64)
        np.add.at(cnt, inv[sel], 1)
        s = np.zeros(K, np.uint64)
        np.add.at(s, inv[sel], v[sel])
        mn = np.full(K, 2**64 - 1, np.uint64)
        np.minimum.at(mn, inv[sel], v[sel])
        mx = np.zeros(K, np.uint64)
        np.maximum.at(mx, inv[sel], v[sel])
        h = np.zeros((K, 32), np.uint32)
        np.add.at(h, (inv[sel], np.minimum(31, _bit_length(v[sel]))), 1)
        out.update({nm + "_cnt": cnt, nm + "_sum": s, nm + "_min": mn, nm + "_max": mx, nm + "_hist": h})
    out["n_overlap"] = int((has & (raw < 0)).sum())
    return out


@pytest.mark.parametrize("seed,kw", [(1, {}), (2, {"overlap_frac": 0.2}), (3, {"zero_frac": 0.3}),
                                     (4, {"big_frac": 0.1, "n_tasks": 1}), (5, {"run_len_max": 1}),
                                     (6, {"n_ids": 1, "n_tasks": 1}), (7, {"n_ids": 200, "n_tasks": 5})])
def test_measure_vs_numpy_groupby(orc, seed, kw):
    tr = F.random_trace(seed, 3000, **kw)
    tab, st, _ = orc.measure(tr.records, tr.names, tr.sigs)
    ref = numpy_groupby(orc, tr.records, tr.names, tr.sigs)
    assert st["code"] == 0 and st["n_overlap_gaps"] == ref["n_overlap"]
    h = tab.head()
    assert tab.n_rows == ref["kernel_id"].shape[0]
    for k, v in ref.items():
        if k != "n_overlap":
            assert np.array_equal(h[k], v), k


def test_measure_halo(orc):
    # a shard's last gap uses the first record of the next shard (multi-GPU split)
    tr = F.random_trace(11, 1000, run_len_max=60)
    full, _, _ = orc.measure(tr.records, tr.names, tr.sigs)
    cut = 437
    a, sa, _ = orc.measure(tr.records[:cut], tr.names, tr.sigs, halo=tr.records[cut])
    b, sb, _ = orc.measure(tr.records[cut:], tr.names, tr.sigs)
    ref = numpy_groupby(orc, tr.records[:cut], tr.names, tr.sigs, halo=tr.records[cut])
    assert np.array_equal(a.head()["gap_sum"], ref["gap_sum"])
    # merge by key: sums add, min/max combine -> equals the unsharded table
    merged = {}
    for t in (a, b):
        for r in range(t.n_rows):
            k = (int(t.task_id[r]), int(t.kernel_id[r]))
            e = merged.setdefault(k, [0, 0, 2**64 - 1, 0])
            e[0] += int(t.gap_cnt[r]); e[1] += int(t.gap_sum[r])
            e[2] = min(e[2], int(t.gap_min[r])); e[3] = max(e[3], int(t.gap_max[r]))
    for r in range(full.n_rows):
        k = (int(full.task_id[r]), int(full.kernel_id[r]))
        assert merged[k] == [int(full.gap_cnt[r]), int(full.gap_sum[r]), int(full.gap_min[r]), int(full.gap_max[r])]


def test_measure_run_order_invariant(orc):
    # SK_j and SG_j are permutation-invariant over run order
    tr = F.random_trace(12, 2000, run_len_max=30)
    rec = tr.records
    runs = np.split(np.arange(rec.shape[0]), np.flatnonzero(np.diff(rec["run_id"].astype(np.int64))) + 1)
    order = np.random.default_rng(1).permutation(len(runs))
    rec2 = rec[np.concatenate([runs[i] for i in order])]
    t1, _, _ = orc.measure(rec, tr.names, tr.sigs)
    t2, _, _ = orc.measure(rec2, tr.names, tr.sigs)
    for k, v in t1.head().items():
        assert np.array_equal(v, t2.head()[k]), k


def test_task_scoping(orc):
    # R3: the same kernel in two tasks is two rows (profiles are per Task Key)
    L = Labeled()
    r0 = L.records([[("a", 10, 5), ("a", 20, None)]], task=0)
    r1 = L.records([[("a", 30, None)]], task=1, run_base=0)
    tab, st, _ = orc.measure(np.concatenate([r0, r1]), *L.strtabs())
    assert tab.n_rows == 2 and tab.kernel_id[0] == tab.kernel_id[1] and list(tab.task_id[:2]) == [0, 1]
    assert list(tab.dur_sum[:2]) == [30, 30] and tab.gap_cnt[0] == 1 and tab.gap_cnt[1] == 0


def test_errors(orc):
    tr = F.random_trace(13, 500)
    rec = tr.records.copy()
    rec["end_ns"][123] = rec["start_ns"][123] - 1  # R4: end < start
    _, st, _ = orc.measure(rec, tr.names, tr.sigs)
    assert st["code"] == orc.E_RECORD and st["first_bad_index"] == 123
    tab, st, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=3)
    full, _, _ = orc.measure(tr.records, tr.names, tr.sigs)
    assert st["code"] == orc.E_CAPACITY and st["n_rows_needed"] == full.n_rows
    tab, st, _ = orc.measure(tr.records[:0], tr.names, tr.sigs)
    assert st["code"] == 0 and tab.n_rows == 0


def test_toy_golden_regression(orc):
    """The oracle still reproduces tests/golden/toy_oracle.json (make_toy.py)."""
    import json
    import os

    from helpers import GOLDEN

    g = json.load(open(os.path.join(GOLDEN, "toy_oracle.json")))
    cfg = F.toy()
    for fb in (1, 0):
        cfg.replay.feedback = fb
        r = orc.pipeline(cfg)
        for k, v in r["table"].head().items():
            assert v.tolist() == g["table"][k], k
        res = r["results"][0]
        assert {k: int(res[k]) for k in res.dtype.names} == g[f"feedback{fb}"]["result"]
        assert r["fill_gap"].tolist() == g[f"feedback{fb}"]["fill_gap"]
