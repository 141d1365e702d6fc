"""Oracle pins for Algorithm 1 (FIKIT), Algorithm 2 (BestPrioFit), runtime
feedback and the batch replay (readings R12-R24).

Pins: Fig. fillIdling, Fig. runtimeFeedback,
SPEC fill/best-fit examples, a sort-based second oracle for
BestPrioFit, brute-force optimal fills on tiny pools, closed forms
(solo JCT, exclusive JCT_B = JCT_A + JCT_B of P:103, perfect prediction), and
replay invariants on random scenarios."""
import itertools

import numpy as np
import pytest

import fikit_synth as F
from helpers import MS, US, golden_lines, hand_table

INF = 2**64 - 1


def _scenario(orc, hp_dur, hp_gap, hp_pred, lp_q, lp_e, lp_level, feedback, threshold=100 * US):
    """HP kernel i uses row i (SG = hp_pred[i]); LP request k uses row n_h + k (SK = lp_q[k])."""
    nh, m = len(hp_dur), len(lp_q)
    pred = list(hp_pred) + [0] * (nh - len(hp_pred))
    tab = hand_table(orc, [1] * nh + list(lp_q), pred + [0] * m)
    return orc.simulate(np.arange(nh), hp_dur, list(hp_gap) + [0], np.arange(nh, nh + m), lp_e, lp_level, tab,
                        threshold=threshold, feedback=feedback)


@pytest.mark.parametrize("feedback", [0, 1])
def test_paper_fill_idling(orc, feedback):
    # Ak1-Bk1-Ck1-Ak2
    res, fg, ls = _scenario(orc, [500 * US, 500 * US], [1000 * US], [1000 * US], [400 * US, 300 * US],
                            [400 * US, 300 * US], [1, 2], feedback)
    assert list(fg) == [0, 0]  # B and C both fill the gap after Ak1
    assert ls[0] == 500 * US and ls[1] == 900 * US  # order A B C, then A at 1500
    assert res["hp_delay"] == 0 and res["hp_jct"] == 2000 * US and res["n_fills"] == 2


def test_paper_fill_idling_variant_early_stop(orc):
    res, fg, ls = _scenario(orc, [500 * US, 500 * US], [300 * US], [1000 * US], [400 * US, 300 * US],
                            [400 * US, 300 * US], [1, 2], 1)
    assert list(fg) == [0, -1] and res["hp_delay"] == 100 * US and res["n_fills"] == 1 and res["n_tail"] == 1


def test_paper_runtime_feedback(orc):
    g = {ln.split()[0]: ln.split()[1:] for ln in golden_lines("paper_runtime_feedback.txt") if not ln.startswith("expect")}
    exp = [ln.split() for ln in golden_lines("paper_runtime_feedback.txt") if ln.startswith("expect")]
    p, a = int(g["p_us"][0]) * US, int(g["a_us"][0]) * US
    q = [int(x) * US for x in g["lp_q_us"]]
    for e in exp:
        fb, nf, dl = int(e[2]), int(e[4]), int(e[6]) * US
        res, fg, _ = _scenario(orc, [1 * MS, 1 * MS], [a], [p], q, q, [1] * len(q), fb)
        assert res["n_fills"] == nf and res["hp_delay"] == dl, e


def test_spec_fill_cases(orc):
    for ln in golden_lines("spec_fill_cases.txt"):
        body = ln.split(";")[0]
        lhs, rhs = body.split("->")
        tok = lhs.split()
        kind, R = tok[0], int(tok[1]) * US
        reqs = [] if tok[2] == "-" else [x.split(":") for x in tok[2].split(",")]
        lv = [int(r[0]) for r in reqs]
        q = [int(r[1]) * US for r in reqs]
        seq = [int(r[2]) if len(r) > 2 else i for i, r in enumerate(reqs)]
        order = np.argsort(seq, kind="stable")  # pool position = arrival seq order
        lv, q, seq = [lv[i] for i in order], [q[i] for i in order], [seq[i] for i in order]
        want = rhs.split()[0]
        if kind == "fill":
            picks, _, _, _, _ = orc.fikit_fill(R, q, q, lv, threshold=100 * US, feedback=0)
            got = [q[k] // US for k in picks]
            assert got == ([] if want == "none" else [int(x) for x in want.split(",")]), ln
        else:
            k, _ = orc.best_prio_fit(q, [1] * len(q), lv, [1] * len(q), R)
            if want == "none":
                assert k == -1, ln
            elif want.startswith("seq"):
                assert seq[k] == int(want[3:]), ln
            else:
                assert q[k] == int(want) * US, ln


def test_no_profile_no_fill(orc):
    # S:271 / R12: no SG entry -> predicted 0 -> zero fills; S:257 / R16: no SK -> never a fill
    res, fg, _ = _scenario(orc, [MS, MS], [5 * MS], [0], [US], [US], [1], 1)
    assert res["n_fills"] == 0 and res["n_tail"] == 1
    nh = 2
    tab = hand_table(orc, [1, 1, 100 * US], [5 * MS, 0, 0], dur_cnt=[1, 1, 0])
    res, fg, _ = orc.simulate([0, 1], [MS, MS], [5 * MS, 0], [2, 77], [100 * US, 100 * US], [1, 1], tab)
    assert res["n_fills"] == 0 and res["n_tail"] == 2


def _sort_best(q, elig, level, alive, R):
    # S:276 second oracle: filter by fit, sort by (level asc, q desc, seq asc), take first
    c = [(level[k], -q[k], k) for k in range(len(q)) if alive[k] and elig[k] and q[k] <= R and 1 <= level[k] <= 9]
    return sorted(c)[0][2] if c else -1


def test_best_prio_fit_vs_sort_oracle(orc):
    rng = np.random.default_rng(0)
    for _ in range(3000):
        m = int(rng.integers(0, 12))
        q = rng.integers(0, 20, size=m)
        lv = rng.integers(1, 4, size=m)
        el = rng.random(m) < 0.9
        al = rng.random(m) < 0.8
        R = int(rng.integers(0, 25))
        k, al2 = orc.best_prio_fit(q, el, lv, al, R)
        assert k == _sort_best(q, el, lv, al, R)
        if k >= 0:
            assert al2[k] == 0 and al2.sum() == al.sum() - 1


def test_bruteforce_optimal_fill(orc):
    """greedy <= OPT <= R; one level, no feedback: greedy >= OPT/2 (SURVEY §8c-5 proof)."""
    rng = np.random.default_rng(1)
    for it in range(400):
        m = int(rng.integers(1, 12))
        q = rng.integers(1, 50, size=m)
        R = int(rng.integers(100, 200))
        single = it % 2 == 0
        lv = np.ones(m, int) if single else rng.integers(1, 4, size=m)
        picks, _, Rl, _, _ = orc.fikit_fill(R, q, q, lv, threshold=0, feedback=0)
        got = int(q[picks].sum())
        opt = max(sum(c) for r in range(m + 1) for c in itertools.combinations(q.tolist(), r) if sum(c) <= R)
        assert got <= opt <= R and Rl == R - got
        if single:
            assert 2 * got >= opt
        # maximality: nothing alive still fits
        rest = np.setdiff1d(np.arange(m), picks)
        assert all(q[k] > Rl for k in rest)


def test_closed_forms(orc):
    rng = np.random.default_rng(2)
    for _ in range(50):
        nh, m = int(rng.integers(1, 20)), int(rng.integers(0, 20))
        d = rng.integers(1, MS, size=nh)
        a = rng.integers(1, 3 * MS, size=nh)
        e = rng.integers(1, MS, size=m)
        lv = rng.integers(1, 4, size=m)
        solo = int(d.sum() + a[:-1].sum())
        # no LP: JCT = sum exec + sum gaps
        res, _, _ = _scenario(orc, d, a[:-1], a[:-1], [], [], [], 1)
        assert res["hp_jct"] == solo and res["lp_jct"] == 0
        # tau = inf: exclusive order A then B, JCT_B,actual = JCT_A + JCT_B
        res, fg, ls = _scenario(orc, d, a[:-1], a[:-1], e, e, lv, 1, threshold=INF)
        assert res["hp_jct"] == solo and (fg == -1).all()
        assert res["lp_jct"] == (solo + int(e.sum()) if m else 0)  # R22: m = 0 -> 0
        # perfect prediction (p = a', q = e): HP unaffected in both feedback modes
        for fb in (0, 1):
            res, fg, ls = _scenario(orc, d, a[:-1], a[:-1], e, e, lv, fb)
            assert res["hp_delay"] == 0 and res["hp_jct"] == solo


def test_replay_invariants(orc):
    rng = np.random.default_rng(3)
    for it in range(300):
        nh, m = int(rng.integers(1, 15)), int(rng.integers(0, 25))
        fb = it % 2
        d = rng.integers(1, MS, size=nh)
        a = rng.integers(1, 3 * MS, size=nh)
        pred = (a * rng.uniform(0.3, 2.5, size=nh)).astype(np.int64)
        q = rng.integers(1, MS, size=m)
        e = (q * rng.uniform(0.5, 1.5, size=m)).astype(np.int64) + 1
        lv = rng.integers(1, 4, size=m)
        res, fg, ls = _scenario(orc, d, a[:-1], pred[:-1], q, e, lv, fb)
        solo = int(d.sum() + a[:-1].sum())
        assert res["hp_jct"] == solo + res["hp_delay"]  # hp_jct = solo + hp_delay
        assert res["n_fills"] + res["n_tail"] == m  # conservation: every request runs once
        assert res["fill_work"] == int(e[fg >= 0].sum())
        # device timeline: HP kernels + LP requests never overlap
        t, hp_iv = 0, []
        for i in range(nh):  # rebuild HP intervals from the schedule
            fills = sorted((ls[k], k) for k in range(m) if fg[k] == i - 1) if i else []
            start = max([t] + [ls[k] + e[k] for _, k in fills])
            if i:
                start = max(start, hp_iv[-1][1] + a[i - 1])
            hp_iv.append((start, start + d[i]))
            t = start + d[i]
        iv = sorted(hp_iv + [(ls[k], ls[k] + e[k]) for k in range(m)])
        assert all(iv[j][1] <= iv[j + 1][0] for j in range(len(iv) - 1))
        assert hp_iv[-1][1] == res["hp_jct"]
        for i in range(nh - 1):
            ks = [k for k in range(m) if fg[k] == i]
            # fit safety: sum of predicted q of the gap's fills <= p_i
            assert sum(q[k] for k in ks) <= pred[i]
            if ks and pred[i] < 100 * US:
                assert False, "gap below threshold was filled"
            # monotone picks: dispatch order follows (level, -q, seq)
            order = sorted(ks, key=lambda k: ls[k])
            keys = [(lv[k], -q[k], k) for k in order]
            assert keys == sorted(keys)
            # feedback bound: delay imposed on HP kernel i+1 <= e of the gap's last fill
            if fb and ks:
                r = hp_iv[i][1] + a[i]
                last = order[-1]
                assert max(0, ls[last] + e[last] - r) <= e[last]
                assert all(ls[k] < r for k in order)  # every fill dispatched before HP's arrival
        # tail in (level, seq) order, back to back after the HP job
        tail = sorted((k for k in range(m) if fg[k] == -1), key=lambda k: ls[k])
        assert [(lv[k], k) for k in tail] == sorted((lv[k], k) for k in tail)
        if tail:
            assert ls[tail[0]] == res["hp_jct"]


def test_feedback_never_worse(orc):
    # feedback delay <= no-feedback delay on every seed
    rng = np.random.default_rng(4)
    for _ in range(200):
        nh, m = int(rng.integers(2, 12)), int(rng.integers(1, 30))
        d = rng.integers(1, MS, size=nh)
        a = rng.integers(1, 2 * MS, size=nh)
        pred = (a * rng.uniform(1.0, 3.0, size=nh)).astype(np.int64)  # over-prediction
        q = rng.integers(1, MS, size=m)
        lv = rng.integers(1, 3, size=m)
        r1, _, _ = _scenario(orc, d, a[:-1], pred[:-1], q, q, lv, 1)
        r0, _, _ = _scenario(orc, d, a[:-1], pred[:-1], q, q, lv, 0)
        assert r1["hp_delay"] <= r0["hp_delay"]


def test_equal_levels_pure_best_fit(orc):
    rng = np.random.default_rng(5)
    for _ in range(200):
        m = int(rng.integers(1, 15))
        q = rng.integers(1, 100, size=m)
        R = int(rng.integers(50, 300))
        picks, _, _, _, _ = orc.fikit_fill(R, q, q, [4] * m, threshold=0, feedback=0)
        rem, al, want = R, np.ones(m, bool), []
        while True:
            c = [k for k in range(m) if al[k] and q[k] <= rem]
            if not c:
                break
            k = max(c, key=lambda k: (q[k], -k))
            want.append(k)
            al[k] = False
            rem -= q[k]
        assert list(picks) == want


def test_simulate_batch_matches_single(orc):
    tr = F.random_trace(21, 2000)
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs)
    rp = F.random_replay(22, tr, 40)
    hr, hd, hg, _ = orc.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, _, _ = orc.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    out, fg, ls, so, st = orc.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level, rp.scenarios, tab, rp.threshold_ns,
                                             rp.feedback, want_schedule=True)
    assert st["code"] == 0
    for s, c in enumerate(rp.scenarios):
        h = slice(c["hp_off"], c["hp_off"] + c["hp_len"])
        l = slice(c["lp_off"], c["lp_off"] + c["lp_len"])
        r1, fg1, ls1 = orc.simulate(hr[h], hd[h], hg[h], lr[l], ld[l], rp.lp_level[l], tab, c["gap_scale_q16"],
                                    rp.threshold_ns, rp.feedback)
        assert r1 == out[s]
        o = int(so[s])
        assert np.array_equal(fg[o:o + c["lp_len"]], fg1) and np.array_equal(ls[o:o + c["lp_len"]], ls1)
