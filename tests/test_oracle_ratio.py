"""Pins of the §4.3.2 ratio sweep (R35-R36), on the
oracle's STREAM-model replay:
- the exclusive arm (threshold = 2^64 - 1: no gap is ever filled) equals the closed form of
  P:103 / P:478, JCT_B,excl = JCT_A + JCT_B, summed here from the resolved kernels with numpy
  (no replay code involved);
- FIKIT never makes the single LP stream finish later than exclusive mode (derivation in
  DESIGN.md R36), and HP JCT = solo + delay;
- prefix: once B has run entirely inside A's first r tasks, more A tasks change nothing;
- the paper's trend on the synthetic pairs: at 1:1 the two modes are close, from 10:1 on the
  exclusive/FIKIT ratio grows linearly with r ("a linear upward trend")."""
import numpy as np
import pytest

import fikit_synth as F
import oracle as O

NO_FILL = (1 << 64) - 1


@pytest.fixture(scope="module")
def sweep():
    cfg, sr, rat = F.ratio_sweep(n_base=12)
    tr, rp = cfg.trace, cfg.replay
    tab, st, _ = O.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    assert st["code"] == 0
    hr, hd, hg, _ = O.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, lg, _ = O.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    args = (hr, hd, hg, lr, ld, rp.lp_level, sr.lp_stream, lg, rp.scenarios, tab)
    fik = O.simulate_stream_batch(*args, rp.threshold_ns, 1)
    exc = O.simulate_stream_batch(*args, NO_FILL, 1)
    return dict(sc=rp.scenarios, rat=rat, hd=hd, hg=hg, ld=ld, lg=lg, fik=fik, exc=exc)


def test_exclusive_arm_is_the_closed_form(sweep):
    sc, hd, hg, ld, lg = sweep["sc"], sweep["hd"], sweep["hg"], sweep["ld"], sweep["lg"]
    exc = sweep["exc"][0]
    assert np.all(exc["n_fills"] == 0) and np.all(exc["hp_delay"] == 0)
    for s, c in enumerate(sc):
        h0, nh, l0, m, q = int(c["hp_off"]), int(c["hp_len"]), int(c["lp_off"]), int(c["lp_len"]), int(c["gap_scale_q16"])
        # JCT_A solo: every HP kernel plus every scaled think time but the last (R20, R24)
        solo = int(hd[h0:h0 + nh].sum()) + sum((int(a) * q) >> 16 for a in hg[h0:h0 + nh - 1])
        # JCT_B solo: one stream (ids equal in the window), kernels plus think times but the last
        jb = int(ld[l0:l0 + m].sum()) + int(lg[l0:l0 + m - 1].sum())
        assert int(exc["hp_jct"][s]) == solo
        assert int(exc["lp_jct"][s]) == solo + jb, s
        assert int(exc["n_tail"][s]) == m


def test_fikit_lp_never_later_than_exclusive(sweep):
    f, e = sweep["fik"][0], sweep["exc"][0]
    assert np.all(f["lp_jct"] <= e["lp_jct"])
    assert np.all(f["hp_jct"] == e["hp_jct"] + f["hp_delay"])  # hp_jct = solo + delay
    assert f["n_fills"].sum() > 0


def test_prefix_more_hp_tasks_change_nothing_once_b_is_done(sweep):
    sc, rat = sweep["sc"], sweep["rat"]
    f, fg, ls, so = sweep["fik"]
    R = len(F.RATIOS)
    done = 0
    for g0 in range(0, sc.shape[0], R):  # one group = one base, scale and pair, all ratios
        for i in range(R):
            if f["n_tail"][g0 + i] == 0:
                for j in range(i + 1, R):
                    a, b = g0 + i, g0 + j
                    assert rat[b] > rat[a]
                    assert (f["lp_jct"][b], f["digest"][b], f["n_fills"][b], f["fill_work"][b]) == \
                           (f["lp_jct"][a], f["digest"][a], f["n_fills"][a], f["fill_work"][a])
                    m = int(sc["lp_len"][a])
                    assert np.array_equal(ls[so[a]:so[a] + m], ls[so[b]:so[b] + m])
                done += 1
                break
    assert done > 0


def _series(sweep, pair, scale_i):
    """mean exclusive/FIKIT LP JCT per ratio for one (pair, scale) series"""
    f, e = sweep["fik"][0], sweep["exc"][0]
    S, R, ns = f.shape[0], len(F.RATIOS), len(F.RATIO_SCALES_Q16)
    s = np.arange(S)
    g = s // R
    out = []
    for ri in range(R):
        sel = (s % R == ri) & (g % ns == scale_i) & ((g // ns) % 2 == pair)
        out.append(float(np.mean(e["lp_jct"][sel] / f["lp_jct"][sel])))
    return np.array(out)


def test_linear_upward_trend(sweep):
    # (A = VGG, B = BERT) at HP gaps x4 and x16: B completes inside A's gaps from 10:1 on, so
    # its FIKIT JCT stays constant while the exclusive one grows by r * JCT_A
    for scale_i in (1, 2):
        y = _series(sweep, 1, scale_i)
        assert y[0] < 1.5  # 1:1: "close to that of the FIKIT mode"
        steps = np.diff(y[1:])  # 10:1 .. 50:1
        assert np.all(steps > 0)
        assert np.max(steps) / np.min(steps) < 1.25  # equal increments: linear
    # (A = BERT, B = VGG) at x1: the first VGG kernel fits no BERT gap, so B waits for the tail
    # in both modes and the ratio stays 1 (a pair that FIKIT cannot help)
    assert np.allclose(_series(sweep, 0, 0), 1.0)
