"""Pins of oracle.predict (R26-R28): the predictor variants are
checked against brute force on the raw samples a row's histogram was built from (numpy
percentiles, bit lengths taken with Python ints), not by re-typing their formulas."""
import numpy as np
import pytest

import oracle as O


def _bin(v: int) -> int:
    return min(31, int(v).bit_length())


def _pctl(vals, P):
    """smallest v with #{x <= v} * 100 >= P * n"""
    s = sorted(vals)
    k = -(-P * len(s) // 100)  # ceil
    return s[max(k, 1) - 1]


def _table(rows):
    """an oracle Table from per-row raw (durations, gaps) lists"""
    n = len(rows)
    z = lambda: np.zeros(n, dtype=np.uint64)
    t = O.Table(n_rows=n, kernel_id=z(), task_id=np.zeros(n, np.uint32), dur_cnt=z(), dur_sum=z(), dur_min=z(),
                dur_max=z(), gap_cnt=z(), gap_sum=z(), gap_min=z(), gap_max=z(),
                dur_hist=np.zeros((n, 32), np.uint32), gap_hist=np.zeros((n, 32), np.uint32), dur_mean=z(),
                gap_mean=z())
    for r, (ds, gs) in enumerate(rows):
        for vals, cnt, sm, mn, mx, h in ((ds, t.dur_cnt, t.dur_sum, t.dur_min, t.dur_max, t.dur_hist),
                                         (gs, t.gap_cnt, t.gap_sum, t.gap_min, t.gap_max, t.gap_hist)):
            cnt[r] = len(vals)
            sm[r] = sum(vals) % (1 << 64)
            mn[r] = min(vals) if vals else (1 << 64) - 1
            mx[r] = max(vals) if vals else 0
            for v in vals:
                h[r, _bin(v)] += 1
    return t


def _random_rows(seed, n_rows=60):
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(n_rows):
        n = int(rng.integers(1, 200))
        kind = rng.integers(0, 4)
        if kind == 0:  # one kernel, +-5 %: a single bin mostly
            base = int(rng.integers(1000, 1 << 22))
            ds = [int(base * rng.uniform(0.95, 1.05)) for _ in range(n)]
        elif kind == 1:  # log-uniform over 2 us .. 2 s, includes bin 31 (>= 2^30 ns)
            ds = [int(np.exp(rng.uniform(np.log(2e3), np.log(2e9)))) for _ in range(n)]
        elif kind == 2:  # zeros and tiny values (bins 0, 1)
            ds = [int(v) for v in rng.integers(0, 3, size=n)]
        else:  # a bimodal mixture ("same ID, different duration")
            ds = [int(rng.choice([50_000, 4_000_000]) * rng.uniform(0.9, 1.1)) for _ in range(n)]
        ng = int(rng.integers(0, n + 1))
        gs = [int(v) for v in np.exp(rng.uniform(np.log(1), np.log(3e7), size=ng)).astype(np.int64)]
        rows.append((ds, gs))
    return rows


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("P", [1, 10, 50, 90, 99])
def test_percentile_brackets_raw_percentile(seed, P):
    rows = _random_rows(seed)
    t = O.predict(_table(rows), O.PREDICT_PERCENTILE, P)
    for r, (ds, gs) in enumerate(rows):
        d, g = int(t.dur_mean[r]), int(t.gap_mean[r])
        v = _pctl(ds, P)  # the P-th percentile duration
        assert v <= d <= max(ds), (r, v, d)  # conservative: never under the percentile, never over the max
        assert _bin(d) == _bin(v) or d == max(ds), (r, v, d)  # and inside its histogram bin
        if gs:
            w = _pctl(gs, 100 - P)  # the (100 - P)-th percentile gap
            assert min(gs) <= g <= w, (r, w, g)
            assert _bin(g) == _bin(w) or g == min(gs), (r, w, g)
        else:
            assert g == 0


def test_single_valued_rows_are_exact():
    # a row whose samples all equal x predicts x (the bin edge is clamped to max / min)
    rows = [([1000] * 7, [700] * 5), ([0] * 3, [0]), ([(1 << 40) + 3] * 2, [(1 << 35)] * 4)]
    t = O.predict(_table(rows), O.PREDICT_PERCENTILE, 90)
    assert t.dur_mean.tolist() == [1000, 0, (1 << 40) + 3]
    assert t.gap_mean.tolist() == [700, 0, 1 << 35]


def test_extremes_and_means():
    rows = _random_rows(9)
    t0 = _table(rows)
    t2 = O.predict(t0, O.PREDICT_EXTREMES)
    for r, (ds, gs) in enumerate(rows):
        assert int(t2.dur_mean[r]) == max(ds)
        assert int(t2.gap_mean[r]) == (min(gs) if gs else 0)
    # mode 0: R8 means, the numpy way (floor + half up)
    t1 = O.predict(t0, O.PREDICT_MEAN)
    for r, (ds, gs) in enumerate(rows):
        for vals, got in ((ds, int(t1.dur_mean[r])), (gs, int(t1.gap_mean[r]))):
            if not vals:
                assert got == 0
                continue
            s, n = sum(vals), len(vals)
            assert got in (s // n, s // n + 1) and abs(2 * (got * n - s)) <= n  # nearest, ties up
            if 2 * (s % n) == n:
                assert got == s // n + 1


def test_measured_table_mode0_matches_measure_and_rows_without_samples():
    import fikit_synth as F

    cfg = F.toy()
    tab, _, _ = O.measure(cfg.trace.records, cfg.trace.names, cfg.trace.sigs)
    t = O.predict(tab, O.PREDICT_MEAN)
    assert np.array_equal(t.dur_mean, tab.dur_mean) and np.array_equal(t.gap_mean, tab.gap_mean)
    empty = _table([([5], []), ([], [])])
    for mode in (0, 1, 2):
        e = O.predict(empty, mode, 50)
        assert int(e.gap_mean[0]) == 0 and int(e.dur_mean[1]) == 0 and int(e.gap_mean[1]) == 0


@pytest.mark.parametrize("mode,P", [(3, 50), (1, 0), (1, 100)])
def test_bad_arguments(mode, P):
    with pytest.raises(ValueError):
        O.predict(_table([([1], [1])]), mode, P)
