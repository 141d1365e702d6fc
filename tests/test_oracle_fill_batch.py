"""Oracle pins for the batch fill (or_fill_batch: Alg. 1 over G independent gaps,
PAPER.md P:328-334) and for the task scoping of the profile lookup (or_resolve,
P:278 "filter out the profiling data matching the Task Key"; reading R3).

or_fill_batch derives each request's predicted duration q from the table (SK of
its row, R16: a row that is absent or has no duration samples never fills),
rebuilds the pool for every gap, and applies the threshold gate and the feedback
deadline per gap.  Each of those steps is pinned here against something other
than the function itself: the SPEC examples laid out as one batch,
hand-worked eligibility cases, and per-gap calls of or_fikit_fill (itself pinned
by test_oracle_fill.py) with q and eligibility taken from the hand table in
plain Python."""
import numpy as np

import fikit_synth as F
from helpers import MS, US, Labeled, golden_lines, hand_table

INF = 2**64 - 1


def _batch(orc, tab, gaps, threshold=100 * US, feedback=0):
    """gaps: list of (R0, deadline, [(row, dur, level), ...])."""
    G = len(gaps)
    R0 = np.array([g[0] for g in gaps], np.uint64)
    dl = np.array([g[1] for g in gaps], np.uint64)
    pool_len = np.array([len(g[2]) for g in gaps], np.uint32)
    pool_off = np.zeros(G, np.uint32)
    if G:
        pool_off[1:] = np.cumsum(pool_len[:-1])
    flat = [r for g in gaps for r in g[2]]
    pool_row = np.array([r[0] for r in flat], np.uint32)
    pool_dur = np.array([r[1] for r in flat], np.uint64)
    pool_level = np.array([r[2] for r in flat], np.uint8)
    picks, poff, npk, Rl, tu, st = orc.fill_batch(R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len, tab,
                                                  threshold=threshold, feedback=feedback)
    assert st["code"] == 0
    return [picks[poff[g]:poff[g] + npk[g]].tolist() for g in range(G)], Rl, tu


def _spec_fill_cases():
    out = []
    for ln in golden_lines("spec_fill_cases.txt"):
        body = ln.split(";")[0]
        lhs, rhs = body.split("->")
        tok = lhs.split()
        if tok[0] != "fill":
            continue
        reqs = [x.split(":") for x in tok[2].split(",")]
        want = rhs.split()[0]
        out.append((int(tok[1]) * US, [(int(r[0]), int(r[1]) * US) for r in reqs],
                    [] if want == "none" else [int(x) * US for x in want.split(",")]))
    return out


def test_spec_cases_as_one_batch(orc):
    """S:249-251 as gaps of one batch; each case twice, the second copy reusing the first's
    table rows: the pool is rebuilt per gap (a request picked in one gap is alive in the next)."""
    cases = _spec_fill_cases()
    assert len(cases) == 3
    qs = sorted({q for _, reqs, _ in cases for _, q in reqs})
    row_of = {q: r for r, q in enumerate(qs)}
    tab = hand_table(orc, qs, [0] * len(qs))  # row r: SK = qs[r], one duration sample
    gaps, want = [], []
    for _rep in range(2):
        for R, reqs, exp in cases:
            gaps.append((R, INF, [(row_of[q], q, lv) for lv, q in reqs]))
            want.append(exp)
    got, Rl, tu = _batch(orc, tab, gaps)
    for g, (picks, exp) in enumerate(zip(got, want)):
        R, reqs, _ = cases[g % len(cases)]
        assert [reqs[k][1] for k in picks] == exp, (g, picks)
        assert int(Rl[g]) == R - sum(exp) and int(tu[g]) == sum(exp)  # actual e = q here


def test_eligibility_from_the_table(orc):
    """R16: a request whose row is absent (>= n_rows) or has no duration samples (dur_cnt = 0)
    never fills, whatever its SK; the others fill by Alg. 2's order."""
    # rows: 0 SK 3 ms (1 sample), 1 SK 2 ms but dur_cnt 0, 2 SK 1 ms (1 sample)
    tab = hand_table(orc, [3 * MS, 2 * MS, 1 * MS], [0, 0, 0], dur_cnt=[1, 0, 1])
    pool = [(1, 2 * MS, 1),    # k0: level 1 but no samples -> never
            (7, 5 * MS, 1),    # k1: absent row -> never
            (0, 3 * MS, 2),    # k2: level 2, q 3 ms
            (2, 1 * MS, 2),    # k3: level 2, q 1 ms
            (2, 1 * MS, 3)]    # k4: level 3, q 1 ms
    got, Rl, tu = _batch(orc, tab, [(10 * MS, INF, pool), (3 * MS, INF, pool), (4500 * US, INF, pool)])
    assert got[0] == [2, 3, 4] and Rl[0] == 5 * MS  # everything eligible fits; level 2 first, q desc
    assert got[1] == [2] and Rl[1] == 0             # 3 ms fills R exactly (q <= R inclusive, R14)
    assert got[2] == [2, 3] and Rl[2] == 500 * US   # 1.5 ms left -> the level-2 1 ms request before level 3
    assert int(tu[2]) == 4 * MS


def test_gate_and_deadline_per_gap(orc):
    """Alg. 1 lines 6-8 (R13: R0 < threshold -> no fill) and the feedback stop (R19: dispatch
    iff t < deadline, tie -> HP), each applied to its own gap of the batch."""
    tab = hand_table(orc, [300 * US], [0])
    pool = [(0, 400 * US, 1), (0, 400 * US, 1), (0, 400 * US, 1)]  # predicted 300 us, actual 400 us
    gaps = [(99 * US, INF, pool),     # below the 0.1 ms gate
            (100 * US, INF, pool),    # at the gate: opens, but no q fits 100 us
            (1000 * US, 0, pool),     # deadline 0: t = 0 >= 0 -> nothing dispatched
            (1000 * US, 400 * US, pool),  # one fill ends at 400 = deadline -> stop (tie -> HP)
            (1000 * US, 401 * US, pool),  # t = 400 < 401 -> a second fill (overruns)
            (1000 * US, INF, pool)]   # three fills (R = 1000 - 3 * 300 = 100)
    got, Rl, tu = _batch(orc, tab, gaps, feedback=1)
    assert [len(g) for g in got] == [0, 0, 0, 1, 2, 3]
    assert list(Rl) == [99 * US, 100 * US, 1000 * US, 700 * US, 400 * US, 100 * US]
    assert list(tu) == [0, 0, 0, 400 * US, 800 * US, 1200 * US]
    got0, _, _ = _batch(orc, tab, gaps, feedback=0)  # feedback off: the deadline is ignored
    assert [len(g) for g in got0] == [0, 0, 3, 3, 3, 3]


def test_batch_equals_per_gap_fill(orc):
    """Random batches: every gap equals or_fikit_fill on that gap's pool alone, with q and the
    eligibility read off the table here (q = SK[row] if row < n_rows and dur_cnt[row] > 0)."""
    rng = np.random.default_rng(7)
    for it in range(40):
        n = int(rng.integers(1, 30))
        sk = rng.integers(0, 3 * MS, size=n)
        cnt = (rng.random(n) < 0.8).astype(np.uint64)
        tab = hand_table(orc, sk, [0] * n, dur_cnt=cnt)
        G = int(rng.integers(1, 25))
        gaps = []
        for _ in range(G):
            m = int(rng.integers(0, 40))
            pool = [(int(rng.integers(0, n + 3)), int(rng.integers(1, 3 * MS)), int(rng.integers(1, 10)))
                    for _ in range(m)]
            R0 = int(rng.integers(0, 10 * MS))
            dl = INF if rng.random() < 0.5 else int(rng.integers(0, 5 * MS))
            gaps.append((R0, dl, pool))
        fb = int(it % 2)
        got, Rl, tu = _batch(orc, tab, gaps, feedback=fb)
        for g, (R0, dl, pool) in enumerate(gaps):
            rows = [p[0] for p in pool]
            el = [1 if (r < n and cnt[r] > 0) else 0 for r in rows]
            q = [int(sk[r]) if e else 0 for r, e in zip(rows, el)]
            picks, _, rl, te, _ = orc.fikit_fill(R0, q, [p[1] for p in pool], [p[2] for p in pool], elig=el,
                                                 deadline=dl, feedback=fb)
            assert got[g] == picks.tolist() and Rl[g] == rl and tu[g] == te, (it, g)


def test_resolve_is_scoped_by_task(orc):
    """P:278 / R3: two tasks launch the identical kernel (same name, grid, block) with different
    durations; each task's fresh launches resolve to its own row (its own SK), and a task
    without a profile resolves to no row even though the kernel ID exists for other tasks."""
    L = Labeled()
    a = L.records([[("shared", 1 * MS, 2 * MS), ("shared", 1 * MS, None)]], task=0)
    b = L.records([[("shared", 5 * MS, 7 * MS), ("shared", 5 * MS, None)]], task=1, run_base=10)
    names, sigs = L.strtabs()
    rec = np.concatenate([a, b])
    tab, st, _ = orc.measure(rec, names, sigs)
    assert st["code"] == 0 and tab.n_rows == 2
    assert tab.kernel_id[0] == tab.kernel_id[1]  # one kernel ID, two Task Keys
    fresh = np.concatenate([L.records([[("shared", 3 * MS, None)]], task=t, run_base=100 + t) for t in (1, 0, 2)])
    rows, dur, gap, st = orc.resolve(fresh, names, sigs, tab)
    assert st["code"] == 0
    assert list(rows) == [1, 0, 0xFFFFFFFF]
    assert tab.task_id[rows[0]] == 1 and tab.dur_mean[rows[0]] == 5 * MS and tab.gap_mean[rows[0]] == 7 * MS
    assert tab.task_id[rows[1]] == 0 and tab.dur_mean[rows[1]] == 1 * MS and tab.gap_mean[rows[1]] == 2 * MS
    assert list(dur) == [3 * MS] * 3 and list(gap) == [0, 0, 0]  # three one-launch runs: no gaps
