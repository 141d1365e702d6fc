"""GPU edge cases through the C-ABI: fikit_lookup, the documented m <= 1024 limits
(FIKIT_E_ARG in the status, include/fikit.h), and the sorted-pool fast path at
idle times >= 2^32 ns (R0, predicted gaps) with more than 32 eligible requests,
including predicted durations at the 32-bit boundary.  Expected values come from
the oracle (oracle/) on the same inputs."""
import numpy as np
import pytest

import fikit_synth as F
from helpers import MS, US, hand_table

pytestmark = pytest.mark.gpu

INF = 2**64 - 1


@pytest.fixture(scope="module")
def fk():
    from conftest import cuda_ok

    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2311_10359_b200 as fk
    from paper_2311_10359_b200 import _build

    _build.build()
    return fk


def _d(a, dt):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()


def device_table(fk, dur_mean, gap_mean, dur_cnt):
    """A device table holding only what the replay reads: n_rows, dur_cnt, SK, SG."""
    import torch

    n = len(dur_mean)
    t = fk.Table(max(8, n))
    sums = np.zeros((t.capacity, 4), np.uint64)
    sums[:n, 0] = dur_cnt
    mean = np.zeros((t.capacity, 2), np.uint64)
    mean[:n, 0] = dur_mean
    mean[:n, 1] = gap_mean
    t.sums.copy_(torch.from_numpy(sums.reshape(-1).view(np.int64)))
    t.mean.copy_(torch.from_numpy(mean.reshape(-1).view(np.int64)))
    t.n_rows_t.fill_(n)
    return t


def _fill_gpu(fk, tab, R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len, poff, feedback):
    import torch

    G = len(R0)
    tot = max(1, int(np.sum(pool_len)))
    ws = fk.Workspace(1, 1, 1)
    g_picks = torch.zeros(tot, dtype=torch.int32, device="cuda")
    g_np = torch.full((G,), -7, dtype=torch.int32, device="cuda")
    g_R = torch.zeros(G, dtype=torch.int64, device="cuda")
    g_t = torch.zeros(G, dtype=torch.int64, device="cuda")
    fk.fill(tab, _d(R0, np.int64), _d(dl, np.int64), _d(pool_row, np.int32), _d(pool_dur, np.int64),
            _d(pool_level, np.uint8), _d(pool_off, np.int32), _d(pool_len, np.int32), G, g_picks,
            _d(poff, np.int32), g_np, g_R, g_t, ws, feedback=feedback)
    return ws, g_picks.cpu().numpy().view(np.uint32), g_np.cpu().numpy(), g_R.cpu().numpy().view(np.uint64), \
        g_t.cpu().numpy().view(np.uint64)


def test_lookup_parity(fk, orc):
    """fikit_lookup(kid, task) = the row or_resolve finds for a launch with that identity and task:
    fresh launches of 3 tasks (some identities absent from the profile, some tasks absent)."""
    import torch

    from paper_2311_10359_b200.pipeline import Pipeline

    tr = F.random_trace(61, 20_000, n_tasks=4, n_ids=300)
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=2048)
    p.run_measure()
    p.check("measure")
    ref_tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=2048)
    # profiled launches under their own task, under another task (0..5: tasks 4, 5 have no
    # profile), and launches of identities nobody profiled
    rng = np.random.default_rng(63)
    fresh = tr.records[rng.integers(0, tr.records.shape[0], size=6000)].copy()
    fresh["task_id"][2000:4000] = rng.integers(0, 6, size=2000)
    other = F.random_trace(62, 2000, n_tasks=4, n_ids=400).records
    other["name_id"] %= tr.names.count
    other["sig_id"] %= tr.sigs.count
    fresh[4000:] = other[:2000]
    kid, st = orc.identify(fresh, tr.names, tr.sigs)
    assert st["code"] == 0
    want, _, _, st = orc.resolve(fresh, tr.names, tr.sigs, ref_tab)
    assert st["code"] == 0
    assert (want == 0xFFFFFFFF).any() and (want != 0xFFFFFFFF).any()
    n = fresh.shape[0]
    out = torch.full((n,), -5, dtype=torch.int32, device="cuda")
    fk.lookup(p.table, _d(kid, np.int64), _d(fresh["task_id"].copy(), np.int32), n, out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    fk.lookup(p.table, None, None, 0, None)  # n = 0: nothing to do, no launch


def test_fill_pool_over_limit_is_e_arg(fk, orc):
    """pool_len 1025 -> FIKIT_E_ARG in the status (include/fikit.h); gaps within the limit are
    still filled exactly"""
    tab_h = hand_table(orc, [200 * US], [0])
    tab = device_table(fk, [200 * US], [0], [1])
    pool_len = np.array([3, 1025, 4], np.uint32)
    pool_off = np.array([0, 3, 1028], np.uint32)
    tot = int(pool_len.sum())
    pool_row = np.zeros(tot, np.uint32)
    pool_dur = np.full(tot, 250 * US, np.uint64)
    pool_level = np.ones(tot, np.uint8)
    R0 = np.array([MS, MS, MS], np.uint64)
    dl = np.full(3, INF, np.uint64)
    poff = pool_off.copy()
    ws, picks, npk, Rl, tu = _fill_gpu(fk, tab, R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len, poff, 0)
    st = fk.get_status(ws)
    assert st["code"] == fk.E_ARG
    rp, rpo, rnp, rRl, rtu, _ = orc.fill_batch(R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len, tab_h,
                                               feedback=0)
    for g in (0, 2):
        assert npk[g] == rnp[g] and Rl[g] == rRl[g] and tu[g] == rtu[g]
        assert np.array_equal(picks[poff[g]:poff[g] + npk[g]], rp[rpo[g]:rpo[g] + rnp[g]])
    assert npk[1] == -7  # left unwritten


def test_simulate_window_over_limit_is_e_arg(fk, orc):
    """lp_len 1025 in one scenario -> FIKIT_E_ARG; the other scenarios match the oracle"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg(S=6, m=1025)
    sc = cfg.replay.scenarios.copy()
    sc["lp_len"][[0, 2, 3, 4, 5]] = [64, 300, 1024, 0, 17]
    rp = F.Replay(cfg.replay.hp_records, cfg.replay.lp_records, cfg.replay.lp_level, sc, cfg.replay.threshold_ns,
                  cfg.replay.feedback)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=rp)
    p.step()
    with pytest.raises(fk.FikitError):
        p.check("window over the limit")
    assert fk.get_status(p.ws)["code"] == fk.E_ARG
    got = p.results()
    ref_tab, _, _ = orc.measure(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024)
    (hr, hd, hg), (lr, ld) = p.resolved()
    sc_ok = sc.copy()
    sc_ok["lp_len"][1] = 0
    ref, _, _, _, st = orc.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level, sc_ok, ref_tab, rp.threshold_ns,
                                          rp.feedback)
    assert st["code"] == 0
    for s in (0, 2, 3, 4, 5):
        assert got[s].tobytes() == ref[s].tobytes(), s


def test_stream_window_over_limit_is_e_arg(fk, orc):
    """STREAM model: m = 1025 in a scenario (two streams) -> FIKIT_E_ARG, not a silent result"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg(S=3, m=1025)
    m_tot = cfg.replay.lp_records.shape[0]
    ids = (np.arange(m_tot) // 600).astype(np.uint32)  # runs of 600: <= 64 streams everywhere
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay,
                 lp_stream=ids)
    p.step()
    st = fk.get_status(p.ws)
    assert st["code"] == fk.E_ARG, st


@pytest.mark.parametrize("feedback", [0, 1])
def test_fill_sorted_pool_beyond_2_32(fk, orc, feedback):
    """Idle times >= 2^32 ns with 33..1024 eligible requests, chunks emptied by earlier picks, and
    predicted durations around the 32-bit boundary (0xFFFFFFFE, 0xFFFFFFFF, 2^32): the sorted
    fast path (q < 2^32 - 1) and the general argmin must both equal the oracle."""
    rng = np.random.default_rng(71)
    specials = [0xFFFFFFFE, 0xFFFFFFFF, 1 << 32, (1 << 32) + 5, 1]
    nrow = 200
    sk = np.concatenate([rng.integers(1, 1 << 31, size=nrow - len(specials)), specials]).astype(np.uint64)
    cnt = np.ones(nrow, np.uint64)
    tab_h = hand_table(orc, sk, [0] * nrow, dur_cnt=cnt)
    tab = device_table(fk, sk, [0] * nrow, cnt)
    G = 300
    pool_len = rng.integers(33, 1025, size=G).astype(np.uint32)
    pool_off = np.zeros(G, np.uint32)
    pool_off[1:] = np.cumsum(pool_len[:-1])
    tot = int(pool_len.sum())
    # half the gaps draw only ordinary rows (fast path), half include the boundary rows
    pool_row = rng.integers(0, nrow - len(specials), size=tot).astype(np.uint32)
    for g in range(0, G, 2):
        o, m = int(pool_off[g]), int(pool_len[g])
        pool_row[o:o + m][rng.random(m) < 0.05] = nrow - len(specials) + rng.integers(0, len(specials))
    pool_dur = rng.integers(1, 1 << 33, size=tot).astype(np.uint64)
    pool_level = rng.integers(1, 4, size=tot).astype(np.uint8)
    R0 = rng.integers(1 << 32, 1 << 40, size=G).astype(np.uint64)
    R0[::7] = (1 << 32) - 1
    R0[1::7] = 1 << 32
    dl = np.where(rng.random(G) < 0.5, rng.integers(1 << 32, 1 << 41, size=G), INF).astype(np.uint64)
    poff = pool_off.copy()
    ws, picks, npk, Rl, tu = _fill_gpu(fk, tab, R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len, poff,
                                       feedback)
    fk.check(ws, "fill beyond 2^32")
    rp, rpo, rnp, rRl, rtu, st = orc.fill_batch(R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len, tab_h,
                                                feedback=feedback)
    assert st["code"] == 0
    assert (rnp > 32).any()  # chunks beyond the first are reached
    assert np.array_equal(npk.view(np.uint32), rnp)
    assert np.array_equal(Rl, rRl) and np.array_equal(tu, rtu)
    for g in range(G):
        assert np.array_equal(picks[poff[g]:poff[g] + npk[g]], rp[rpo[g]:rpo[g] + rnp[g]]), g


def test_replay_huge_gaps_many_requests(fk, orc):
    """Pass 2 (m > 64, shared-memory sorted pool) with predicted gaps >= 2^32 ns: every chunk can
    be emptied by fills inside one gap and BestPrioFit must move past them"""
    import torch

    rng = np.random.default_rng(81)
    n_hp_rows, n_lp_rows = 16, 64
    sg = rng.integers(1 << 32, 1 << 36, size=n_hp_rows).astype(np.uint64)
    sk = rng.integers(1, 1 << 24, size=n_lp_rows).astype(np.uint64)
    dur_mean = np.concatenate([np.ones(n_hp_rows, np.uint64), sk])
    gap_mean = np.concatenate([sg, np.zeros(n_lp_rows, np.uint64)])
    cnt = np.ones(n_hp_rows + n_lp_rows, np.uint64)
    tab_h = hand_table(orc, dur_mean, gap_mean, dur_cnt=cnt)
    tab = device_table(fk, dur_mean, gap_mean, cnt)
    S = 200
    n_h = rng.integers(2, 12, size=S)
    m = rng.integers(65, 1025, size=S)
    hp_off = np.concatenate([[0], np.cumsum(n_h[:-1])])
    lp_off = np.concatenate([[0], np.cumsum(m[:-1])])
    nh_tot, m_tot = int(n_h.sum()), int(m.sum())
    hp_row = rng.integers(0, n_hp_rows, size=nh_tot).astype(np.uint32)
    hp_dur = rng.integers(1, 1 << 30, size=nh_tot).astype(np.uint64)
    hp_gap = rng.integers(0, 1 << 35, size=nh_tot).astype(np.uint64)
    lp_row = (n_hp_rows + rng.integers(0, n_lp_rows, size=m_tot)).astype(np.uint32)
    lp_dur = rng.integers(1, 1 << 25, size=m_tot).astype(np.uint64)
    lp_level = rng.integers(1, 4, size=m_tot).astype(np.uint8)
    sc = np.zeros(S, dtype=F.SCEN_DTYPE)
    sc["hp_off"], sc["hp_len"], sc["lp_off"], sc["lp_len"] = hp_off, n_h, lp_off, m
    sc["gap_scale_q16"] = 1 << 16
    for fb in (0, 1):
        ref, rfg, rls, so, st = orc.simulate_batch(hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, sc, tab_h,
                                                   100 * US, fb, want_schedule=True)
        assert st["code"] == 0
        ws = fk.Workspace(1, 1, 1)
        out = torch.empty(S * 48, dtype=torch.uint8, device="cuda")
        fg = torch.empty(m_tot, dtype=torch.int32, device="cuda")
        ls = torch.empty(m_tot, dtype=torch.int64, device="cuda")
        fk.simulate_batch(tab, _d(hp_row, np.int32), _d(hp_dur, np.int64), _d(hp_gap, np.int64),
                          _d(lp_row, np.int32), _d(lp_dur, np.int64), _d(lp_level, np.uint8),
                          _d(sc.view(np.uint8), np.uint8), S, out, ws, threshold_ns=100 * US, feedback=fb,
                          fill_gap=fg, lp_start=ls, sched_off=_d(so, np.int64))
        fk.check(ws, "replay huge gaps")
        got = out.cpu().numpy().view(ref.dtype)
        assert got.tobytes() == ref.tobytes()
        assert np.array_equal(fg.cpu().numpy(), rfg) and np.array_equal(ls.cpu().numpy().view(np.uint64), rls)
        assert int(ref["n_fills"].max()) > 64


@pytest.mark.parametrize("n_ids,reuse", [(1000, True), (1000, False), (12000, True)])
def test_resolve_parity_table_sizes(fk, orc, n_ids, reuse):
    """fikit_resolve(_ex) against the oracle's or_resolve (Alg. 1 lines 3-5): tables with
    K <= 8192 rows (keys staged in shared memory) and K > 8192 (global binary search), with the
    string hashes reused from the measure call (FIKIT_RESOLVE_REUSE_HASHES) or recomputed."""
    import torch

    from paper_2311_10359_b200.pipeline import Pipeline

    tr = F.random_trace(40 + n_ids, 60000, n_tasks=5, n_ids=n_ids, run_len_max=30, overlap_frac=0.05)
    ref, st, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1 << 16)
    assert st["code"] == 0
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=1 << 16)
    p.run_measure()
    rng = np.random.default_rng(n_ids)
    recs = tr.records[np.sort(rng.choice(tr.records.shape[0], 20000, replace=False))].copy()
    recs["grid_x"][rng.random(20000) < 0.1] += 7  # ~10 % identities without a profile
    d = fk.records_to_device(recs)
    n = recs.shape[0]
    row = torch.empty(n, dtype=torch.int32, device="cuda")
    dur = torch.empty(n, dtype=torch.int64, device="cuda")
    gap = torch.empty(n, dtype=torch.int64, device="cuda")
    fk.resolve(d, n, p.names, p.sigs, p.table, row, dur, gap, p.ws, reuse_hashes=reuse)
    st = fk.check(p.ws, "resolve")
    r_row, r_dur, r_gap, r_st = orc.resolve(recs, tr.names, tr.sigs, ref)
    assert (ref.n_rows > 8192) == (n_ids > 8192)
    assert np.array_equal(row.cpu().numpy().view(np.uint32), r_row)
    assert np.array_equal(dur.cpu().numpy().view(np.uint64), r_dur)
    assert np.array_equal(gap.cpu().numpy().view(np.uint64), r_gap)
    assert st["n_overlap_gaps"] == r_st["n_overlap_gaps"]
    assert 0.5 < (r_row != 0xFFFFFFFF).mean() < 0.99  # most fresh launches have a profile
