"""GPU <-> oracle parity through the C-ABI (bit-exact: all work is integer).

Every test runs the CUDA path (libfikit.so via the thin binding) and the CPU
oracle on the same seeded inputs and compares element by element."""
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


def run_measure(fk, tr, capacity=None, halo=None, want_rows=False):
    from paper_2311_10359_b200.pipeline import Pipeline

    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=capacity, want_rows=want_rows, halo=halo)
    p.run_measure()
    return p


def test_toy_end_to_end(fk, orc):
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.toy()
    for fb in (1, 0):
        cfg.replay.feedback = fb
        ref = orc.pipeline(cfg, capacity=64)
        p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=64, replay=cfg.replay,
                     want_schedule=True, checked=True)
        p.run_measure()
        st = p.check()
        p.run_replay()
        assert st["n_overlap_gaps"] == ref["status"]["n_overlap_gaps"]
        assert_tables_equal(p.table.to_numpy(), ref["table"], "toy")
        (hr, hd, hg), (lr, ld) = p.resolved()
        assert np.array_equal(hr, ref["hp"][0]) and np.array_equal(hd, ref["hp"][1]) and np.array_equal(hg, ref["hp"][2])
        assert np.array_equal(lr, ref["lp"][0]) and np.array_equal(ld, ref["lp"][1])
        assert p.results().tobytes() == ref["results"].tobytes()
        fg, ls = p.schedule()
        assert np.array_equal(fg, ref["fill_gap"]) and np.array_equal(ls, ref["lp_start"])


@pytest.mark.parametrize("seed,n,kw", [
    (1, 1, {}), (2, 31, {}), (3, 32, {}), (4, 33, {}), (5, 255, {}), (6, 256, {}), (7, 257, {}),
    (8, 5000, {"overlap_frac": 0.2}), (9, 5000, {"zero_frac": 0.3}), (10, 5000, {"big_frac": 0.1}),
    (11, 5000, {"run_len_max": 1}), (12, 5000, {"n_ids": 1, "n_tasks": 1}),
    (13, 20000, {"n_ids": 900, "n_tasks": 4, "n_names": 300}),  # > kHotMax rows: cold path
    (14, 70000, {"n_ids": 3000, "n_tasks": 7, "n_names": 800, "overlap_frac": 0.05}),
    # many tasks: more task buckets than CTAs (several phases per CTA, merged tail phase)
    (15, 20000, {"n_ids": 500, "n_tasks": 100, "n_names": 300, "run_len_max": 200}),
    (16, 2000, {"n_ids": 50, "n_tasks": 100, "run_len_max": 64}),
    (17, 300000, {"n_ids": 400, "n_tasks": 40, "n_names": 300, "run_len_max": 400}),
])
def test_measure_random(fk, orc, seed, n, kw):
    tr = F.random_trace(seed, n, **kw)
    ref, rst, rrows = orc.measure(tr.records, tr.names, tr.sigs, want_rows=True)
    p = run_measure(fk, tr, capacity=max(16, 2 * ref.n_rows), want_rows=True)
    st = p.check()
    assert st["n_overlap_gaps"] == rst["n_overlap_gaps"]
    assert st["n_rows_needed"] == ref.n_rows
    assert_tables_equal(p.table.to_numpy(), ref, f"seed {seed}")
    assert np.array_equal(p.rows(), rrows)
    if seed >= 13:  # far more rows than one hot set: the task-partitioned schedule runs
        assert st["schedule"] == 1 and st["n_task_buckets"] > 1, st


@pytest.mark.parametrize("mode", ["wide_task", "wide_name", "mixed"])
def test_measure_wide_ids(fk, orc, mode):
    """Identities with name, sig or task ids >= 2^16 are never kept in the compressed shared
    dictionary (they always take the cold path); parity must hold for them and for traces
    mixing them with compressible ones, in both schedules."""
    tr = F.random_trace(71, 60000, n_ids=700, n_tasks=6, n_names=300, run_len_max=300)
    rec = tr.records.copy()
    names = tr.names
    rng = np.random.default_rng(7)
    if mode in ("wide_task", "mixed"):
        wide = rec["task_id"] % 2 == 1 if mode == "mixed" else np.ones(rec.shape[0], bool)
        rec["task_id"][wide] += np.uint32(1 << 16) + np.uint32(12345)
    if mode in ("wide_name", "mixed"):
        # copies of every name at indices >= 2^16: the same strings, so the same kernel IDs
        base = [names.get(j) for j in range(names.count)]
        pad = [b"pad%d" % j for j in range((1 << 16) - len(base))]
        names = F.StrTab.from_list(base + pad + base)
        move = rng.random(rec.shape[0]) < (1.0 if mode == "wide_name" else 0.3)
        rec["name_id"][move] += np.uint32(1 << 16)
    tr2 = F.Trace(rec, names, tr.sigs)
    ref, rst, _ = orc.measure(tr2.records, tr2.names, tr2.sigs, want_rows=True)
    p = run_measure(fk, tr2, capacity=max(16, 2 * ref.n_rows))
    st = p.check()
    assert st["n_rows_needed"] == ref.n_rows
    assert st["n_overlap_gaps"] == rst["n_overlap_gaps"]
    assert_tables_equal(p.table.to_numpy(), ref, mode)


def test_identify_random(fk, orc):
    import torch

    tr = F.random_trace(21, 10007, n_ids=500, n_names=200)
    ref, _ = orc.identify(tr.records, tr.names, tr.sigs)
    recs = fk.records_to_device(tr.records)
    names, sigs = fk.strtab_to_device(tr.names), fk.strtab_to_device(tr.sigs)
    out = torch.empty(tr.records.shape[0], dtype=torch.int64, device="cuda")
    ws = fk.Workspace(1, tr.names.count, tr.sigs.count)
    fk.identify(recs, tr.records.shape[0], names, sigs, out, ws)
    fk.check(ws)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref)


@pytest.mark.parametrize("field,val", [("grid_x", 0), ("block_z", 0), ("name_id", 10**6), ("sig_id", 10**6),
                                       ("flags", 3), ("end_ns", 0)])
def test_invalid_record_index(fk, orc, field, val):
    tr = F.random_trace(22, 3000)
    rec = tr.records.copy()
    for i in (1777, 2900, 2001):
        rec[field][i] = val
        if field == "end_ns":
            rec["start_ns"][i] = 5
    _, rst, _ = orc.measure(rec, tr.names, tr.sigs)
    assert rst["code"] == orc.E_RECORD and rst["first_bad_index"] == 1777
    bad = F.Trace(rec, tr.names, tr.sigs)
    p = run_measure(fk, bad, capacity=256)
    st = fk.get_status(p.ws)
    assert st["code"] == fk.E_RECORD and st["first_bad_index"] == 1777


def test_capacity_and_empty_name(fk, orc):
    tr = F.random_trace(23, 4000, n_ids=60, n_tasks=3)
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs)
    _, rst, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=10)
    p = run_measure(fk, tr, capacity=10)
    st = fk.get_status(p.ws)
    assert st["code"] == fk.E_CAPACITY == rst["code"] and st["n_rows_needed"] == rst["n_rows_needed"] == ref.n_rows
    names = F.StrTab.from_list([tr.names.get(i) for i in range(tr.names.count)] + [b""])
    p = run_measure(fk, F.Trace(tr.records, names, tr.sigs), capacity=512)
    assert fk.get_status(p.ws)["code"] == fk.E_NAME


def test_halo(fk, orc):
    tr = F.random_trace(24, 3001, run_len_max=80)
    for cut in (1, 1000, 2048, 3000):
        a = F.Trace(tr.records[:cut], tr.names, tr.sigs)
        ref, rst, _ = orc.measure(a.records, a.names, a.sigs, halo=tr.records[cut])
        p = run_measure(fk, a, capacity=512, halo=tr.records[cut])
        st = p.check()
        assert_tables_equal(p.table.to_numpy(), ref, f"halo cut {cut}")
        assert st["n_overlap_gaps"] == rst["n_overlap_gaps"]


def test_resnet_full(fk, orc):
    cfg = F.resnet_trace()
    ref, rst, _ = orc.measure(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=4096)
    p = run_measure(fk, cfg.trace, capacity=4096)
    p.check()
    assert ref.n_rows == 96
    assert_tables_equal(p.table.to_numpy(), ref, "resnet")
    assert p.check()["schedule"] == 0  # 96 rows: one global hot set, address-order sweep


def _replay_parity(fk, orc, cfg, capacity, check_schedule=True):
    from paper_2311_10359_b200.pipeline import Pipeline

    ref = orc.pipeline(cfg, capacity=capacity)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=capacity, replay=cfg.replay,
                 want_schedule=check_schedule, checked=True)
    p.step()
    assert_tables_equal(p.table.to_numpy(), ref["table"], cfg.name)
    (hr, hd, hg), (lr, ld) = p.resolved()
    assert np.array_equal(hr, ref["hp"][0]) and np.array_equal(hg, ref["hp"][2]) and np.array_equal(lr, ref["lp"][0])
    got = p.results()
    if got.tobytes() != ref["results"].tobytes():
        bad = np.flatnonzero(got != ref["results"])[:5]
        raise AssertionError(f"{cfg.name}: scenarios {bad.tolist()} differ: {got[bad]} vs {ref['results'][bad]}")
    if check_schedule:
        fg, ls = p.schedule()
        assert np.array_equal(fg, ref["fill_gap"]) and np.array_equal(ls, ref["lp_start"])
    return ref


def test_random_replay(fk, orc):
    tr = F.random_trace(31, 4000, n_ids=40)
    for seed in range(4):
        rp = F.random_replay(40 + seed, tr, 300, m_max=70, n_h_max=50, levels=9,
                             gap_scale=(1 << 14, 1 << 16, 1 << 19))
        _replay_parity(fk, orc, F.Config("random", tr, rp), 256)


def test_bert_vgg_full(fk, orc):
    cfg = F.bert_vgg()
    ref = _replay_parity(fk, orc, cfg, 1024, check_schedule=True)
    assert ref["results"]["n_fills"].sum() > 0


def test_sweep_sample(fk, orc):
    cfg = F.sweep(S=4000)
    _replay_parity(fk, orc, cfg, 1024, check_schedule=True)


def test_zipf_small_full(fk, orc):
    cfg = F.zipf_trace(n_runs=8000)  # 2.05 M records, all 8,192-row structure, hot + cold paths
    ref, rst, _ = orc.measure(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=8192)
    p = run_measure(fk, cfg.trace, capacity=8192)
    st = p.check()
    assert ref.n_rows > 640  # more rows than the shared-memory hot cache
    assert_tables_equal(p.table.to_numpy(), ref, "zipf-2M")
    assert st["n_overlap_gaps"] == rst["n_overlap_gaps"]
    assert st["schedule"] == 1 and st["n_task_buckets"] == 32, st  # 32 tasks, one bucket each


@pytest.mark.parametrize("G,m_max", [(3000, 80), (400, 1025)])
def test_fill_batch(fk, orc, G, m_max):
    """fikit_fill over G independent gaps; pools up to 1024 requests exercise the sorted pool's
    chunk minima (32 chunks) and the fused bitonic network"""
    import torch

    tr = F.random_trace(51, 3000, n_ids=30)
    ref_tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs)
    from paper_2311_10359_b200.pipeline import Pipeline

    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=128)
    p.run_measure()
    rng = np.random.default_rng(52)
    pool_len = rng.integers(0, m_max, size=G).astype(np.uint32)
    pool_off = np.zeros(G, np.uint32)
    pool_off[1:] = np.cumsum(pool_len[:-1])
    tot = int(pool_len.sum())
    pool_row = rng.integers(0, ref_tab.n_rows + 3, size=tot).astype(np.uint32)  # some absent rows
    pool_dur = rng.integers(1, 3 * F.MS, size=tot).astype(np.uint64)
    pool_level = rng.integers(1, 10, size=tot).astype(np.uint8)
    R0 = rng.integers(0, 10 * F.MS, size=G).astype(np.uint64)
    dl = np.where(rng.random(G) < 0.5, rng.integers(0, 5 * F.MS, size=G), 2**64 - 1).astype(np.uint64)
    for fb in (0, 1):
        picks, poff, npk, Rl, tu, st = orc.fill_batch(R0, dl, pool_row, pool_dur, pool_level, pool_off, pool_len,
                                                      ref_tab, feedback=fb)
        d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
        g_picks = torch.zeros(max(1, tot), dtype=torch.int32, device="cuda")
        g_np = torch.zeros(G, dtype=torch.int32, device="cuda")
        g_R = torch.zeros(G, dtype=torch.int64, device="cuda")
        g_t = torch.zeros(G, dtype=torch.int64, device="cuda")
        fk.fill(p.table, d(R0, np.int64), d(dl, np.int64), d(pool_row, np.int32), d(pool_dur, np.int64),
                d(pool_level, np.uint8), d(pool_off, np.int32), d(pool_len, np.int32), G, g_picks,
                d(poff, np.int32), g_np, g_R, g_t, p.ws, feedback=fb)
        fk.check(p.ws)
        assert np.array_equal(g_np.cpu().numpy().view(np.uint32), npk)
        assert np.array_equal(g_R.cpu().numpy().view(np.uint64), Rl)
        assert np.array_equal(g_t.cpu().numpy().view(np.uint64), tu)
        gp = g_picks.cpu().numpy().view(np.uint32)
        for g in range(G):
            o = int(poff[g])
            assert np.array_equal(gp[o:o + npk[g]], picks[o:o + npk[g]]), g


@pytest.mark.parametrize("P", [2, 3, 8])
def test_sharded_merge_one_gpu(fk, orc, P):
    """Multi-GPU merge kernels on one GPU: P record shards (+ halos) measured
    separately, keys 'all-gathered' by stacking, fikit_dict_union +
    fikit_table_remap + fikit_table_bias, the collectives replaced by torch
    sum / max over the P dense tables, then fikit_table_means: equals the
    unsharded oracle table."""
    import torch

    from paper_2311_10359_b200.dist import shard_range

    cfg = F.zipf_trace(n_runs=3000)  # 768k records, > kHotMax rows
    tr = cfg.trace
    N = tr.records.shape[0]
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=8192)
    cap = 8192
    locs = []
    for r in range(P):
        lo, hi = shard_range(N, r, P)
        sub = F.Trace(tr.records[lo:hi], tr.names, tr.sigs)
        p = run_measure(fk, sub, capacity=cap, halo=tr.records[hi] if hi < N else None)
        p.check()
        locs.append(p)
    n_all = torch.cat([p.table.n_rows_t for p in locs])
    all_kid = torch.stack([p.table.kernel_id for p in locs])
    all_task = torch.stack([p.table.task_id for p in locs])
    denses = []
    for r, p in enumerate(locs):
        ws = fk.Workspace(1, 1, 1, extra=64 * P * cap + (1 << 20))
        d = fk.Table(cap)
        ukid = torch.empty(cap, dtype=torch.int64, device="cuda")
        utask = torch.empty(cap, dtype=torch.int32, device="cuda")
        un = torch.zeros(1, dtype=torch.int32, device="cuda")
        l2u = torch.empty(cap, dtype=torch.int32, device="cuda")
        fk.dict_union(all_kid, all_task, n_all, P, cap, r, ukid, utask, cap, un, l2u, ws)
        fk.check(ws)
        fk.table_remap(p.table, l2u, ukid, utask, un, d)
        fk.table_bias(d)
        denses.append(d)
    out = denses[0]
    out.sums.copy_(torch.stack([d.sums for d in denses]).sum(0))
    out.hist.copy_(torch.stack([d.hist for d in denses]).sum(0))
    out.ext.copy_(torch.stack([d.ext for d in denses]).max(0).values)
    fk.table_bias(out)
    fk.table_means(out)
    assert_tables_equal(out.to_numpy(), ref, f"merge P={P}")


@pytest.mark.parametrize("extra", [1 << 52, 1 << 33, 20_000_000])
def test_replay_huge_durations_slow_path(fk, orc, extra):
    """Requests with large SK leave the fast paths: SK >= 2^50 (or 2^32) ns the exact argmin path,
    SK >= 2^22 ns (here 20 ms) the 32-bit register pool (pass 1 defers to the shared-memory pass 2);
    the replay must agree with the oracle on each."""
    tr = F.random_trace(61, 3000, n_ids=25)
    rec = tr.records.copy()
    big = rec["name_id"] == rec["name_id"][0]
    rec["end_ns"][big] += np.uint64(extra)
    tr2 = F.Trace(rec, tr.names, tr.sigs)
    rp = F.random_replay(62, tr2, 200, m_max=60, n_h_max=40, levels=4)
    _replay_parity(fk, orc, F.Config("huge", tr2, rp), 256)


@pytest.mark.parametrize("mode,pct", [(0, 50), (1, 10), (1, 50), (1, 90), (2, 50)])
def test_table_predict_parity(fk, orc, mode, pct):
    """fikit_table_predict (R26-R28) vs oracle.predict on measured tables: a random trace with
    zero / huge values and overlaps, and the Zipf structure"""
    for tr in (F.random_trace(81, 30000, n_ids=300, n_tasks=4, zero_frac=0.1, big_frac=0.05, overlap_frac=0.05),
               F.zipf_trace(n_runs=2000).trace):
        ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=8192)
        want = orc.predict(ref, mode, pct)
        p = run_measure(fk, tr, capacity=8192)
        fk.table_predict(p.table, mode, pct)
        p.check()
        got = p.table.to_numpy()
        n = ref.n_rows
        assert np.array_equal(got["dur_mean"], want.dur_mean[:n]), (mode, pct)
        assert np.array_equal(got["gap_mean"], want.gap_mean[:n]), (mode, pct)


@pytest.mark.parametrize("predictor", [(1, 90), (2, 50)])
def test_replay_with_predictor(fk, orc, predictor):
    """the whole path with a predictor variant: the replay reads the rewritten predictions"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg()
    ref = orc.pipeline(cfg, capacity=1024, predictor=predictor)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay,
                 want_schedule=True, checked=True, predictor=predictor)
    p.step()
    assert p.results().tobytes() == ref["results"].tobytes()
    fg, ls = p.schedule()
    assert np.array_equal(fg, ref["fill_gap"]) and np.array_equal(ls, ref["lp_start"])
    base = orc.pipeline(cfg, capacity=1024)
    assert ref["results"].tobytes() != base["results"].tobytes()  # the predictor changes the schedule


def test_table_predict_bad_args(fk):
    tr = F.random_trace(82, 500)
    p = run_measure(fk, tr, capacity=64)
    for mode, pct in ((3, 50), (1, 0), (1, 100)):
        with pytest.raises(Exception):
            fk.table_predict(p.table, mode, pct)


def _stream_ref(orc, cfg, sr, feedback):
    tr, rp = cfg.trace, cfg.replay
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    hr, hd, hg, _ = orc.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, lg, _ = orc.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    return orc.simulate_stream_batch(hr, hd, hg, lr, ld, rp.lp_level, sr.lp_stream, lg, rp.scenarios, tab,
                                     rp.threshold_ns, feedback)


@pytest.mark.parametrize("feedback", [1, 0])
def test_stream_replay_parity(fk, orc, feedback):
    """STREAM-model replay (R29-R32): GPU vs oracle, results and schedule, on the BERT/VGG stream
    workload (4 VGG or 2 BERT inference streams per scenario, gap scales 1-8)"""
    from dataclasses import replace

    from paper_2311_10359_b200.pipeline import Pipeline

    cfg, sr = F.bert_vgg_stream(S=3000, n_lp_runs=600)
    cfg = F.Config(cfg.name, cfg.trace, replace(cfg.replay, feedback=feedback))
    out, fg, ls, _ = _stream_ref(orc, cfg, sr, feedback)
    assert out["n_fills"].sum() > 0
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay,
                 want_schedule=True, checked=True, lp_stream=sr.lp_stream)
    p.step()
    got = p.results()
    if got.tobytes() != out.tobytes():
        bad = np.flatnonzero(got != out)[:5]
        raise AssertionError(f"scenarios {bad.tolist()} differ: {got[bad]} vs {out[bad]}")
    gfg, gls = p.schedule()
    assert np.array_equal(gfg, fg) and np.array_equal(gls, ls)


def test_stream_singletons_equal_pool_on_gpu(fk, orc):
    """singleton streams (ids 0..m-1) through the STREAM kernel = the POOL replay (m <= 64)"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg(S=2000)
    ids = np.arange(cfg.replay.lp_records.shape[0], dtype=np.uint32)
    a = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay,
                 want_schedule=True, checked=True, lp_stream=ids)
    b = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay,
                 want_schedule=True, checked=True)
    a.step()
    b.step()
    assert a.results().tobytes() == b.results().tobytes()


def test_stream_limits_flag(fk, orc):
    """more than 64 streams in a scenario is an argument error (status), not a wrong answer"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg(S=4, m=128)
    ids = np.arange(cfg.replay.lp_records.shape[0], dtype=np.uint32)  # 128 singleton streams
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay,
                 lp_stream=ids)
    p.step()
    assert p.check.__self__ is p
    with pytest.raises(Exception):
        p.check("stream limits")


@pytest.mark.parametrize("feedback", [1, 0])
def test_case_a_parity(fk, orc, feedback):
    """Case A preemption (R33-R34): the HP job arrives while the LP streams hold the GPU"""
    from dataclasses import replace

    from paper_2311_10359_b200.pipeline import Pipeline

    cfg, sr = F.bert_vgg_stream(S=2000, n_lp_runs=400)
    cfg = F.Config(cfg.name, cfg.trace, replace(cfg.replay, feedback=feedback))
    arrive = np.random.default_rng(5).integers(0, 5_000_000, size=2000).astype(np.uint64)
    tr, rp = cfg.trace, cfg.replay
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    hr, hd, hg, _ = orc.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, lg, _ = orc.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    out, fg, ls, _ = orc.simulate_stream_batch(hr, hd, hg, lr, ld, rp.lp_level, sr.lp_stream, lg, rp.scenarios, tab,
                                               rp.threshold_ns, feedback, hp_arrival=arrive)
    assert np.all(out["hp_jct"] >= arrive) and out["n_fills"].sum() > 0
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=1024, replay=rp, want_schedule=True, checked=True,
                 lp_stream=sr.lp_stream, hp_arrival=arrive)
    p.step()
    got = p.results()
    if got.tobytes() != out.tobytes():
        bad = np.flatnonzero(got != out)[:5]
        raise AssertionError(f"scenarios {bad.tolist()} differ: {got[bad]} vs {out[bad]}")
    gfg, gls = p.schedule()
    assert np.array_equal(gfg, fg) and np.array_equal(gls, ls)


@pytest.mark.parametrize("feedback", [1, 0])
def test_ratio_sweep_parity(fk, orc, feedback):
    """§4.3.2 ratio sweep: HP windows of 1..50 inferences (up to
    8800 HP kernels per scenario) against one LP inference stream; FIKIT arm and exclusive arm
    (threshold 2^64 - 1) both bit-exact vs the oracle"""
    from dataclasses import replace

    from paper_2311_10359_b200.pipeline import NO_FILL, Pipeline

    cfg, sr, rat = F.ratio_sweep(n_base=24)
    cfg = F.Config(cfg.name, cfg.trace, replace(cfg.replay, feedback=feedback))
    tr, rp = cfg.trace, cfg.replay
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    hr, hd, hg, _ = orc.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, lg, _ = orc.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    args = (hr, hd, hg, lr, ld, rp.lp_level, sr.lp_stream, lg, rp.scenarios, tab)
    out, fg, ls, _ = orc.simulate_stream_batch(*args, rp.threshold_ns, feedback)
    exc, _, _, _ = orc.simulate_stream_batch(*args, NO_FILL, feedback)
    assert out["n_fills"].sum() > 0 and np.all(exc["n_fills"] == 0)
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=1024, replay=rp, want_schedule=True, checked=True,
                 lp_stream=sr.lp_stream, exclusive_arm=True)
    p.step()
    for got, ref in ((p.results(), out), (p.exclusive_results(), exc)):
        if got.tobytes() != ref.tobytes():
            bad = np.flatnonzero(got != ref)[:5]
            raise AssertionError(f"scenarios {bad.tolist()} (ratios {rat[bad].tolist()}) differ: "
                                 f"{got[bad]} vs {ref[bad]}")
    gfg, gls = p.schedule()
    assert np.array_equal(gfg, fg) and np.array_equal(gls, ls)


def test_empty_inputs(fk, orc):
    """degenerate sizes: an empty trace (no rows, status OK), an empty replay batch, and a replay
    against the empty profile (no predictions: every LP request runs in the tail)"""
    from dataclasses import replace

    from paper_2311_10359_b200.pipeline import Pipeline

    tr = F.random_trace(3, 0)
    ref, rst, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=16)
    assert ref.n_rows == 0 and rst["code"] == 0
    p = run_measure(fk, tr, capacity=16)
    st = p.check()
    assert st["code"] == 0 and st["n_rows_needed"] == 0 and p.table.n_rows() == 0
    src = F.random_trace(4, 500, n_ids=12)
    rp = F.random_replay(5, src, 40, m_max=20, n_h_max=12)
    cfg = F.Config("empty-profile", tr, rp)
    out = _replay_parity(fk, orc, cfg, 16)["results"]
    assert np.all(out["n_fills"] == 0) and np.array_equal(out["n_tail"], rp.scenarios["lp_len"])
    none = replace(rp, scenarios=rp.scenarios[:0])
    _replay_parity(fk, orc, F.Config("no-scenarios", src, none), 64, check_schedule=False)


@pytest.mark.parametrize("zero_frac", [0.5, 1.0])
def test_zero_durations_and_zero_threshold(fk, orc, zero_frac):
    """R18: q = 0 requests keep fitting (each dequeued once); tau = 0 opens every gap with p >= 0
    (zero_frac 1.0: every profiled duration and gap is 0)"""
    from dataclasses import replace

    tr = F.random_trace(41, 6000, n_ids=30, zero_frac=zero_frac)
    for fb in (1, 0):
        rp = replace(F.random_replay(42, tr, 400, m_max=80, n_h_max=40, levels=9), threshold_ns=0, feedback=fb)
        ref = _replay_parity(fk, orc, F.Config("zero", tr, rp), 128)
        assert ref["results"]["n_fills"].sum() > 0


def test_sweep_full_size_sampled(fk, orc):
    """configs[4] at its full size (1M scenarios, m = 8..1024, gap scales 1/4..32) as bench.py
    runs it; 1,500 sampled scenarios replayed one by one by the oracle (results and schedule)"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.sweep()
    tr, rp = cfg.trace, cfg.replay
    S = rp.scenarios.shape[0]
    assert S == 1_000_000
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=4096, replay=rp, want_schedule=True)
    p.step()
    p.check("sweep full size")
    got = p.results()
    gfg, gls = p.schedule()
    m = rp.scenarios["lp_len"].astype(np.int64)
    so = np.concatenate([[0], np.cumsum(m[:-1])])
    pick = np.sort(np.random.default_rng(9).choice(S, 1500, replace=False))
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=4096)
    sc = rp.scenarios[pick].copy()
    hp_idx = np.concatenate([np.arange(c["hp_off"], c["hp_off"] + c["hp_len"]) for c in sc])
    lp_idx = np.concatenate([np.arange(c["lp_off"], c["lp_off"] + c["lp_len"]) for c in sc])
    hr, hd, hg, _ = orc.resolve(rp.hp_records[hp_idx], tr.names, tr.sigs, tab)
    lr, ld, _, _ = orc.resolve(rp.lp_records[lp_idx], tr.names, tr.sigs, tab)
    sc["hp_off"] = np.concatenate([[0], np.cumsum(sc["hp_len"][:-1])])
    sc["lp_off"] = np.concatenate([[0], np.cumsum(sc["lp_len"][:-1])])
    out, fg, ls, rso, _ = orc.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level[lp_idx], sc, tab, rp.threshold_ns,
                                             rp.feedback, want_schedule=True)
    assert got[pick].tobytes() == out.tobytes()
    for j, s in enumerate(pick):
        a, b, n = int(so[s]), int(rso[j]), int(m[s])
        assert np.array_equal(gfg[a:a + n], fg[b:b + n]) and np.array_equal(gls[a:a + n], ls[b:b + n]), s


def test_replay_without_schedule_outputs(fk, orc):
    """the launch configuration bench.py times: no fill_gap / lp_start buffers (the kernels'
    no-schedule instantiations), POOL and STREAM replays, results bit-exact vs the oracle"""
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg(S=20000)
    ref = orc.pipeline(cfg, capacity=1024)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay, checked=True)
    p.step()
    assert "fill_gap" not in p.replay and p.results().tobytes() == ref["results"].tobytes()
    cfg, sr = F.bert_vgg_stream(S=3000, n_lp_runs=600)
    out, _, _, _ = _stream_ref(orc, cfg, sr, 1)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=1024, replay=cfg.replay, checked=True,
                 lp_stream=sr.lp_stream)
    p.step()
    assert p.results().tobytes() == out.tobytes()


def test_replay_huge_lp_durations(fk, orc):
    """LP requests whose actual duration is >= 2^32 ns leave the 32-bit register pool (pass 2)"""
    from dataclasses import replace

    tr = F.random_trace(63, 3000, n_ids=25)
    rp = F.random_replay(64, tr, 200, m_max=60, n_h_max=40, levels=4)
    lp = rp.lp_records.copy()
    big = np.random.default_rng(65).random(lp.shape[0]) < 0.05
    lp["end_ns"][big] += np.uint64(1 << 33)
    ref = _replay_parity(fk, orc, F.Config("huge-e", tr, replace(rp, lp_records=lp)), 256)
    assert ref["results"]["n_fills"].sum() > 0


@pytest.mark.parametrize("feedback", [1, 0])
def test_stream_replay_many_streams(fk, orc, feedback):
    """33-64 streams per scenario: heads in both register slots of a lane (sid = 32 + lane), the
    REDUX picks over both, and the lone-stream tail drain reached from many streams"""
    from dataclasses import replace

    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.bert_vgg(S=1500, m=128)
    cfg = F.Config(cfg.name, cfg.trace, replace(cfg.replay, feedback=feedback))
    tr, rp = cfg.trace, cfg.replay
    ids = (np.arange(rp.lp_records.shape[0]) // 3).astype(np.uint32)  # ~43 streams of 3 per window
    tab, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    hr, hd, hg, _ = orc.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, lg, _ = orc.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    out, fg, ls, _ = orc.simulate_stream_batch(hr, hd, hg, lr, ld, rp.lp_level, ids, lg, rp.scenarios, tab,
                                               rp.threshold_ns, feedback)
    assert out["n_fills"].sum() > 0
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=1024, replay=rp, want_schedule=True, checked=True,
                 lp_stream=ids)
    p.step()
    got = p.results()
    if got.tobytes() != out.tobytes():
        bad = np.flatnonzero(got != out)[:5]
        raise AssertionError(f"scenarios {bad.tolist()} differ: {got[bad]} vs {out[bad]}")
    gfg, gls = p.schedule()
    assert np.array_equal(gfg, fg) and np.array_equal(gls, ls)
