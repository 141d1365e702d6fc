"""Pins of the STREAM-model replay oracle (R29-R32):
- singleton streams are the POOL model (oracle.simulate_batch), exactly;
- hand-worked examples of the arrival rules (wait within the predicted idle, the feedback
  deadline, arrivals after the HP job);
- structural invariants on the BERT/VGG stream workload (every request once, stream order and
  think times respected, fills inside the HP job)."""
from types import SimpleNamespace

import numpy as np
import pytest

import fikit_synth as F
import oracle as O


def _tab(dur_mean, dur_cnt, gap_mean):
    return SimpleNamespace(dur_mean=np.asarray(dur_mean, np.uint64), dur_cnt=np.asarray(dur_cnt, np.uint64),
                           gap_mean=np.asarray(gap_mean, np.uint64), n_rows=len(dur_mean))


def _scen(n_h, m, scale=1 << 16):
    sc = np.zeros(1, dtype=F.SCEN_DTYPE)
    sc["hp_len"], sc["lp_len"], sc["gap_scale_q16"] = n_h, m, scale
    return sc


# rows: 0 = the HP kernel (predicted gap 5000), 1 = the LP kernel (predicted duration 1000)
TAB = _tab([1000, 1000], [1, 1], [5000, 0])


def _two_kernel_stream(think, feedback=1):
    # HP: 1000 ns, gap 5000, 1000 ns.  LP: one stream of two 1000-ns kernels, think time `think`
    out, fg, ls, _ = O.simulate_stream_batch(
        hp_row=[0, 0], hp_dur=[1000, 1000], hp_gap=[5000, 0], lp_row=[1, 1], lp_dur=[1000, 1000], lp_level=[1, 1],
        lp_stream=[7, 7], lp_think=[think, 0], scenarios=_scen(2, 2), tab=TAB, threshold=100, feedback=feedback)
    return out[0], fg.tolist(), ls.tolist()


def test_wait_for_an_arrival_inside_the_gap():
    # HP0 ends at 1000, next HP launch r = 6000, R = 5000.  k0 at 1000 (R 4000); k1 arrives at
    # 2000 + 500: waiting 500 consumes predicted idle (R 3500), k1 at 2500 (R 2500).
    o, fg, ls = _two_kernel_stream(500)
    assert fg == [0, 0] and ls == [1000, 2500]
    assert (o["hp_jct"], o["hp_delay"], o["lp_jct"], o["n_fills"], o["n_tail"]) == (7000, 0, 3500, 2, 0)


def test_arrival_at_or_after_the_hp_launch_is_not_awaited():
    # k1 arrives at 2000 + 4500 = 6500 >= r = 6000 (feedback) -> no wait; it runs after HP1
    o, fg, ls = _two_kernel_stream(4500)
    assert fg == [0, -1] and ls == [1000, 7000]
    assert (o["hp_jct"], o["lp_jct"], o["n_fills"], o["n_tail"]) == (7000, 8000, 1, 1)
    # without feedback it is the predicted idle that rules: 6500 - 2000 = 4500 > R = 4000
    o, fg, ls = _two_kernel_stream(4500, feedback=0)
    assert fg == [0, -1] and ls == [1000, 7000]


def test_waiting_consumes_the_predicted_idle():
    # no feedback: k1 arrives at 5500 (5500 - 2000 = 3500 <= R = 4000) -> wait, R = 500 < q(k1)
    o, fg, ls = _two_kernel_stream(3500, feedback=0)
    assert fg == [0, -1] and ls == [1000, 7000] and o["n_fills"] == 1


def test_tail_waits_for_arrivals_in_level_order():
    # no HP gap fits (threshold above every gap): the tail runs the heads in level order, a
    # stream's next kernel only after its think time
    out, fg, ls, _ = O.simulate_stream_batch(
        hp_row=[0], hp_dur=[1000], hp_gap=[0], lp_row=[1, 1, 1], lp_dur=[100, 200, 300], lp_level=[2, 2, 1],
        lp_stream=[1, 1, 2], lp_think=[1000, 0, 0], scenarios=_scen(1, 3), tab=TAB, threshold=10**9, feedback=1)
    # t = 1000: heads k0 (level 2) and k2 (level 1) -> k2 [1000, 1300), k0 [1300, 1400); k1 arrives
    # at 1400 + 1000 = 2400 -> [2400, 2600)
    assert ls.tolist() == [1300, 2400, 1000] and fg.tolist() == [-1, -1, -1]
    assert out[0]["lp_jct"] == 2600 and out[0]["n_tail"] == 3


def _resolved(cfg):
    tr, rp = cfg.trace, cfg.replay
    tab, _, _ = O.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    hr, hd, hg, _ = O.resolve(rp.hp_records, tr.names, tr.sigs, tab)
    lr, ld, lg, _ = O.resolve(rp.lp_records, tr.names, tr.sigs, tab)
    return tab, hr, hd, hg, lr, ld, lg


@pytest.mark.parametrize("feedback", [1, 0])
def test_singleton_streams_are_the_pool_model(feedback):
    cfg = F.bert_vgg(S=600)
    rp = cfg.replay
    tab, hr, hd, hg, lr, ld, lg = _resolved(cfg)
    sc = rp.scenarios.copy()
    sc["gap_scale_q16"] = (1 << 16) << (np.arange(sc.shape[0]) % 5).astype(np.uint32)  # more fills
    pool, pfg, pls, _, _ = O.simulate_batch(hr, hd, hg, lr, ld, rp.lp_level, sc, tab, rp.threshold_ns, feedback,
                                            want_schedule=True)
    out, fg, ls, _ = O.simulate_stream_batch(hr, hd, hg, lr, ld, rp.lp_level, np.arange(lr.shape[0], dtype=np.uint32),
                                             lg, sc, tab, rp.threshold_ns, feedback)
    assert pool["n_fills"].sum() > 0
    assert out.tobytes() == pool.tobytes()
    assert np.array_equal(fg, pfg) and np.array_equal(ls, pls)


def test_stream_workload_invariants():
    cfg, sr = F.bert_vgg_stream(S=400, n_lp_runs=200)
    rp = cfg.replay
    tab, hr, hd, hg, lr, ld, lg = _resolved(cfg)
    out, fg, ls, so = O.simulate_stream_batch(hr, hd, hg, lr, ld, rp.lp_level, sr.lp_stream, lg, rp.scenarios, tab,
                                              rp.threshold_ns, rp.feedback)
    assert out["n_fills"].sum() > 0
    for s, c in enumerate(rp.scenarios):
        m, o, base = int(c["lp_len"]), int(c["lp_off"]), int(so[s])
        starts, gaps = ls[base:base + m].astype(np.int64), fg[base:base + m]
        e, think, sid = ld[o:o + m].astype(np.int64), lg[o:o + m].astype(np.int64), sr.lp_stream[o:o + m]
        assert out[s]["n_fills"] + out[s]["n_tail"] == m
        assert int((gaps >= 0).sum()) == out[s]["n_fills"]
        assert out[s]["lp_jct"] == int((starts + e).max())
        for k in range(m - 1):  # a stream's kernels in order, each after the previous one's think time
            if sid[k + 1] == sid[k]:
                assert starts[k + 1] >= starts[k] + e[k] + think[k]
        fills = gaps >= 0  # fills run inside the HP job
        assert np.all(starts[fills] < int(out[s]["hp_jct"]))


# ---- Case A (§8f row 2; R33-R34): the LP streams hold the GPU until the HP job arrives ----
def _case_a(t_arrive):
    # LP: one stream of three 1000-ns kernels, no think time; HP: one 1000-ns kernel
    out, fg, ls, _ = O.simulate_stream_batch(
        hp_row=[0], hp_dur=[1000], hp_gap=[0], lp_row=[1, 1, 1], lp_dur=[1000, 1000, 1000], lp_level=[1, 1, 1],
        lp_stream=[3, 3, 3], lp_think=[0, 0, 0], scenarios=_scen(1, 3), tab=TAB, threshold=100, feedback=1,
        hp_arrival=[t_arrive])
    return out[0], fg.tolist(), ls.tolist()


def test_case_a_running_kernel_is_not_preempted():
    # HP arrives at 2500 while k2 runs [2000, 3000): the HP kernel starts when k2 ends
    o, fg, ls = _case_a(2500)
    assert ls == [0, 1000, 2000] and fg == [-1, -1, -1]
    assert (o["hp_jct"], o["lp_jct"], o["n_fills"], o["n_tail"]) == (4000, 3000, 0, 0)


def test_case_a_next_launch_is_withheld():
    # HP arrives at 2000, the moment k2 would launch: k2 is withheld and runs after the HP job
    o, fg, ls = _case_a(2000)
    assert ls == [0, 1000, 3000] and fg == [-1, -1, -1]
    assert (o["hp_jct"], o["lp_jct"], o["n_fills"], o["n_tail"]) == (3000, 4000, 0, 1)


def test_case_a_arrival_zero_is_the_stream_model():
    cfg, sr = F.bert_vgg_stream(S=200, n_lp_runs=100)
    rp = cfg.replay
    tab, hr, hd, hg, lr, ld, lg = _resolved(cfg)
    args = (hr, hd, hg, lr, ld, rp.lp_level, sr.lp_stream, lg, rp.scenarios, tab, rp.threshold_ns, rp.feedback)
    a = O.simulate_stream_batch(*args)
    b = O.simulate_stream_batch(*args, hp_arrival=np.zeros(200, np.uint64))
    assert a[0].tobytes() == b[0].tobytes() and np.array_equal(a[2], b[2])
    # and a late arrival: the HP response time never beats running alone, fills still exact
    late = np.full(200, 3_000_000, np.uint64)
    c = O.simulate_stream_batch(*args, hp_arrival=late)
    assert np.all(c[0]["hp_jct"] >= late) and c[0]["n_fills"].sum() > 0
