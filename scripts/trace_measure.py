"""Per-CTA timeline of k_measure (diagnosis build, -DFIKIT_TRACE) on Zipf traces of several sizes.

  python scripts/trace_measure.py build            (here: build/trace/libfikit.so)
  python scripts/trace_measure.py run [N ...]      (on the GPU box)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "build", "trace", "libfikit.so")

if sys.argv[1] == "build":
    from paper_2311_10359_b200 import _build

    print(_build.build(defines=("FIKIT_TRACE",), out=LIB))
    sys.exit(0)

os.environ["FIKIT_DIAG_LIB"] = LIB
import torch  # noqa: E402

import fikit_synth as F  # noqa: E402
import paper_2311_10359_b200 as fk  # noqa: E402
from paper_2311_10359_b200.pipeline import Pipeline  # noqa: E402

L = fk.lib()
L.fikit_debug_trace.argtypes = [C.c_void_p, C.c_int]
for arg in sys.argv[2:] or ["12500000"]:
    wl, N = (arg.split(":") + [None])[:2] if ":" in arg else ("zipf", arg)
    if wl == "resnet":
        cfg = F.resnet_trace()
    else:
        cfg = F.zipf_trace(n_runs=int(N) // 256, threads=16)
    tr = cfg.trace
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=8192 if wl != "resnet" else 4096)
    for _ in range(3):
        p.run_measure()
    torch.cuda.synchronize()
    assert L.fikit_debug_trace(None, 1) == 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    fk.measure(p.recs, p.n, p.names, p.sigs, p.table, p.ws, halo=p.halo)
    ev1.record()
    torch.cuda.synchronize()
    buf = np.zeros(1024 * 16, dtype=np.uint64)
    assert L.fikit_debug_trace(buf.ctypes.data, 0) == 0
    t = buf.reshape(1024, 16).astype(np.int64)
    act = t[:, 2] > 0
    t = t[act]
    t0 = t[:, 0].min()
    us = lambda x: np.round(x / 1000.0, 1)
    st = fk.get_status(p.ws)
    print(f"== {wl} N={tr.records.shape[0]:,}: measure call {ev0.elapsed_time(ev1) * 1e3:.1f} us, {act.sum()} CTAs, "
          f"schedule={st['schedule']} buckets={st['n_task_buckets']}")
    print(f"   entry spread {us(t[:, 0].max() - t0)} us; streaming start: min {us(t[:, 1].min() - t0)} "
          f"med {us(np.median(t[:, 1] - t0))} max {us(t[:, 1].max() - t0)}")
    print(f"   exit: min {us(t[:, 2].min() - t0)} med {us(np.median(t[:, 2] - t0))} max {us(t[:, 2].max() - t0)}")
    print(f"   phases/CTA: mean {t[:, 3].mean():.2f} max {t[:, 3].max()}; tiles/CTA: min {t[:, 4].min()} "
          f"mean {t[:, 4].mean():.0f} max {t[:, 4].max()}")
    print(f"   per CTA (mean us): hot-set loads {us(t[:, 5].mean())}, phase tails {us(t[:, 6].mean())}, "
          f"flush+pick {us(t[:, 7].mean())}; cold batches/CTA {t[:, 8].mean():.1f}")
    order = np.argsort(t[:, 2])
    print("   slowest CTAs (exit us, phases, tiles, load, tail, flush):")
    for i in order[-5:]:
        print(f"     {us(t[i, 2] - t0)} {t[i, 3]} {t[i, 4]} {us(t[i, 5])} {us(t[i, 6])} {us(t[i, 7])}")

    # k_prep / k_plan blocks (g_trace_pre): role, start, end
    L.fikit_debug_trace_pre.argtypes = [C.c_void_p]
    pre = np.zeros(2048 * 8, dtype=np.uint64)
    assert L.fikit_debug_trace_pre(pre.ctypes.data) == 0
    pre = pre.reshape(2048, 8).astype(np.int64)
    pb, qb = pre[:1024], pre[1024:]
    base = min(pb[pb[:, 0] > 0, 0].min(), t0)
    for role, name in ((1, "prep hash"), (2, "prep sample"), (3, "prep groups")):
        r = pb[pb[:, 7] == role]
        if len(r):
            print(f"   {name:12s} blocks {len(r):4d}: start {us(r[:, 0].min() - base)}..{us(r[:, 0].max() - base)}"
                  f" end med {us(np.median(r[:, 1]) - base)} max {us(r[:, 1].max() - base)}")
    for role, name in ((10, "plan hot"), (11, "plan scatter")):
        r = qb[qb[:, 7] == role]
        if len(r):
            msg = (f"   {name:12s} blocks {len(r):4d}: start {us(r[:, 0].min() - base)}..{us(r[:, 0].max() - base)}"
                   f" end med {us(np.median(r[:, 4]) - base)} max {us(r[:, 4].max() - base)}")
            if role == 10:
                msg += (f"; phases (med us) hist+T {us(np.median(r[:, 2] - r[:, 0]))} choose "
                        f"{us(np.median(r[:, 3] - r[:, 2]))} resolve {us(np.median(r[:, 4] - r[:, 3]))}"
                        f" (max {us((r[:, 4] - r[:, 3]).max())})")
            print(msg)
            if role == 10:  # the slowest hot blocks (block 64 = the global set): start, hist+T, choose, resolve
                idx = np.where(qb[:, 7] == role)[0]
                slow = idx[np.argsort(qb[idx, 4])[-4:]]
                print("     slowest hot blocks (block: end, hist+T, choose, resolve us): " + "; ".join(
                    f"{b}: {us(qb[b, 4] - base)}, {us(qb[b, 2] - qb[b, 0])}, {us(qb[b, 3] - qb[b, 2])}, "
                    f"{us(qb[b, 4] - qb[b, 3])}" for b in slow))
    print(f"   k_measure entry at {us(t0 - base)} us after the first k_prep block started")
