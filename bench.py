#!/usr/bin/env python
"""bench.py -- FIKIT hot path on B200: launch-records/s (identify+measure) and
fill-scenarios/s, with the HBM roofline of the measure kernel.

A step = one pass of the whole hot path over one batch (SURVEY §8a rows
a1-a10): fikit_measure (stream + validate + identify + per-ID statistics) ->
fikit_table_finalize -> [P > 1: dictionary union + NCCL merge] ->
fikit_resolve (HP and LP launches) -> fikit_simulate_batch.

  python bench.py [--gpus N --steps K --warmup W] [--workload zipf|resnet|bert_vgg|sweep]
  python bench.py --impl reference ...   # the CPU oracle, timed on host cores

Default workload (N=1): configs[3], the 100M-launch Zipf trace (4.8 GB, the
largest single-GPU configuration and the one the >= 60 % HBM target is quoted
on) + a 100k-scenario replay batch over its table.  Multi-GPU: records shard
contiguously with a one-record halo (strong scaling: the 100M total is fixed),
scenarios shard s mod N.  Inputs are synthetic (fikit_synth, seeded).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "launch-records/s (identify+measure) and fill-scenarios/s at 1/2/4/8 B200; % HBM peak"
UNIT = "launch-records/s"
REC_BYTES = 48  # algorithmic bytes per launch record
L2_BYTES = 126 << 20  # B200 L2
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fikit", choices=["fikit", "reference"])
    ap.add_argument("--workload", default="zipf",
                    choices=["zipf", "z64k", "resnet", "bert_vgg", "sweep", "stream", "preempt", "ratio", "identify"])
    ap.add_argument("--records", type=int, default=None, help="override the Zipf trace length (runs x 256)")
    ap.add_argument("--scenarios", type=int, default=100_000)
    ap.add_argument("--predictor", default=None,
                    help="mode,pct for fikit_table_predict before each replay (SURVEY §8f row 3; default: the "
                         "paper's means)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-configs2", action="store_true",
                    help="skip the configs[2] (BERT/VGG 100k-scenario replay) leg of the default line")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every timed step's calls directly instead of replaying a CUDA graph of them")
    ap.add_argument("--graph-multi", action="store_true",
                    help="N > 1: replay two CUDA graphs per step around the merge (untested with NCCL: off by "
                         "default; with gloo on one GPU it measured slower)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo + --same-device: test the N>1 path on one GPU)")
    ap.add_argument("--same-device", action="store_true", help="every rank on cuda:0 (testing only)")
    ap.add_argument("--merge", default="dict", choices=["dict", "union"],
                    help="N>1 table merge: 'dict' = every step measures against the dictionary the first "
                         "warm-up step built (fikit_measure_dict; the merge is two all-reduces), 'union' = "
                         "key all-gathers + union + remap + all-reduces every step")
    ap.add_argument("--dict", action="store_true",
                    help="N=1: measure against the dictionary of the first warm-up step (fikit_measure_dict)")
    ap.add_argument("--no-plan-reuse", action="store_true",
                    help="dictionary mode: rebuild the hot sets every step (no FIKIT_MEASURE_REUSE_PLAN)")
    ap.add_argument("--verify-merge", action="store_true",
                    help="N>1: rank 0 re-measures the whole trace on one GPU and checks the merged table bit-exactly")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
def make_workload(args, rank, world):
    """This rank's inputs: (records, halo, names, sigs, replay subset, meta)."""
    import fikit_synth as F
    from paper_2311_10359_b200.dist import scenario_shard, shard_range

    if args.workload in ("zipf", "z64k"):
        # z64k: SURVEY §8d's stress variant of configs[3] (2,048-kernel vocabularies: up to 65,536 rows)
        vocab = 2048 if args.workload == "z64k" else 256
        runs = 390_625 if args.records is None else max(1, args.records // 256)
        N = runs * 256
        lo, hi = shard_range(N, rank, world)
        cfg = F.zipf_trace(n_runs=runs, rec_lo=lo, rec_hi=min(N, hi + 1), threads=min(16, os.cpu_count() or 8),
                           vocab_per_task=vocab)
        recs = cfg.trace.records
        halo = recs[hi - lo] if hi < N else None
        recs = recs[: hi - lo]
        replay = F.zipf_replay(cfg, S=args.scenarios)
        cap = 32 * vocab
        desc = (f"zipf-{N / 1e6:g}M (configs[3]" + (", Z64k stress: 2048-kernel vocabularies" if vocab > 256 else "")
                + f") + replay-{args.scenarios / 1000:g}k")
    elif args.workload in ("stream", "preempt"):  # LP kernel streams (+ Case A)
        cfg, sr = F.bert_vgg_stream(S=args.scenarios)
        N = cfg.trace.records.shape[0]
        lo, hi = shard_range(N, rank, world)
        recs = cfg.trace.records[lo:hi]
        halo = cfg.trace.records[hi] if hi < N else None
        replay = cfg.replay
        lp_stream = sr.lp_stream
        hp_arrival = None
        cap = 4096
        desc = f"bert_vgg_stream-{args.scenarios // 1000}k (STREAM-model replay, §8f row 1)"
        if args.workload == "preempt":  # the HP job arrives U[0, 5 ms) into the LP streams' run
            hp_arrival = np.random.default_rng(5).integers(0, 5_000_000, size=args.scenarios).astype(np.uint64)
            desc = f"bert_vgg_preempt-{args.scenarios // 1000}k (Case A preemption, §8f row 2)"
    elif args.workload == "ratio":  # the §4.3.2 A:B task-ratio sweep, FIKIT + exclusive arms
        cfg, sr, ratio = F.ratio_sweep(n_base=max(1, args.scenarios // (2 * len(F.RATIO_SCALES_Q16) * len(F.RATIOS))))
        N = cfg.trace.records.shape[0]
        lo, hi = shard_range(N, rank, world)
        recs = cfg.trace.records[lo:hi]
        halo = cfg.trace.records[hi] if hi < N else None
        replay = cfg.replay
        lp_stream = sr.lp_stream
        hp_arrival = None
        cap = 4096
        desc = (f"ratio_sweep-{replay.scenarios.shape[0] // 1000}k (§4.3.2 A:B = 1..50:1, BERT/VGG stream pairs, "
                f"HP gaps x1/x4/x16; FIKIT arm + exclusive arm)")
    else:
        cfg = {"resnet": F.resnet_trace, "bert_vgg": F.bert_vgg, "sweep": F.sweep}[args.workload]()
        N = cfg.trace.records.shape[0]
        lo, hi = shard_range(N, rank, world)
        recs = cfg.trace.records[lo:hi]
        halo = cfg.trace.records[hi] if hi < N else None
        replay = cfg.replay
        cap = 4096
        desc = {"resnet": "resnet-3M (configs[1])", "bert_vgg": "bert_vgg-100k (configs[2])",
                "sweep": "sweep-1M (configs[4])"}[args.workload]
    ratio = ratio if args.workload == "ratio" else None
    lp_stream = lp_stream if args.workload in ("stream", "preempt", "ratio") else None
    if replay is not None and world > 1:
        sel = scenario_shard(replay.scenarios.shape[0], rank, world)
        if ratio is not None:
            ratio = ratio[sel]
        replay = F.Replay(replay.hp_records, replay.lp_records, replay.lp_level, replay.scenarios[sel],
                          replay.threshold_ns, replay.feedback)
        replay, lp_stream = compact_replay(replay, lp_stream)  # this rank's launches only
        if args.workload == "preempt":
            hp_arrival = hp_arrival[sel]
    return dict(records=recs, halo=halo, names=cfg.trace.names, sigs=cfg.trace.sigs, replay=replay, N=N, cap=cap,
                desc=desc, cfg=cfg, lp_stream=lp_stream,
                hp_arrival=hp_arrival if args.workload == "preempt" else None, ratio=ratio)


def compact_replay(rp, lp_stream=None):
    """Keep only the HP / LP launches this rank's scenarios reference (every window whole, in
    order) and remap the scenarios' offsets: a rank resolves and stages its share of the
    launches, not all of them (host-side data placement, outside the timed region)."""
    import fikit_synth as F

    sc = rp.scenarios.copy()

    def keep(n, off, ln):
        mark = np.zeros(n + 1, np.int64)
        np.add.at(mark, off, 1)
        np.add.at(mark, off + ln, -1)
        need = np.cumsum(mark[:n]) > 0
        return need, np.cumsum(need) - 1

    off_h, len_h = sc["hp_off"].astype(np.int64), sc["hp_len"].astype(np.int64)
    off_l, len_l = sc["lp_off"].astype(np.int64), sc["lp_len"].astype(np.int64)
    need_h, map_h = keep(rp.hp_records.shape[0], off_h, len_h)
    need_l, map_l = keep(rp.lp_records.shape[0], off_l, len_l)
    sc["hp_off"] = np.where(len_h > 0, map_h[np.minimum(off_h, max(0, need_h.shape[0] - 1))], 0)
    sc["lp_off"] = np.where(len_l > 0, map_l[np.minimum(off_l, max(0, need_l.shape[0] - 1))], 0)
    out = F.Replay(rp.hp_records[need_h], rp.lp_records[need_l], rp.lp_level[need_l], sc, rp.threshold_ns,
                   rp.feedback)
    return out, (lp_stream[need_l] if lp_stream is not None else None)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50", "-i",
                 str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per fikit_measure launch from the committed ncu --set full capture, if present."""
    p = os.path.join(ROOT, "profiles", "measure_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_record"), d.get("source")
    except Exception:
        return None, None


# ---------------------------------------------------------------------------------------------
def cpu_info():
    """Host CPU model and the threads this process may use (the baseline's core count)."""
    import oracle.sharded as OS

    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": OS.host_threads(), "cpu_count": os.cpu_count()}


def oracle_pass(wl, frac, threads):
    """The CPU oracle (as it stands) over a leading fraction of the workload: the first frac*N
    records are measured, then the first frac*S scenarios are resolved (only the launches they
    reference) and replayed against that table.  threads > 1: the all-core sharded driver
    (oracle/sharded.py: record shards + halo merged by or_table_merge, scenario slices); 1: the
    single-threaded oracle.  Returns (seconds, records, scenarios)."""
    import oracle
    import oracle.sharded as OS
    import fikit_synth as F

    oracle.build()
    recs, names, sigs = wl["records"], wl["names"], wl["sigs"]
    N = recs.shape[0]
    n1 = max(1, min(N, int(round(frac * N))))
    rp = wl["replay"]
    prep = None
    if rp is not None:  # host-side data placement (outside the timed part): the scenarios' launches only
        S = rp.scenarios.shape[0]
        s_n = max(1, min(S, int(round(frac * S))))
        sel = F.Replay(rp.hp_records, rp.lp_records, rp.lp_level, rp.scenarios[:s_n].copy(), rp.threshold_ns,
                       rp.feedback)
        lp_stream = wl["lp_stream"]
        sub, sub_stream = compact_replay(sel, lp_stream)
        prep = (sub, sub_stream, s_n)
    t = time.perf_counter()
    tab, st = OS.measure(recs[:n1], names, sigs, capacity=max(65536, wl["cap"]), threads=threads)
    if st["code"] != 0:
        raise RuntimeError(f"oracle measure: {st}")
    s_n = 0
    if prep is not None:
        sub, sub_stream, s_n = prep
        hr, hd, hg = OS.resolve(sub.hp_records, names, sigs, tab, threads=threads)
        lr, ld, lg = OS.resolve(sub.lp_records, names, sigs, tab, threads=threads)
        if sub_stream is not None:  # STREAM model (think times: the resolved LP gaps)
            ha = wl["hp_arrival"][:s_n] if wl.get("hp_arrival") is not None else None
            OS.simulate_stream_batch(hr, hd, hg, lr, ld, sub.lp_level, sub_stream, lg, sub.scenarios, tab,
                                     sub.threshold_ns, sub.feedback, hp_arrival=ha, threads=threads)
            if wl.get("ratio") is not None:  # the exclusive arm (no gap filled)
                OS.simulate_stream_batch(hr, hd, hg, lr, ld, sub.lp_level, sub_stream, lg, sub.scenarios, tab,
                                         (1 << 64) - 1, sub.feedback, threads=threads)
        else:
            OS.simulate_batch(hr, hd, hg, lr, ld, sub.lp_level, sub.scenarios, tab, sub.threshold_ns, sub.feedback,
                              threads=threads)
    return time.perf_counter() - t, n1, s_n


def calibrate_frac(wl, threads, seconds):
    """The workload fraction the oracle finishes in about `seconds` with `threads` threads."""
    N = wl["records"].shape[0]
    f0 = min(1.0, max(1.0 / N, 2e5 * threads / N))
    t0, _, _ = oracle_pass(wl, f0, threads)
    return min(1.0, f0 * seconds / max(1e-3, t0))


def cpu_baseline(wl, budget_s):
    """SURVEY §8d oracle timing: (ii) all host threads (the sharded driver) -- a full,
    non-extrapolated pass when it fits the budget, else the largest leading fraction that does;
    (i) one thread on a bounded leading fraction, extrapolated.  The baseline value is (ii)."""
    import oracle.sharded as OS

    info = cpu_info()
    T = OS.host_threads()
    N = wl["N"]
    f_all = calibrate_frac(wl, T, budget_s * 0.6)
    t_all, n_all, s_all = oracle_pass(wl, f_all, T)
    f_one = calibrate_frac(wl, 1, budget_s * 0.25)
    t_one, n_one, s_one = oracle_pass(wl, f_one, 1)
    S = wl["replay"].scenarios.shape[0] if wl["replay"] is not None else 0
    full = n_all == wl["records"].shape[0] and s_all == S
    desc = (f"oracle, {T} threads (oracle/sharded.py): "
            + ("the FULL workload, not extrapolated" if full else f"the first {n_all:,} records + {s_all:,} "
               f"scenarios (a {n_all / N:.3f} fraction)") + f" in {t_all:.2f} s")
    return {"value": n_all / t_all, "unit": UNIT, "cores": T, "kind": "oracle", "sample": desc,
            "full_pass": bool(full), "seconds": t_all, **info,
            "single_core": {"value": n_one / t_one, "unit": UNIT, "cores": 1,
                            "sample": f"the first {n_one:,} records + {s_one:,} scenarios in {t_one:.2f} s "
                                      f"(value = records / time of that leading fraction)"}}


def ratio_summary(fik, exc, ratio, sc):
    """Per (pair, HP gap scale) series: the mean over scenarios of exclusive / FIKIT LP JCT and
    the mean HP slowdown (hp_delay / solo) per A:B ratio (reporting only, host side)."""
    import fikit_synth as F

    out = {}
    pair = np.where(sc["hp_len"] // ratio == 176, "A=BERT,B=VGG", "A=VGG,B=BERT")
    for pr in ("A=BERT,B=VGG", "A=VGG,B=BERT"):
        for q in F.RATIO_SCALES_Q16:
            key = f"{pr},gaps_x{q >> 16}"
            ser = {}
            for r in F.RATIOS:
                sel = (pair == pr) & (sc["gap_scale_q16"] == q) & (ratio == r)
                if not sel.any():
                    continue
                solo = (fik["hp_jct"][sel] - fik["hp_delay"][sel]).astype(np.float64)
                ser[f"{r}:1"] = {"lp_excl_over_fikit": round(float(np.mean(exc["lp_jct"][sel] / fik["lp_jct"][sel])), 3),
                                 "hp_slowdown": round(float(np.mean(fik["hp_delay"][sel] / solo)), 4),
                                 "lp_in_gaps": round(float(np.mean(fik["n_tail"][sel] == 0)), 3)}
            out[key] = ser
    return out


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) on every host thread (the
    sharded driver), rank 0 only.  A step = one oracle pass over a leading fraction of the same
    workload (records and scenarios in the workload's proportion), sized so the whole
    --steps/--warmup run takes about 2.5 minutes; value = records per step / step time, the same
    definition as the fikit arm's (records / time of a step that measures and replays)."""
    import oracle.sharded as OS

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = make_workload(args, 0, 1)
    T = OS.host_threads()
    per_step = max(0.3, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    frac = calibrate_frac(wl, T, per_step)
    times, n1, s1 = [], 0, 0
    for i in range(args.warmup + args.steps):
        t, n1, s1 = oracle_pass(wl, frac, T)
        if i >= args.warmup:
            times.append(t)
    step_s = float(np.mean(times))
    value = n1 / step_s
    desc = (f"oracle on {T} threads (oracle/sharded.py); each step: the first {n1:,} of {wl['N']:,} records + "
            f"{s1:,} scenarios")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic (fikit_synth, seeded)",
            "config": {"workload": wl["desc"], "records": wl["N"], "records_per_step": n1, "scenarios_per_step": s1},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "oracle", "sample": desc,
                             **cpu_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def replay_roofline(workload, scenarios, sim_ms, sm_mhz):
    """Issue roofline of the replay kernels: achieved warp-instructions/s (ncu's per-scenario count,
    profiles/replay_inst.json, x the scenarios of a step / the replay call's live time) against
    the SM issue peak (SMs x 4 schedulers x one warp-instruction per cycle at the measured clock)."""
    import torch

    rec = None
    try:
        with open(os.path.join(ROOT, "profiles", "replay_inst.json")) as f:
            rec = json.load(f).get(workload)
    except Exception:
        pass
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    out = {"bound": "issue", "kernel": "fikit_simulate_batch (k_simulate_reg + k_simulate)", "call_ms": sim_ms,
           "scenarios": scenarios, "scenarios_per_s": scenarios / (sim_ms * 1e-3)}
    if rec and sm_mhz:
        ach = rec["warp_inst_per_scenario"] * scenarios / (sim_ms * 1e-3) / 1e9
        peak = sms * 4 * sm_mhz * 1e6 / 1e9
        out.update({"achieved": ach, "peak": peak, "unit": "G warp-instructions/s", "frac": ach / peak,
                    "warp_inst_per_scenario": rec["warp_inst_per_scenario"], "inst_source": rec.get("source"),
                    "peak_source": f"{sms} SMs x 4 issue slots x {sm_mhz:.0f} MHz (measured under load)"})
    return out


def configs2_leg(fk, Pipeline, stream, args, steps=20, warmup=3):
    """BASELINE configs[2] in the default line: the BERT/VGG trace (216k launches) measured and its
    100k scenarios (one warp each) replayed, timed per step with L2 flushed before each step."""
    import torch

    import fikit_synth as F

    cfg = F.bert_vgg()
    q = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=4096, replay=cfg.replay)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    for _ in range(warmup):
        q.step()
    q.check("configs2 warm-up")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        q.run_measure()
        q.run_replay(sim_events=(ev[i][1], ev[i][2]))
        ev[i][3].record(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([e[0].elapsed_time(e[3]) for e in ev]))
    sim = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    S = cfg.replay.scenarios.shape[0]
    return {"workload": "bert_vgg-100k (configs[2]): 216k-launch measurement + 100k scenarios, m = 64",
            "scenarios_per_s": S / (ms * 1e-3), "ms_per_step": ms, "replay_call_ms": sim,
            "replay_scenarios_per_s": S / (sim * 1e-3), "steps": steps, "warmup": warmup,
            "l2": "inputs fit the L2: a 256 MB write flushes it before every step (outside the step's events)"}


def run_identify(args):
    """--workload identify: fikit_identify alone over the 100M-launch Zipf trace (configs[3]),
    SURVEY §8d "identify-only: 56 B/record" (48 B read + an 8-B kernel ID written per launch).
    1 GPU; the roofline is the whole call (string hashing + k_identify) against the copy peak."""
    import torch

    import fikit_synth as F
    from paper_2311_10359_b200 import _build

    _build.build()
    import paper_2311_10359_b200 as fk

    runs = 390_625 if args.records is None else max(1, args.records // 256)
    cfg = F.zipf_trace(n_runs=runs, threads=min(16, os.cpu_count() or 8))
    tr = cfg.trace
    N = tr.records.shape[0]
    recs = fk.records_to_device(tr.records)
    names, sigs = fk.strtab_to_device(tr.names), fk.strtab_to_device(tr.sigs)
    out = torch.empty(N, dtype=torch.int64, device="cuda")
    ws = fk.Workspace(1, names.count, sigs.count)
    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        fk.identify(recs, N, names, sigs, out, ws)
        if i == 0:
            fk.check(ws, "identify warm-up")
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = fk.launch_count()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(args.steps):
            fk.identify(recs, N, names, sigs, out, ws)
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    peak, peak_src = peaks()
    ach = 56 * N / (ms * 1e-3) / 1e9
    line = {"metric": "launch-records/s (identify only)", "value": N / (ms * 1e-3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic (fikit_synth, seeded)",
            "config": {"workload": f"identify over zipf-{N / 1e6:g}M (configs[3] trace)", "records": N,
                       "l2": "inputs (4.8 GB) larger than the L2: steps back to back, no flush"},
            "roofline": {"bound": "hbm", "kernel": "fikit_identify (k_strtab_hash + k_identify)", "achieved": ach,
                         "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": 56, "traffic": None},
            "gpu_launches": int(fk.launch_count() - launches0), "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "identify":
        return run_identify(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev_index = 0 if args.same_device else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")

    from paper_2311_10359_b200 import _build

    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()
    import paper_2311_10359_b200 as fk
    from paper_2311_10359_b200.dist import LibOps, merge_tables, merge_tables_dict
    from paper_2311_10359_b200.pipeline import Pipeline

    t_gen = time.perf_counter()
    wl = make_workload(args, rank, world)
    t_gen = time.perf_counter() - t_gen
    stream = torch.cuda.current_stream()
    pred = tuple(int(x) for x in args.predictor.split(",")) if args.predictor else None
    p = Pipeline(wl["records"], wl["names"], wl["sigs"], capacity=wl["cap"], replay=wl["replay"], halo=wl["halo"],
                 predictor=pred, lp_stream=wl["lp_stream"], hp_arrival=wl["hp_arrival"],
                 exclusive_arm=wl["ratio"] is not None)
    n_local = p.n
    dense = fk.Table(wl["cap"]) if world > 1 else None
    ops = LibOps(fk.Workspace(1, 1, 1, extra=64 * world * wl["cap"] + (1 << 20))) if world > 1 else None
    S_local = p.replay["S"] if p.replay else 0
    ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(5)]  # (stage events)
    for e in ev:
        e.record(stream)
    stage_ms = np.zeros(4)

    # k_measure alone, live in every timed step: one event pair per step (fikit_measure_timed)
    # (external: inside a captured step graph they are event-record nodes that time every replay)
    kev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
           for _ in range(args.steps)]
    for a, b in kev:  # (torch creates the CUDA events on first record)
        a.record(stream)
        b.record(stream)
    # the replay call alone (fikit_simulate_batch: its two kernels), live in every timed step
    rev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
           for _ in range(args.steps)]
    for a, b in rev:
        a.record(stream)
        b.record(stream)

    # dictionary mode (repeated services keep their kernel IDs): the first
    # warm-up step measures and merges with the general path; its (merged) table's keys become the
    # dictionary every later step measures against (fikit_measure_dict), so the N>1 merge is the
    # two all-reduces alone
    use_dict = (world > 1 and args.merge == "dict") or (world == 1 and args.dict)
    dict_state = None
    plan_ready = [False]  # the workspace holds a dictionary call's plan (FIKIT_MEASURE_REUSE_PLAN)

    # a step = part A (measure + finalize), the N > 1 merge (collectives), part B (resolve + replay)
    def part_a(kpair=None, checked=False, timed=False):
        if timed:
            ev[0].record()  # (current stream: the capture stream inside a graph)
        fk.measure(p.recs, p.n, p.names, p.sigs, p.table, p.ws, halo=p.halo, events=kpair, dictionary=dict_state,
                   reuse_plan=dict_state is not None and plan_ready[0])
        if dict_state is not None:
            plan_ready[0] = not args.no_plan_reuse  # (the next dictionary step reuses this one's plan)
        p.measured = True  # (the workspace holds the string hashes: resolve reuses them)
        st = fk.check(p.ws, "bench warm-up: measure") if checked else None
        if timed:
            ev[1].record()
        fk.table_finalize(p.table, p.ws)
        return st

    def part_b(tab, spair=None, checked=False):
        if p.replay:
            p.checked = checked
            p.run_replay(table=tab, sim_events=spair)  # (checked: after each resolve and replay call)
            p.checked = False

    def step(timed, kpair=None, checked=False, spair=None):
        # checked (first warm-up step): the workspace status after EVERY call (each validating
        # call resets it, so one check at the end would only see the last call)
        st = part_a(kpair, checked, timed)
        tab = p.table
        if world > 1 and dict_state is not None:
            merge_tables_dict(p.table, ops)
            if checked:
                fk.check(ops.ws, "bench warm-up: merge")
        elif world > 1:
            merge_tables(p.table, dense, ops)
            if checked:
                fk.check(ops.ws, "bench warm-up: merge")
            tab = dense
        if timed:
            ev[2].record()
        part_b(tab, spair, checked)
        if timed:
            ev[3].record()
        return st

    def step_merge():  # the N > 1 merge of a graph-replayed step (direct collectives)
        if dict_state is not None:
            merge_tables_dict(p.table, ops)
        else:
            merge_tables(p.table, dense, ops)

    st = None
    for i in range(args.warmup):
        s_i = step(False, checked=(i <= 1))
        st = s_i if s_i is not None else st
        if i == 0 and use_dict:
            src = dense if world > 1 else p.table
            K = src.n_rows()
            dict_state = (src.kernel_id[:K].clone(), src.task_id[:K].clone(), K)
            dense = None if world > 1 else dense
    torch.cuda.synchronize()
    # per-stage breakdown on separately timed steps (events between the calls), launched the way the
    # timed steps are: a CUDA graph of the step with the stage events as external event nodes (1 GPU),
    # else direct launches
    n_stage = min(20, args.steps)
    stage_graph = None
    if world == 1 and not args.no_graph:
        stage_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(stage_graph):
            step(True)
        stage_graph.replay()
        torch.cuda.synchronize()
    for _ in range(n_stage):
        if stage_graph is not None:
            stage_graph.replay()
        else:
            step(True)
        torch.cuda.synchronize()
        stage_ms += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), 0]
    stage_ms /= n_stage

    # ---- timed region: K steps, barrier + sync on both sides.  Inputs larger than 2x the L2
    # (the Zipf trace: 4.8 GB) stream from HBM anyway: the K steps run back to back between two
    # events.  Smaller inputs (BERT/VGG: 10 MB) would stay L2-resident, so L2 is flushed before
    # every step (a 256 MB write, outside the step's own event pair) and the step time is the sum
    # of the per-step event pairs. ----
    in_bytes = p.recs.numel() + (sum(p.replay[k].numel() * p.replay[k].element_size()
                                     for k in ("hp_recs", "lp_recs", "lp_level", "sc")) if p.replay else 0)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda") if in_bytes < 2 * L2_BYTES else None
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)] \
        if flush is not None else None
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # Every timed 1-GPU step replays a CUDA graph captured from the same calls (one per step: each
    # holds its own k_measure / replay event pairs).  N > 1 with --graph-multi: part A (measure +
    # finalize) and part B (resolve + replay) are two graphs and the merge's torch.distributed
    # collectives run between them, outside any graph; by default N > 1 launches directly.  The
    # library's launch counter counts at capture, so the step's launches are counted there.
    graphs = None
    launches_per_graph = 0
    merged_tab = dense if (world > 1 and dict_state is None) else p.table  # (the table part B replays against)
    if not args.no_graph and (world == 1 or args.graph_multi):
        graphs = []
        for i in range(args.steps):
            l0 = fk.launch_count()
            ga = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ga):
                if world == 1:
                    step(False, kev[i], spair=rev[i] if p.replay else None)
                else:
                    part_a(kev[i])
            gb = None
            if world > 1 and p.replay:
                gb = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gb):
                    part_b(merged_tab, rev[i])
            launches_per_graph = fk.launch_count() - l0
            graphs.append((ga, gb))
        for ga, gb in graphs[:2]:  # (first replays upload the graphs)
            ga.replay()
            if world > 1:
                step_merge()
            if gb is not None:
                gb.replay()
        torch.cuda.synchronize()
    launches0 = fk.launch_count()
    with ClockSampler(dev_index) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
                sev[i][0].record(stream)
            if graphs is not None:
                graphs[i][0].replay()
                if world > 1:
                    step_merge()
                if graphs[i][1] is not None:
                    graphs[i][1].replay()
            else:
                step(False, kev[i], spair=rev[i] if p.replay else None)
            if flush is not None:
                sev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = (sum(a.elapsed_time(b) for a, b in sev) if flush is not None else t0.elapsed_time(t1)) / args.steps
    l2_note = (f"inputs ({in_bytes / 1e6:.0f} MB) larger than 2x the 126 MB L2: steps back to back, no flush"
               if flush is None else f"inputs ({in_bytes / 1e6:.1f} MB) fit the L2: a {L2_FLUSH_BYTES >> 20} MB "
               f"write flushes L2 before every step (outside the step's event pair)")
    launches = fk.launch_count() - launches0 + (launches_per_graph * args.steps if graphs is not None else 0)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    N = wl["N"]
    S_total = wl["replay"].scenarios.shape[0] * (world if world > 1 else 1) if wl["replay"] is not None else 0
    if wl["replay"] is not None and world > 1:
        S_total = int(torch.tensor([S_local], device="cuda").sum().item())
        t = torch.tensor([S_local], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        S_total = int(t.item())
    value = N / (ms * 1e-3)

    # ---- roofline of the dominant kernel (k_measure: 48 algorithmic bytes per launch), its
    # average launch duration from the event pairs of the timed region ----
    peak, peak_src = peaks()
    kmeas_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    meas_ms = stage_ms[0]
    achieved = REC_BYTES * n_local / (kmeas_ms * 1e-3) / 1e9
    trf, trf_src = ncu_traffic()
    roof = {"bound": "hbm", "kernel": "k_measure (the fused identify + measure streaming kernel)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": REC_BYTES * n_local,
            "traffic": (trf * n_local if trf is not None else None), "traffic_source": trf_src,
            "kernel_ms": kmeas_ms, "kernel_ms_source": "CUDA events around k_measure in every timed step",
            "measure_call_ms": meas_ms,
            "measure_call_frac": REC_BYTES * n_local / (meas_ms * 1e-3) / 1e9 / peak}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (fikit_synth, seeded)",
            "config": {"workload": wl["desc"] + (f" predictor={args.predictor}" if args.predictor else ""),
                       "records": N, "records_per_gpu": n_local, "scenarios": S_total,
                       "table_rows": (dense if dense is not None else p.table).n_rows(),
                       "merge": ("dictionary (fikit_measure_dict against the first warm-up step's merged keys; "
                                 "merge = 2 all-reduces" + ("; plan reused" if plan_ready[0] else "") + ")"
                                 if dict_state is not None else
                                 "union (key all-gathers + union + remap + 2 all-reduces)") if world > 1 else
                                ("dictionary (fikit_measure_dict against the first warm-up step's keys"
                                 + ("; plan reused" if plan_ready[0] else "") + ")"
                                 if dict_state is not None else "none (1 GPU)"),
                       "l2": l2_note,
                       "launch": ((f"CUDA graph per step ({launches_per_graph} libfikit kernels, captured after warm-up)"
                                   if world == 1 else
                                   f"two CUDA graphs per step (measure + finalize; resolve + replay: {launches_per_graph} "
                                   f"libfikit kernels, captured after warm-up) around the merge's collectives")
                                  if graphs is not None else "direct launches"),
                       "parallelism": f"dp{world} (record shards + halo, NCCL table merge)" if world > 1 else "1 GPU"},
            "scenarios_per_s": (S_total / (ms * 1e-3)) if S_total else None,
            "stages_ms": {"measure": stage_ms[0], "finalize+merge": stage_ms[1], "resolve+replay": stage_ms[2]},
            "measure_records_per_s": n_local / (stage_ms[0] * 1e-3),
            "roofline": roof, "gpu_launches": int(launches), "clocks": clk.summary(),
            "status": {"code": st["code"], "n_rows_needed": st["n_rows_needed"]},
            "gen_s": round(t_gen, 2)}

    if p.replay:  # the replay kernels: issue-bound, warp-instructions per scenario from ncu
        sim_ms = float(np.mean([a.elapsed_time(b) for a, b in rev]))
        line["replay_roofline"] = replay_roofline(args.workload, S_local, sim_ms, line["clocks"].get("sm_mhz"))
    if rank == 0 and world == 1 and args.workload == "zipf" and not args.no_configs2:
        line["configs2_bert_vgg"] = configs2_leg(fk, Pipeline, stream, args)

    if wl["ratio"] is not None:  # §4.3.2 trend: mean exclusive / FIKIT LP JCT per A:B ratio and series
        line["ratio_sweep"] = ratio_summary(p.results(), p.exclusive_results(), wl["ratio"], wl["replay"].scenarios)

    # ---- end to end through the C-ABI with host buffers (H2D + step + D2H inside the region) ----
    if not args.no_e2e:
        pin = torch.from_numpy(np.ascontiguousarray(wl["records"]).view(np.uint8).reshape(-1)).pin_memory()
        host_out = torch.empty(p.table.block.numel(), dtype=torch.uint8).pin_memory()
        rep_out = torch.empty(p.replay["out"].numel(), dtype=torch.uint8).pin_memory() if p.replay else None
        h2d = pin.numel()
        d2h = host_out.numel() + (rep_out.numel() if rep_out is not None else 0)
        if p.replay:
            rp_pins = [p.replay[k].cpu().pin_memory() for k in ("hp_recs", "lp_recs", "lp_level", "sc")]
            h2d += sum(x.numel() * x.element_size() for x in rp_pins)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            p.recs.copy_(pin, non_blocking=True)
            if p.replay:
                for k, x in zip(("hp_recs", "lp_recs", "lp_level", "sc"), rp_pins):
                    p.replay[k].copy_(x, non_blocking=True)
            step(False)
            host_out.copy_((dense if dense is not None else p.table).block, non_blocking=True)
            if rep_out is not None:
                rep_out.copy_(p.replay["out"], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / args.e2e_steps
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        line["e2e"] = {"value": N / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms, "steps": args.e2e_steps,
                       "path": "pinned host -> device copies + fikit_* C-ABI calls + result copies back"}

    # ---- N>1: the merged table must equal a 1-GPU measure of the whole trace ----
    if world > 1 and args.verify_merge and rank == 0:
        full = make_workload(args, 0, 1)
        q = Pipeline(full["records"], full["names"], full["sigs"], capacity=wl["cap"])
        q.run_measure()
        q.check("verify-merge")
        a, b = (dense if dense is not None else p.table).to_numpy(), q.table.to_numpy()
        same = all(np.array_equal(a[k], b[k]) for k in a)
        line["verify_merge"] = {"equal_to_1gpu": bool(same), "rows": int(a["kernel_id"].shape[0])}
        if not same:
            print("verify-merge: MISMATCH", file=sys.stderr)
    # ---- CPU baseline: the oracle on the host cores, rank 0, N=1 only ----
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, args.cpu_budget_s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
