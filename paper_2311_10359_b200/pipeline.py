"""Device-resident end-to-end hot path: measure -> finalize -> resolve -> simulate.

Holds the device buffers of one configuration (a trace, optionally a replay
batch) and calls the C-ABI in order.  Marshalling only; the computation is
in libfikit.so.  Input arrays use the 48-byte record layout of
include/fikit.h and the scenario layout fikit_scenario_t.
"""
from __future__ import annotations

import numpy as np

from . import (RESULT_DTYPE, DevStrTab, Table, Workspace, _torch, check, measure, records_to_device, resolve,
               simulate_batch, simulate_stream_batch, strtab_to_device, table_finalize, table_predict)

NO_FILL = (1 << 64) - 1  # a threshold no predicted gap reaches: the exclusive-mode arm


class Pipeline:
    def __init__(self, records: np.ndarray, names, sigs, capacity: int | None = None, replay=None, device="cuda",
                 want_rows: bool = False, want_schedule: bool = False, halo: np.ndarray | None = None,
                 checked: bool = False, predictor: tuple | None = None, lp_stream: np.ndarray | None = None,
                 hp_arrival: np.ndarray | None = None, exclusive_arm: bool = False):
        """checked: verify the workspace status after every call (tests); the
        bench leaves it off and checks once after warm-up.  predictor: (mode, pct) for
        fikit_table_predict before every replay (None: the finalized means, the paper's).
        lp_stream: a stream id per LP request -> the STREAM-model replay (fikit_simulate_stream_batch,
        think times = the LP launches' resolved gaps); None -> the POOL model.  hp_arrival: with lp_stream,
        the HP job's arrival per scenario (Case A preemption).  exclusive_arm: every replay is followed
        by a second one with threshold 2^64 - 1 (no gap is filled: B runs after A, the exclusive-mode
        analogue of P:103 / P:478) into exclusive_results()."""
        torch = _torch()
        self.measured = False  # (set by run_measure: the workspace then holds the string hashes)
        self.checked = checked
        self.predictor = predictor
        self.device = device
        self.n = int(records.shape[0])
        self.capacity = int(capacity if capacity is not None else max(1, min(self.n, 1 << 16)))
        self.recs = records_to_device(records, device) if self.n else torch.zeros(48, dtype=torch.uint8,
                                                                                    device=device)
        self.halo = records_to_device(halo.reshape(1), device) if halo is not None else None
        self.names: DevStrTab = strtab_to_device(names, device)
        self.sigs: DevStrTab = strtab_to_device(sigs, device)
        self.table = Table(self.capacity, device)
        self.ws = Workspace(self.capacity, max(1, names.count), max(1, sigs.count), device, n_records=self.n)
        self.out_row = torch.empty(max(1, self.n), dtype=torch.int32, device=device) if want_rows else None
        self.replay = None
        if replay is not None:
            self._setup_replay(replay, want_schedule)
            if exclusive_arm:
                self.replay["out_excl"] = torch.empty_like(self.replay["out"])
            if lp_stream is not None:
                self.replay["lp_stream"] = torch.from_numpy(np.ascontiguousarray(lp_stream, dtype=np.uint32)
                                                            .view(np.int32)).to(device)
            if hp_arrival is not None:
                self.replay["hp_arrival"] = torch.from_numpy(np.ascontiguousarray(hp_arrival, dtype=np.uint64)
                                                             .view(np.int64)).to(device)

    def _setup_replay(self, rp, want_schedule):
        torch = _torch()
        dev = self.device
        nh, nl = int(rp.hp_records.shape[0]), int(rp.lp_records.shape[0])
        S = int(rp.scenarios.shape[0])
        # HP and LP launches resolved by ONE fikit_resolve call over their concatenation (one launch
        # instead of two) when that is exact: the last HP launch then has a next launch, so its
        # gap must stay 0 -- a different (task, run) than the first LP launch guarantees it (R5)
        both = (nh > 0 and nl > 0 and (int(rp.hp_records["task_id"][-1]) != int(rp.lp_records["task_id"][0])
                                        or int(rp.hp_records["run_id"][-1]) != int(rp.lp_records["run_id"][0])))
        r = {
            "nh": nh, "nl": nl, "S": S, "threshold_ns": int(rp.threshold_ns), "feedback": int(rp.feedback),
            "hp_recs": records_to_device(rp.hp_records, dev) if nh else torch.zeros(48, dtype=torch.uint8,
                                                                                     device=dev),
            "lp_recs": records_to_device(rp.lp_records, dev) if nl else torch.zeros(48, dtype=torch.uint8,
                                                                                     device=dev),
            "lp_level": torch.from_numpy(np.ascontiguousarray(rp.lp_level, dtype=np.uint8)).to(dev)
            if nl else torch.zeros(1, dtype=torch.uint8, device=dev),
            "sc": torch.from_numpy(np.ascontiguousarray(rp.scenarios).view(np.uint8).reshape(-1)).to(dev)
            if S else torch.zeros(24, dtype=torch.uint8, device=dev),
            "hp_row": torch.empty(max(1, nh), dtype=torch.int32, device=dev),
            "hp_dur": torch.empty(max(1, nh), dtype=torch.int64, device=dev),
            "hp_gap": torch.empty(max(1, nh), dtype=torch.int64, device=dev),
            "lp_row": torch.empty(max(1, nl), dtype=torch.int32, device=dev),
            "lp_dur": torch.empty(max(1, nl), dtype=torch.int64, device=dev),
            "lp_gap": torch.empty(max(1, nl), dtype=torch.int64, device=dev),
            "out": torch.empty(max(1, S) * 48, dtype=torch.uint8, device=dev),
        }
        if both:  # one buffer per quantity, the HP / LP arrays are views of it
            recs = records_to_device(np.concatenate([rp.hp_records, rp.lp_records]), dev)
            r["recs_both"] = recs
            r["hp_recs"], r["lp_recs"] = recs[: 48 * nh], recs[48 * nh:]
            for k, dt in (("row", torch.int32), ("dur", torch.int64), ("gap", torch.int64)):
                t = torch.empty(nh + nl, dtype=dt, device=dev)
                r[k + "_both"] = t
                r["hp_" + k], r["lp_" + k] = t[:nh], t[nh:]
        if want_schedule and S:
            m = rp.scenarios["lp_len"].astype(np.uint64)
            so = np.zeros(S, dtype=np.uint64)
            so[1:] = np.cumsum(m[:-1])
            tot = max(1, int(m.sum()))
            r["sched_off"] = torch.from_numpy(so.view(np.int64)).to(dev)
            r["fill_gap"] = torch.empty(tot, dtype=torch.int32, device=dev)
            r["lp_start"] = torch.empty(tot, dtype=torch.int64, device=dev)
        self.replay = r

    # -- a1..a6: identify + measure + finalize --------------------------------------------
    def run_measure(self, stream=None):
        self.measured = True
        measure(self.recs, self.n, self.names, self.sigs, self.table, self.ws, halo=self.halo, out_row=self.out_row,
                stream=stream)
        self._chk("measure", stream)
        table_finalize(self.table, self.ws, out_row=self.out_row, n=self.n if self.out_row is not None else 0,
                       stream=stream)

    # -- a8..a10: resolve the replay's launches, then the batch replay ------------------------
    def run_replay(self, stream=None, table: Table | None = None, sim_events=None):
        """table: the profile to replay against (default: this pipeline's; the merged one for P > 1).
        sim_events: (start, stop) torch.cuda.Event pair recorded around the replay call(s) alone."""
        r = self.replay
        tab = self.table if table is None else table
        if self.predictor is not None:
            table_predict(tab, *self.predictor, stream=stream)
        # (the measure call on this workspace hashed these string tables: no re-hashing)
        if "recs_both" in r:
            resolve(r["recs_both"], r["nh"] + r["nl"], self.names, self.sigs, tab, r["row_both"], r["dur_both"],
                    r["gap_both"], self.ws, stream=stream, reuse_hashes=self.measured)
            self._chk("resolve(hp + lp)", stream)
        else:
            resolve(r["hp_recs"], r["nh"], self.names, self.sigs, tab, r["hp_row"], r["hp_dur"], r["hp_gap"],
                    self.ws, stream=stream, reuse_hashes=self.measured)
            self._chk("resolve(hp)", stream)
            resolve(r["lp_recs"], r["nl"], self.names, self.sigs, tab, r["lp_row"], r["lp_dur"], r["lp_gap"],
                    self.ws, stream=stream, reuse_hashes=True)
            self._chk("resolve(lp)", stream)
        if sim_events is not None:
            sim_events[0].record(stream)
        self._simulate(tab, r["out"], r["threshold_ns"], True, stream)
        if "out_excl" in r:
            self._simulate(tab, r["out_excl"], NO_FILL, False, stream)
        if sim_events is not None:
            sim_events[1].record(stream)

    def _simulate(self, tab, out, threshold_ns, with_schedule, stream):
        r = self.replay
        sched = dict(fill_gap=r.get("fill_gap"), lp_start=r.get("lp_start"), sched_off=r.get("sched_off")) \
            if with_schedule else {}
        if "lp_stream" in r:
            simulate_stream_batch(tab, r["hp_row"], r["hp_dur"], r["hp_gap"], r["lp_row"], r["lp_dur"], r["lp_level"],
                                  r["lp_stream"], r["lp_gap"], r["sc"], r["S"], out, self.ws,
                                  threshold_ns=threshold_ns, feedback=r["feedback"], stream=stream,
                                  hp_arrival=r.get("hp_arrival"), **sched)
        else:
            simulate_batch(tab, r["hp_row"], r["hp_dur"], r["hp_gap"], r["lp_row"], r["lp_dur"], r["lp_level"],
                           r["sc"], r["S"], out, self.ws, threshold_ns=threshold_ns, feedback=r["feedback"],
                           stream=stream, **sched)
        self._chk("simulate_batch", stream)

    def _chk(self, what, stream):
        if self.checked:
            self.last_status = check(self.ws, what, stream)

    def step(self, stream=None):
        self.run_measure(stream)
        if self.replay is not None:
            self.run_replay(stream)

    def check(self, what="pipeline", stream=None):
        return check(self.ws, what, stream)

    # -- host views ------------------------------------------------------------------------------
    def results(self) -> np.ndarray:
        r = self.replay
        return r["out"].cpu().numpy()[: r["S"] * 48].view(RESULT_DTYPE)

    def exclusive_results(self) -> np.ndarray:
        r = self.replay
        return r["out_excl"].cpu().numpy()[: r["S"] * 48].view(RESULT_DTYPE)

    def schedule(self):
        r = self.replay
        return r["fill_gap"].cpu().numpy(), r["lp_start"].cpu().numpy().view(np.uint64)

    def resolved(self):
        r = self.replay
        u = lambda t, n, dt: t.cpu().numpy().view(dt)[:n]
        return ((u(r["hp_row"], r["nh"], np.uint32), u(r["hp_dur"], r["nh"], np.uint64),
                 u(r["hp_gap"], r["nh"], np.uint64)),
                (u(r["lp_row"], r["nl"], np.uint32), u(r["lp_dur"], r["nl"], np.uint64)))

    def rows(self) -> np.ndarray:
        return self.out_row.cpu().numpy().view(np.uint32)[: self.n]
