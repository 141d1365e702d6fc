"""Shared test helpers (fixture parsing, hand-made profiles, small traces).

No method arithmetic lives here: helpers only build inputs and parse the
golden text files; the computations under test are in oracle/ or the CUDA
library.
"""
import os
import shlex

import numpy as np

import fikit_synth as F

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
US, MS = F.US, F.MS


def golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for ln in f:
            ln = ln.strip()
            if ln and not ln.startswith("#"):
                yield ln


def hand_table(orc, dur_mean, gap_mean, dur_cnt=None):
    """A hand-made profile (row r has SK = dur_mean[r], SG = gap_mean[r])."""
    n = len(dur_mean)
    z = lambda dt=np.uint64: np.zeros(max(n, 1), dtype=dt)
    t = orc.Table(n_rows=n, kernel_id=z(), task_id=z(np.uint32), dur_cnt=z(), dur_sum=z(), dur_min=z(),
                  dur_max=z(), gap_cnt=z(), gap_sum=z(), gap_min=z(), gap_max=z(),
                  dur_hist=np.zeros((max(n, 1), 32), np.uint32), gap_hist=np.zeros((max(n, 1), 32), np.uint32),
                  dur_mean=z(), gap_mean=z())
    t.dur_mean[:n] = dur_mean
    t.gap_mean[:n] = gap_mean
    t.dur_cnt[:n] = 1 if dur_cnt is None else dur_cnt
    return t


class Labeled:
    """Build launch records from kernel labels: each distinct label is a
    distinct identity (distinct name), optionally per task."""

    def __init__(self):
        self.names = []
        self.ids = {}

    def name_id(self, label):
        if label not in self.ids:
            self.ids[label] = len(self.names)
            self.names.append(("kern_" + label).encode())
        return self.ids[label]

    def records(self, runs, task=0, run_base=0):
        """runs: list of runs; each run = list of (label, dur_ns, gap_ns or None)."""
        out = []
        t = 0
        for ri, run in enumerate(runs):
            for (label, d, g) in run:
                r = np.zeros(1, dtype=F.REC_DTYPE)
                r["start_ns"] = t
                r["end_ns"] = t + d
                r["name_id"] = self.name_id(label)
                r["grid_x"] = r["grid_y"] = r["grid_z"] = 1
                r["block_x"] = 128
                r["block_y"] = r["block_z"] = 1
                r["run_id"] = run_base + ri
                r["task_id"] = task
                out.append(r)
                t += d + (g if g is not None else F.RUN_PAUSE_NS)
        return np.concatenate(out) if out else np.zeros(0, F.REC_DTYPE)

    def strtabs(self):
        return F.StrTab.from_list(self.names), F.StrTab.from_list([b""])


def parse_kv(tokens):
    return shlex.split(tokens)
