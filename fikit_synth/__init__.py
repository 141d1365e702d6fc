"""Seeded synthetic inputs for the FIKIT hot path (shared by the oracle side and the CUDA side).

This module holds NONE of the method's arithmetic: it never hashes a kernel
identity, never groups, never averages and never schedules.  It only draws
seeded random numbers and lays them out in the byte formats the two sides
consume:

* launch records (48 B, little-endian; the same field order both sides
  declare independently — DESIGN.md "Data layout"),
* string tables (interned kernel names and argument-type signatures),
* replay inputs: high-priority (HP) template runs, low-priority (LP) request
  populations with their priority levels, and scenario descriptors.

The shapes follow PAPER.md's workloads as restated in SURVEY.md §8(d):
kernels of "typically 0.1 ms to 2 ms", "large" inter-kernel gaps
(P:27), runs of N_t kernels repeated T times,
ResNet/BERT/VGG-like kernel counts (Table 1).  The distributions
themselves are assumptions (the paper publishes none); DESIGN.md "Input
recipe" lists them.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# byte layouts (input formats)
# ---------------------------------------------------------------------------
REC_DTYPE = np.dtype(
    [
        ("start_ns", "<u8"),
        ("end_ns", "<u8"),
        ("name_id", "<u4"),
        ("sig_id", "<u4"),
        ("grid_x", "<u4"),
        ("grid_y", "<u2"),
        ("grid_z", "<u2"),
        ("block_x", "<u2"),
        ("block_y", "<u2"),
        ("block_z", "<u2"),
        ("flags", "<u2"),
        ("run_id", "<u4"),
        ("task_id", "<u4"),
    ]
)
assert REC_DTYPE.itemsize == 48

SCEN_DTYPE = np.dtype(
    [
        ("hp_off", "<u4"),
        ("hp_len", "<u4"),
        ("lp_off", "<u4"),
        ("lp_len", "<u4"),
        ("gap_scale_q16", "<u4"),
        ("pad", "<u4"),
    ]
)
assert SCEN_DTYPE.itemsize == 24

US = 1000  # ns per microsecond
MS = 1000 * US
RUN_PAUSE_NS = 1 * MS  # pause between runs (not a gap: run_id changes)


@dataclass
class StrTab:
    """count strings; string j = data[offsets[j]:offsets[j+1]]."""

    data: np.ndarray  # uint8
    offsets: np.ndarray  # uint32, count+1

    @property
    def count(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @staticmethod
    def from_list(strings: list[bytes]) -> "StrTab":
        offs = np.zeros(len(strings) + 1, dtype=np.uint32)
        offs[1:] = np.cumsum([len(s) for s in strings], dtype=np.uint64).astype(np.uint32)
        data = np.frombuffer(b"".join(strings) or b"\0", dtype=np.uint8).copy()
        return StrTab(data=data, offsets=offs)

    def get(self, j: int) -> bytes:
        return self.data[int(self.offsets[j]) : int(self.offsets[j + 1])].tobytes()


@dataclass
class Trace:
    records: np.ndarray  # REC_DTYPE
    names: StrTab
    sigs: StrTab


@dataclass
class Replay:
    """Inputs of a batch replay.  HP/LP kernels are given as launch records
    (their identity is resolved against the measured table by the method)."""

    hp_records: np.ndarray  # REC_DTYPE, HP template runs back to back
    lp_records: np.ndarray  # REC_DTYPE, LP requests (start 0, end = e)
    lp_level: np.ndarray  # uint8 in [1, 9], one per LP request
    scenarios: np.ndarray  # SCEN_DTYPE
    threshold_ns: int = 100 * US  # P:330 "smaller than 0.1ms"
    feedback: int = 1


@dataclass
class Config:
    name: str
    trace: Trace
    replay: Replay | None = None
    meta: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# vocabulary: distinct kernel identities (name, signature, grid, block)
# ---------------------------------------------------------------------------
_ALPHA = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz0123456789_", dtype=np.uint8)
_SIG_TYPES = [b"float const*", b"float*", b"int", b"long", b"c10::Half const*", b"c10::BFloat16*",
              b"at::native::ReduceOp<float>", b"unsigned int", b"double", b"bool", b"void*", b"int const*"]


def _mangled_names(rng: np.random.Generator, n: int, lo: int = 60, hi: int = 250) -> list[bytes]:
    out = []
    seen = set()
    while len(out) < n:
        L = int(rng.integers(lo, hi + 1))
        body = _ALPHA[rng.integers(0, len(_ALPHA), size=max(L - 14, L))].tobytes()
        s = (b"_ZN2at6native" + bytes([48 + len(out) % 10]) + body) if L >= 16 else body
        if s not in seen:
            seen.add(s)
            out.append(s[:L])
    return out


def _signatures(rng: np.random.Generator, n: int) -> list[bytes]:
    out = [b""]  # entry 0 = empty signature (the paper's ID, reading C1)
    seen = {b""}
    while len(out) < n:
        k = int(rng.integers(1, 7))
        s = b"(" + b", ".join(_SIG_TYPES[i] for i in rng.integers(0, len(_SIG_TYPES), size=k)) + b")"
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


@dataclass
class Vocab:
    name_id: np.ndarray
    sig_id: np.ndarray
    grid: np.ndarray  # (K, 3)
    block: np.ndarray  # (K, 3)

    def __len__(self):
        return int(self.name_id.shape[0])


def _vocab(rng: np.random.Generator, K: int, n_names: int, n_sigs: int, name_base: int = 0,
           sig_base: int = 0) -> Vocab:
    """K distinct (name, sig, grid, block) tuples drawn over n_names names."""
    seen = set()
    rows = []
    while len(rows) < K:
        nm = name_base + int(rng.integers(0, n_names))
        sg = sig_base + int(rng.integers(0, n_sigs))
        gx = int(rng.choice([1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 65536]))
        gy = int(rng.choice([1, 1, 1, 2, 3, 4, 8]))
        gz = int(rng.choice([1, 1, 1, 1, 2]))
        bx = int(rng.choice([32, 64, 128, 256, 512, 1024]))
        by = int(rng.choice([1, 1, 1, 2, 4]))
        bz = 1
        key = (nm, sg, gx, gy, gz, bx, by, bz)
        if key in seen:
            continue
        seen.add(key)
        rows.append(key)
    a = np.array(rows, dtype=np.int64)
    return Vocab(name_id=a[:, 0].astype(np.uint32), sig_id=a[:, 1].astype(np.uint32),
                 grid=a[:, 2:5].astype(np.uint32), block=a[:, 5:8].astype(np.uint32))


def _fill_identity(rec: np.ndarray, vocab: Vocab, kidx: np.ndarray) -> None:
    rec["name_id"] = vocab.name_id[kidx]
    rec["sig_id"] = vocab.sig_id[kidx]
    rec["grid_x"] = vocab.grid[kidx, 0]
    rec["grid_y"] = vocab.grid[kidx, 1]
    rec["grid_z"] = vocab.grid[kidx, 2]
    rec["block_x"] = vocab.block[kidx, 0]
    rec["block_y"] = vocab.block[kidx, 1]
    rec["block_z"] = vocab.block[kidx, 2]
    rec["flags"] = 0


def _timestamps(rec: np.ndarray, dur: np.ndarray, gap: np.ndarray, run_len: int, t0: int = 0) -> int:
    """Lay runs of `run_len` kernels back to back: start_{i+1} = end_i + gap_i
    inside a run, RUN_PAUSE_NS between runs.  gap[i] of a run's last kernel is
    ignored.  Returns the end time of the last run."""
    n = dur.shape[0]
    step = dur.astype(np.uint64) + gap.astype(np.uint64)
    last = (np.arange(n) % run_len) == run_len - 1
    step[last] = dur[last].astype(np.uint64) + RUN_PAUSE_NS
    ends_excl = np.cumsum(step, dtype=np.uint64)
    start = np.empty(n, dtype=np.uint64)
    start[0] = 0
    start[1:] = ends_excl[:-1]
    start += np.uint64(t0)
    rec["start_ns"] = start
    rec["end_ns"] = start + dur.astype(np.uint64)
    return int(start[-1] + np.uint64(dur[-1])) + RUN_PAUSE_NS if n else t0


def _loguniform(rng, lo, hi, size):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size=size))


def _gap_mixture(rng, size, p_small=0.9, med_small=12 * US, sig_small=0.6, med_large=250 * US, sig_large=0.8):
    small = rng.random(size) < p_small
    g = np.where(small, rng.lognormal(np.log(med_small), sig_small, size),
                 rng.lognormal(np.log(med_large), sig_large, size))
    return g


# ---------------------------------------------------------------------------
# a "model": a kernel template walked once per inference run
# ---------------------------------------------------------------------------
@dataclass
class Model:
    vocab: Vocab
    template: np.ndarray  # vocabulary index per position
    base_dur: np.ndarray  # ns per vocabulary entry
    base_gap: np.ndarray  # ns per template position
    dur_jitter: float
    gap_jitter: float
    task_id: int

    def runs(self, rng, n_runs: int, run_base: int, t0: int = 0) -> tuple[np.ndarray, int]:
        L = self.template.shape[0]
        n = n_runs * L
        rec = np.zeros(n, dtype=REC_DTYPE)
        kidx = np.tile(self.template, n_runs)
        _fill_identity(rec, self.vocab, kidx)
        dur = self.base_dur[kidx] * rng.uniform(1 - self.dur_jitter, 1 + self.dur_jitter, n)
        gap = np.tile(self.base_gap, n_runs) * rng.uniform(1 - self.gap_jitter, 1 + self.gap_jitter, n)
        dur = np.maximum(np.rint(dur), 1).astype(np.uint64)
        gap = np.clip(np.rint(gap), 1 * US, 20 * MS).astype(np.uint64)
        tend = _timestamps(rec, dur, gap, L, t0)
        rec["run_id"] = run_base + np.repeat(np.arange(n_runs, dtype=np.uint32), L)
        rec["task_id"] = self.task_id
        return rec, tend

    def requests(self, rng, n_req: int, task_id: int | None = None) -> np.ndarray:
        """LP kernel requests: uniform over template positions, jittered
        execution time e; each request is its own 1-kernel 'run'."""
        pos = rng.integers(0, self.template.shape[0], size=n_req)
        kidx = self.template[pos]
        rec = np.zeros(n_req, dtype=REC_DTYPE)
        _fill_identity(rec, self.vocab, kidx)
        e = self.base_dur[kidx] * rng.uniform(1 - self.dur_jitter, 1 + self.dur_jitter, n_req)
        rec["start_ns"] = 0
        rec["end_ns"] = np.maximum(np.rint(e), 1).astype(np.uint64)
        rec["run_id"] = np.arange(n_req, dtype=np.uint32)
        rec["task_id"] = self.task_id if task_id is None else task_id
        return rec


def _template_from_walk(rng, K: int, L: int) -> np.ndarray:
    """A template of length L that uses every one of the K ids at least once."""
    t = np.concatenate([np.arange(K), rng.integers(0, K, size=L - K)])
    # keep a model-like structure: repeated blocks are contiguous-ish
    return t[np.argsort(rng.random(L) + np.arange(L) / L * 4.0, kind="stable")].astype(np.int64)


def resnet50_model(rng, names_n: int, sigs_n: int, task_id: int, name_base=0, sig_base=0) -> Model:
    """~300 kernels/inference over 96 distinct IDs: stem; 3-4-6-3 bottlenecks
    (conv->2 kernels, bn, relu, add); avgpool; fc."""
    vocab = _vocab(rng, 96, names_n, sigs_n, name_base, sig_base)
    seq = []
    nxt = iter(range(96))
    ids = {}

    def kid(tag):
        if tag not in ids:
            ids[tag] = next(nxt, None)
            if ids[tag] is None:
                ids[tag] = int(rng.integers(0, 96))
        return ids[tag]

    seq += [kid("stem_conv_a"), kid("stem_conv_b"), kid("stem_bn"), kid("stem_relu"), kid("maxpool")]
    for stage, nblk in enumerate([3, 4, 6, 3]):
        for b in range(nblk):
            for c in range(3):
                ctag = f"s{stage}c{c}" + ("first" if b == 0 else "")
                seq += [kid(ctag + "a"), kid(ctag + "b"), kid(f"s{stage}bn{c}")]
                if c < 2:
                    seq += [kid(f"s{stage}relu{c}")]
            if b == 0:
                seq += [kid(f"s{stage}down_a"), kid(f"s{stage}down_b"), kid(f"s{stage}down_bn")]
            seq += [kid(f"s{stage}add"), kid(f"s{stage}relu_out")]
    seq += [kid("avgpool"), kid("fc_gemm"), kid("fc_bias")]
    seq = np.array(seq, dtype=np.int64)
    used = np.unique(seq)
    # use all 96 ids: pad the walk with the unused ones (aux kernels: copies, casts)
    unused = np.setdiff1d(np.arange(96), used)
    ins = np.sort(rng.integers(0, len(seq), size=len(unused)))
    seq = np.insert(seq, ins, unused)
    if seq.shape[0] < 300:
        extra = rng.integers(0, 96, size=300 - seq.shape[0])
        seq = np.insert(seq, np.sort(rng.integers(0, len(seq), size=len(extra))), extra)
    seq = seq[:300]
    base_dur = _loguniform(rng, 5 * US, 400 * US, 96)
    base_gap = _gap_mixture(rng, 300, 0.9)
    return Model(vocab, seq, base_dur, base_gap, 0.05, 0.2, task_id)


def bert_model(rng, names_n, sigs_n, task_id, name_base=0, sig_base=0) -> Model:
    vocab = _vocab(rng, 22, names_n, sigs_n, name_base, sig_base)
    t = _template_from_walk(rng, 22, 176)
    return Model(vocab, t, _loguniform(rng, 8 * US, 300 * US, 22), _gap_mixture(rng, 176, 0.85), 0.05, 0.2,
                 task_id)


def vgg_model(rng, names_n, sigs_n, task_id, name_base=0, sig_base=0) -> Model:
    vocab = _vocab(rng, 30, names_n, sigs_n, name_base, sig_base)
    t = _template_from_walk(rng, 30, 40)
    return Model(vocab, t, _loguniform(rng, 50 * US, 2 * MS, 30), _gap_mixture(rng, 40, 0.95), 0.05, 0.2,
                 task_id)


# ---------------------------------------------------------------------------
# configs (BASELINE.json configs[0..4])
# ---------------------------------------------------------------------------
def toy(seed: int = 1) -> Config:
    """configs[0]: HP task 0 = 20-kernel template over 8 IDs, LP task 1 =
    50-kernel template over 12 IDs, T = 10 runs each (200 + 500 records);
    replay: one scenario, HP = a fresh 11th run, LP pool = the 50 kernels of
    one fresh LP run at level 1."""
    rng = np.random.default_rng(seed)
    names = _mangled_names(rng, 16)
    sigs = _signatures(rng, 6)
    hp_v = _vocab(rng, 8, 8, 6)
    lp_v = _vocab(rng, 12, 8, 6, name_base=8)
    hp_t = _template_from_walk(rng, 8, 20)
    lp_t = _template_from_walk(rng, 12, 50)
    hp_gap = np.where(rng.random(20) < 0.6, rng.uniform(5 * US, 80 * US, 20), rng.uniform(150 * US, 3 * MS, 20))
    hp = Model(hp_v, hp_t, rng.uniform(50 * US, 1.5 * MS, 8), hp_gap, 0.05, 0.05, 0)
    lp = Model(lp_v, lp_t, rng.uniform(100 * US, 2 * MS, 12), rng.uniform(5 * US, 200 * US, 50), 0.05, 0.05, 1)
    r_hp, t1 = hp.runs(rng, 10, 0)
    r_lp, _ = lp.runs(rng, 10, 0, t0=t1)
    trace = Trace(np.concatenate([r_hp, r_lp]), StrTab.from_list(names), StrTab.from_list(sigs))
    hp_fresh, _ = hp.runs(rng, 1, 10)
    lp_run, _ = lp.runs(rng, 1, 10)
    # the fresh LP run's kernels become 50 independent requests (reading C21)
    lp_fresh = lp_run.copy()
    lp_fresh["end_ns"] = lp_run["end_ns"] - lp_run["start_ns"]
    lp_fresh["start_ns"] = 0
    lp_fresh["run_id"] = np.arange(50, dtype=np.uint32)
    sc = np.zeros(1, dtype=SCEN_DTYPE)
    sc[0] = (0, 20, 0, 50, 1 << 16, 0)
    rep = Replay(hp_fresh, lp_fresh, np.ones(50, dtype=np.uint8), sc)
    return Config("toy", trace, rep, {"seed": seed})


def resnet_trace(seed: int = 2, n_runs: int = 10_000) -> Config:
    """configs[1]: ResNet-50-like inference trace, 300 kernels/inference over
    96 distinct IDs, 10,000 runs -> 3,000,000 records (144 MB), task 0."""
    rng = np.random.default_rng(seed)
    names = _mangled_names(rng, 40)
    sigs = _signatures(rng, 24)
    m = resnet50_model(rng, 40, 24, 0)
    rec, _ = m.runs(rng, n_runs, 0)
    return Config("resnet", Trace(rec, StrTab.from_list(names), StrTab.from_list(sigs)), None,
                  {"seed": seed, "runs": n_runs})


def bert_vgg(seed: int = 3, T: int = 1000, n_hp_runs: int = 1000, pop: int = 1 << 20, S: int = 100_000,
             m: int = 64) -> Config:
    """configs[2]: BERT-base-like (176 kernels, 22 IDs) + VGG-16-like (40
    kernels, 30 IDs), T runs each for measurement; HP templates = fresh runs;
    LP populations of `pop` requests per model, level U{1,2,3}; S scenarios,
    half (HP BERT, LP VGG) and half (HP VGG, LP BERT), m LP requests each."""
    rng = np.random.default_rng(seed)
    names = _mangled_names(rng, 48)
    sigs = _signatures(rng, 16)
    bert = bert_model(rng, 24, 16, 0)
    vgg = vgg_model(rng, 24, 16, 1, name_base=24)
    rb, t1 = bert.runs(rng, T, 0)
    rv, _ = vgg.runs(rng, T, 0, t0=t1)
    trace = Trace(np.concatenate([rb, rv]), StrTab.from_list(names), StrTab.from_list(sigs))
    hb, _ = bert.runs(rng, n_hp_runs, T)
    hv, _ = vgg.runs(rng, n_hp_runs, T)
    hp = np.concatenate([hb, hv])
    lb = bert.requests(rng, pop)
    lv = vgg.requests(rng, pop)
    lp = np.concatenate([lv, lb])  # [0,pop) = VGG population, [pop,2pop) = BERT population
    lvl = rng.integers(1, 4, size=2 * pop).astype(np.uint8)
    s = np.arange(S, dtype=np.int64)
    half = S // 2
    sc = np.zeros(S, dtype=SCEN_DTYPE)
    hp_bert = s < half
    run = s % n_hp_runs
    sc["hp_off"] = np.where(hp_bert, run * 176, n_hp_runs * 176 + run * 40)
    sc["hp_len"] = np.where(hp_bert, 176, 40)
    win = (s * m) % (pop - m + 1)
    sc["lp_off"] = np.where(hp_bert, win, pop + win)
    sc["lp_len"] = m
    sc["gap_scale_q16"] = 1 << 16
    return Config("bert_vgg", trace, Replay(hp, lp, lvl, sc), {"seed": seed, "S": S, "m": m})


@dataclass
class StreamReplay:
    """STREAM-model replay inputs: as Replay, plus per LP request its stream
    id (a stream = a maximal run of equal consecutive ids in a scenario's window).  The think
    time after each LP kernel is its trace gap, resolved like the HP gaps."""

    replay: Replay
    lp_stream: np.ndarray  # uint32, one per LP request


def bert_vgg_stream(seed: int = 3, T: int = 1000, n_hp_runs: int = 1000, n_lp_runs: int = 4000, S: int = 100_000,
                    vgg_streams: int = 4, bert_streams: int = 2) -> tuple[Config, StreamReplay]:
    """The BERT/VGG pair of configs[2] (same models and measurement trace) as kernel streams:
    half the scenarios run an HP BERT inference against `vgg_streams` VGG inferences (40-kernel
    streams), half HP VGG against `bert_streams` BERT inferences (176-kernel streams).  The LP
    inferences are fresh runs with their own gaps (think times); every stream has one level
    U{1,2,3}; HP gaps are replayed at scales 1, 2, 4, 8 (s mod 4)."""
    rng = np.random.default_rng(seed)
    names = _mangled_names(rng, 48)
    sigs = _signatures(rng, 16)
    bert = bert_model(rng, 24, 16, 0)
    vgg = vgg_model(rng, 24, 16, 1, name_base=24)
    rb, t1 = bert.runs(rng, T, 0)
    rv, _ = vgg.runs(rng, T, 0, t0=t1)
    trace = Trace(np.concatenate([rb, rv]), StrTab.from_list(names), StrTab.from_list(sigs))
    hb, _ = bert.runs(rng, n_hp_runs, T)
    hv, _ = vgg.runs(rng, n_hp_runs, T)
    hp = np.concatenate([hb, hv])
    lv, _ = vgg.runs(rng, n_lp_runs, T + n_hp_runs)  # [0, 40 n) VGG streams
    lb, _ = bert.runs(rng, n_lp_runs, T + n_hp_runs)  # then BERT streams
    lp = np.concatenate([lv, lb])
    run_lvl = rng.integers(1, 4, size=2 * n_lp_runs).astype(np.uint8)
    lvl = np.concatenate([np.repeat(run_lvl[:n_lp_runs], 40), np.repeat(run_lvl[n_lp_runs:], 176)])
    stream = np.concatenate([np.repeat(np.arange(n_lp_runs, dtype=np.uint32), 40),
                             np.repeat(np.arange(n_lp_runs, 2 * n_lp_runs, dtype=np.uint32), 176)])
    s = np.arange(S, dtype=np.int64)
    half = S // 2
    sc = np.zeros(S, dtype=SCEN_DTYPE)
    hp_bert = s < half
    run = s % n_hp_runs
    sc["hp_off"] = np.where(hp_bert, run * 176, n_hp_runs * 176 + run * 40)
    sc["hp_len"] = np.where(hp_bert, 176, 40)
    w_v = (s % (n_lp_runs - vgg_streams + 1)) * 40
    w_b = 40 * n_lp_runs + (s % (n_lp_runs - bert_streams + 1)) * 176
    sc["lp_off"] = np.where(hp_bert, w_v, w_b)
    sc["lp_len"] = np.where(hp_bert, 40 * vgg_streams, 176 * bert_streams)
    sc["gap_scale_q16"] = (1 << 16) << (s % 4)  # HP gaps x1, 2, 4, 8 (R24)
    rp = Replay(hp, lp, lvl, sc)
    cfg = Config("bert_vgg_stream", trace, rp, {"seed": seed, "S": S})
    return cfg, StreamReplay(rp, stream)


RATIOS = (1, 10, 20, 30, 40, 50)  # A:B task ratios of §4.3.2
RATIO_SCALES_Q16 = (1 << 16, 1 << 18, 1 << 20)  # HP gaps x1, x4, x16 (R24)


def ratio_sweep(seed: int = 3, n_base: int = 2000, T: int = 1000, n_hp_runs: int = 1000, n_lp_runs: int = 4000,
                ratios=RATIOS, scales=RATIO_SCALES_Q16) -> tuple[Config, StreamReplay, np.ndarray]:
    """SURVEY §8f row 4, the synthetic §4.3.2 experiment: the HP service A issues
    r tasks (r consecutive fresh inference runs, launched back to back) for every task of the
    LP service B (one inference, a kernel stream with its own think times), r in `ratios`.
    Models, measurement trace and runs are those of bert_vgg_stream (same seed): pairs
    (A BERT, B VGG) and (A VGG, B BERT), each at the HP gap scales `scales`.

    Scenario s: ratio index s % R; group g = s // R -> scale index g % n_scales, pair
    (g // n_scales) % 2, base b = g // (2 n_scales).  The HP window starts at run
    b mod (n_hp_runs - max r + 1) for every ratio of a group, so the windows of one group
    share their prefix (the prefix pin of tests/test_oracle_ratio.py).  Returns (config,
    stream replay, ratio per scenario).  S = 2 * n_scales * R * n_base."""
    cfg, sr = bert_vgg_stream(seed=seed, T=T, n_hp_runs=n_hp_runs, n_lp_runs=n_lp_runs, S=1)
    R, ns = len(ratios), len(scales)
    S = 2 * ns * R * n_base
    s = np.arange(S, dtype=np.int64)
    r = np.asarray(ratios, dtype=np.int64)[s % R]
    g = s // R
    scale = np.asarray(scales, dtype=np.int64)[g % ns]
    pair = (g // ns) % 2  # 0: A = BERT, B = VGG; 1: A = VGG, B = BERT
    b = g // (2 * ns)
    run = b % (n_hp_runs - max(ratios) + 1)
    L_hp = np.where(pair == 0, 176, 40)
    sc = np.zeros(S, dtype=SCEN_DTYPE)
    sc["hp_off"] = np.where(pair == 0, 0, n_hp_runs * 176) + run * L_hp
    sc["hp_len"] = r * L_hp
    lp_run = b % n_lp_runs
    sc["lp_off"] = np.where(pair == 0, lp_run * 40, 40 * n_lp_runs + lp_run * 176)
    sc["lp_len"] = np.where(pair == 0, 40, 176)
    sc["gap_scale_q16"] = scale
    rp = cfg.replay
    rp = Replay(rp.hp_records, rp.lp_records, rp.lp_level, sc, rp.threshold_ns, rp.feedback)
    return (Config("ratio_sweep", cfg.trace, rp, {"seed": seed, "S": S, "ratios": list(ratios)}),
            StreamReplay(rp, sr.lp_stream), r.astype(np.uint32))


ZIPF_S = 1.1


def _zipf_p(n: int, s: float = ZIPF_S) -> np.ndarray:
    p = np.arange(1, n + 1, dtype=np.float64) ** -s
    return p / p.sum()


def zipf_trace(seed: int = 4, n_runs: int = 390_625, run_len: int = 256, n_tasks: int = 32, vocab_per_task: int = 256,
               chunk_runs: int = 8192, rec_lo: int = 0, rec_hi: int | None = None, threads: int = 8) -> Config:
    """configs[3]: multi-model trace with Zipf(1.1) kernel-ID skew: 32 tasks x a
    256-kernel vocabulary each (<= 8,192 rows); runs of 256 launches; each
    run's task ~ Zipf(1.1) over 32 tasks; each launch's kernel ~ Zipf(1.1)
    over its task's vocabulary.  390,625 runs -> 100,000,000 records (4.8 GB).
    Durations log-U[2 us, 2 ms] per row x U[0.9, 1.1]; gaps as config R.

    Runs are generated in chunks of `chunk_runs`, each from its own seeded
    stream and time origin (chunk * 2^42 ns), so any record range
    [rec_lo, rec_hi) -- a rank's shard plus its halo -- is reproducible alone."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(seed)
    n_names = 2048
    names = _mangled_names(rng, n_names)
    sigs = _signatures(rng, 64)
    vocabs = [_vocab(rng, vocab_per_task, n_names, 64) for _ in range(n_tasks)]
    # share some identical tuples across tasks (rows are task-scoped, reading C3)
    for t in range(1, n_tasks):
        j = int(rng.integers(0, vocab_per_task // 4))
        for f in ("name_id", "sig_id"):
            getattr(vocabs[t], f)[j] = getattr(vocabs[0], f)[j]
        vocabs[t].grid[j] = vocabs[0].grid[j]
        vocabs[t].block[j] = vocabs[0].block[j]
    base_dur = _loguniform(rng, 2 * US, 2 * MS, (n_tasks, vocab_per_task))
    # rank -> vocabulary index permutation per task (hot kernels are not index 0)
    perm = np.stack([rng.permutation(vocab_per_task) for _ in range(n_tasks)])
    p_task = _zipf_p(n_tasks)
    p_k = _zipf_p(vocab_per_task)
    N = n_runs * run_len
    rec_hi = N if rec_hi is None else min(rec_hi, N)
    rec_lo = max(0, min(rec_lo, rec_hi))
    rec = np.zeros(rec_hi - rec_lo, dtype=REC_DTYPE)
    all_name = np.stack([v.name_id for v in vocabs])
    all_sig = np.stack([v.sig_id for v in vocabs])
    all_grid = np.stack([v.grid for v in vocabs])
    all_block = np.stack([v.block for v in vocabs])
    CR = chunk_runs * run_len

    def gen(c):
        r0 = c * chunk_runs
        nr = min(chunk_runs, n_runs - r0)
        n = nr * run_len
        crng = np.random.default_rng([seed, c])
        sl = np.zeros(n, dtype=REC_DTYPE)
        task = crng.choice(n_tasks, size=nr, p=p_task)
        task_r = np.repeat(task, run_len)
        kk = perm[task_r, crng.choice(vocab_per_task, size=n, p=p_k)]
        sl["name_id"] = all_name[task_r, kk]
        sl["sig_id"] = all_sig[task_r, kk]
        sl["grid_x"] = all_grid[task_r, kk, 0]
        sl["grid_y"] = all_grid[task_r, kk, 1]
        sl["grid_z"] = all_grid[task_r, kk, 2]
        sl["block_x"] = all_block[task_r, kk, 0]
        sl["block_y"] = all_block[task_r, kk, 1]
        sl["block_z"] = all_block[task_r, kk, 2]
        dur = np.maximum(np.rint(base_dur[task_r, kk] * crng.uniform(0.9, 1.1, n)), 1).astype(np.uint64)
        gap = np.clip(np.rint(_gap_mixture(crng, n) * crng.uniform(0.8, 1.2, n)), 1 * US, 20 * MS).astype(np.uint64)
        _timestamps(sl, dur, gap, run_len, c << 42)
        sl["run_id"] = r0 + np.repeat(np.arange(nr, dtype=np.uint32), run_len)
        sl["task_id"] = task_r.astype(np.uint32)
        a, b = max(rec_lo, c * CR), min(rec_hi, c * CR + n)
        rec[a - rec_lo : b - rec_lo] = sl[a - c * CR : b - c * CR]

    chunks = range(rec_lo // CR, (rec_hi - 1) // CR + 1) if rec_hi > rec_lo else range(0)
    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(gen, chunks))
    return Config("zipf", Trace(rec, StrTab.from_list(names), StrTab.from_list(sigs)), None,
                  {"seed": seed, "runs": n_runs, "run_len": run_len, "tasks": n_tasks, "vocab": vocab_per_task,
                   "p_task": p_task, "p_k": p_k, "perm": perm, "vocabs": vocabs, "N": N, "rec_lo": rec_lo,
                   "rec_hi": rec_hi})


def zipf_replay(cfg: Config, seed: int = 44, n_hp_runs: int = 1000, pop: int = 1 << 20, S: int = 100_000,
                m: int = 64) -> Replay:
    """Replay batch over the Z trace's tasks (the bench's a8-a10 leg): HP =
    fresh runs of the hottest task, LP = requests drawn from the next three
    tasks' vocabularies with the trace's Zipf kernel skew, level U{1,2,3}."""
    rng = np.random.default_rng(seed)
    md = cfg.meta
    vocabs, perm, p_k = md["vocabs"], md["perm"], md["p_k"]
    L = md["run_len"]

    def fresh(task, n, rng):
        kk = perm[task, rng.choice(len(vocabs[task]), size=n, p=p_k)]
        out = np.zeros(n, dtype=REC_DTYPE)
        _fill_identity(out, vocabs[task], kk)
        out["task_id"] = task
        return out, kk

    hp, _ = fresh(0, n_hp_runs * L, rng)
    dur = np.rint(_loguniform(rng, 2 * US, 2 * MS, hp.shape[0])).astype(np.uint64)
    gap = np.clip(np.rint(_gap_mixture(rng, hp.shape[0])), 1 * US, 20 * MS).astype(np.uint64)
    _timestamps(hp, dur, gap, L, 0)
    hp["run_id"] = np.repeat(np.arange(n_hp_runs, dtype=np.uint32), L)
    parts = []
    for t in (1, 2, 3):
        lp, _ = fresh(t, pop // 3 + (1 if t == 1 else 0) * (pop - 3 * (pop // 3)), rng)
        parts.append(lp)
    lp = np.concatenate(parts)
    lp["start_ns"] = 0
    lp["end_ns"] = np.rint(_loguniform(rng, 2 * US, 2 * MS, lp.shape[0])).astype(np.uint64)
    lp["run_id"] = np.arange(lp.shape[0], dtype=np.uint32)
    lvl = rng.integers(1, 4, size=lp.shape[0]).astype(np.uint8)
    s = np.arange(S, dtype=np.int64)
    sc = np.zeros(S, dtype=SCEN_DTYPE)
    sc["hp_off"] = (s % n_hp_runs) * L
    sc["hp_len"] = L
    sc["lp_off"] = (s * m) % (lp.shape[0] - m + 1)
    sc["lp_len"] = m
    # the Z gap mixture averages ~47 us, under the 0.1 ms gate: replay at scales 1, 2, 4, 8 (R24)
    sc["gap_scale_q16"] = (1 << 16) << (s % 4)
    return Replay(hp, lp, lvl, sc)


SWEEP_M = (8, 16, 32, 64, 128, 256, 512, 1024)
SWEEP_SCALE_Q16 = (1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 21)  # 1/4 .. 32


def sweep(seed: int = 5, T: int = 1000, n_hp_runs: int = 1000, pop: int = 1 << 20, S: int = 1_000_000) -> Config:
    """configs[4]: S scenarios over 64 sweep points (m in 8..1024 x gap scale
    in 1/4..32, point = s mod 64); HP template = {ResNet, BERT, VGG}[s mod 3]
    run (s/3) mod n_hp_runs; LP = the next model's population."""
    rng = np.random.default_rng(seed)
    names = _mangled_names(rng, 112)
    sigs = _signatures(rng, 40)
    models = [resnet50_model(rng, 40, 24, 0), bert_model(rng, 24, 16, 1, name_base=40),
              vgg_model(rng, 24, 16, 2, name_base=64, sig_base=16)]
    t = 0
    parts = []
    for mdl in models:
        r, t = mdl.runs(rng, T, 0, t0=t)
        parts.append(r)
    trace = Trace(np.concatenate(parts), StrTab.from_list(names), StrTab.from_list(sigs))
    hp_parts, hp_base = [], []
    off = 0
    for i, mdl in enumerate(models):
        r, _ = mdl.runs(rng, n_hp_runs, T)
        hp_parts.append(r)
        hp_base.append(off)
        off += r.shape[0]
    lp_parts = [mdl.requests(rng, pop) for mdl in models]
    hp = np.concatenate(hp_parts)
    lp = np.concatenate(lp_parts)
    lvl = rng.integers(1, 4, size=lp.shape[0]).astype(np.uint8)
    s = np.arange(S, dtype=np.int64)
    point = s % 64
    mm = np.array(SWEEP_M, dtype=np.int64)[point % 8]
    scale = np.array(SWEEP_SCALE_Q16, dtype=np.int64)[point // 8]
    hm = s % 3
    L = np.array([m.template.shape[0] for m in models], dtype=np.int64)
    run = (s // 3) % n_hp_runs
    sc = np.zeros(S, dtype=SCEN_DTYPE)
    sc["hp_off"] = np.array(hp_base, dtype=np.int64)[hm] + run * L[hm]
    sc["hp_len"] = L[hm]
    lm = (hm + 1) % 3
    sc["lp_off"] = lm * pop + (s * 1031) % (pop - mm + 1)
    sc["lp_len"] = mm
    sc["gap_scale_q16"] = scale
    return Config("sweep", trace, Replay(hp, lp, lvl, sc), {"seed": seed, "S": S})


# ---------------------------------------------------------------------------
# small random traces / pools for parity and property tests
# ---------------------------------------------------------------------------
def random_trace(seed: int, n: int, n_tasks: int = 3, n_ids: int = 20, run_len_max: int = 40, n_names: int = 12,
                 n_sigs: int = 5, overlap_frac: float = 0.0, zero_frac: float = 0.0, big_frac: float = 0.0) -> Trace:
    """Small random trace: runs of random length 1..run_len_max, random task
    per run, ids drawn from a per-trace vocabulary; optional overlapping
    launches (negative gaps), zero durations/gaps and > 2^32 ns values."""
    rng = np.random.default_rng(seed)
    names = _mangled_names(rng, n_names, 3, 40)
    sigs = _signatures(rng, n_sigs)
    v = _vocab(rng, n_ids, n_names, n_sigs)
    rec = np.zeros(n, dtype=REC_DTYPE)
    kidx = rng.integers(0, n_ids, size=n)
    _fill_identity(rec, v, kidx)
    dur = rng.integers(0, 3 * MS, size=n).astype(np.uint64)
    gap = rng.integers(0, 2 * MS, size=n).astype(np.int64)
    if zero_frac:
        dur[rng.random(n) < zero_frac] = 0
        gap[rng.random(n) < zero_frac] = 0
    if big_frac:
        dur[rng.random(n) < big_frac] += np.uint64(1 << 33)
    if overlap_frac:
        ov = rng.random(n) < overlap_frac
        gap[ov] = -rng.integers(1, 500 * US, size=int(ov.sum()))
    t = 10 * MS
    run, task = 0, int(rng.integers(0, n_tasks))
    left = int(rng.integers(1, run_len_max + 1))
    starts = np.empty(n, dtype=np.uint64)
    runs = np.empty(n, dtype=np.uint32)
    tasks = np.empty(n, dtype=np.uint32)
    for i in range(n):
        starts[i] = t
        runs[i] = run
        tasks[i] = task
        t = t + int(dur[i])
        left -= 1
        if left == 0:
            run += 1
            task = int(rng.integers(0, n_tasks))
            left = int(rng.integers(1, run_len_max + 1))
            t += RUN_PAUSE_NS
        else:
            t = max(0, t + int(gap[i]))
    rec["start_ns"] = starts
    rec["end_ns"] = starts + dur
    rec["run_id"] = runs
    rec["task_id"] = tasks
    return Trace(rec, StrTab.from_list(names), StrTab.from_list(sigs))


def random_replay(seed: int, trace: Trace, n_scen: int, m_max: int = 40, n_h_max: int = 30, levels: int = 3,
                  gap_scale=(1 << 16,), absent_frac: float = 0.05) -> Replay:
    """Random scenarios whose HP/LP kernels are drawn from `trace`'s own
    identities (plus a few identities absent from it), with fresh timings."""
    rng = np.random.default_rng(seed)
    src = trace.records
    hp_parts, lp_parts, lvl_parts = [], [], []
    sc = np.zeros(n_scen, dtype=SCEN_DTYPE)
    hoff = loff = 0
    for s in range(n_scen):
        nh = int(rng.integers(0, n_h_max + 1))
        m = int(rng.integers(0, m_max + 1))
        h = src[rng.integers(0, src.shape[0], size=nh)].copy() if src.shape[0] else np.zeros(0, REC_DTYPE)
        if nh:
            d = rng.integers(1, 2 * MS, size=nh).astype(np.uint64)
            g = np.where(rng.random(nh) < 0.5, rng.integers(1, 100 * US, size=nh),
                         rng.integers(100 * US, 5 * MS, size=nh)).astype(np.uint64)
            _timestamps(h, d, g, nh, 0)
            h["run_id"] = s
            bad = rng.random(nh) < absent_frac
            h["grid_x"][bad] += 7  # identity not in the trace -> no profile (p = 0)
        l = src[rng.integers(0, src.shape[0], size=m)].copy() if src.shape[0] else np.zeros(0, REC_DTYPE)
        if m:
            l["start_ns"] = 0
            l["end_ns"] = rng.integers(1, 3 * MS, size=m).astype(np.uint64)
            l["run_id"] = np.arange(m, dtype=np.uint32)
            bad = rng.random(m) < absent_frac
            l["grid_x"][bad] += 7  # no SK -> never a fill, still runs in the tail
        hp_parts.append(h)
        lp_parts.append(l)
        lvl_parts.append(rng.integers(1, levels + 1, size=m).astype(np.uint8))
        sc[s] = (hoff, nh, loff, m, int(rng.choice(gap_scale)), 0)
        hoff += nh
        loff += m
    cat = lambda ps: np.concatenate(ps) if ps else np.zeros(0, REC_DTYPE)
    return Replay(cat(hp_parts), cat(lp_parts), np.concatenate(lvl_parts) if lvl_parts else np.zeros(0, np.uint8),
                  sc, threshold_ns=100 * US, feedback=int(rng.integers(0, 2)))
