"""Thin Python binding of libfikit.so (include/fikit.h): the B200 hot path of FIKIT.

Argument marshalling only -- every step of identify / measure / finalize /
resolve / fill / simulate runs in the library's CUDA kernels.  PyTorch
supplies device memory and streams.  There is no CPU fallback: importing
this module without the built library, or calling it without a CUDA device,
raises.

Function names follow the C-ABI (fikit_<name> -> <name>).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FIKIT_DIAG_LIB") or os.path.join(_HERE, "libfikit.so")  # (diagnosis builds: scripts/)

OK, E_ARG, E_RECORD, E_CAPACITY, E_CUDA, E_NAME, E_DICT = 0, -1, -2, -3, -4, -5, -6
NO_ROW = 0xFFFFFFFF
NBINS = 32
SYMBOLS = ("fikit_ws_bytes", "fikit_table_bytes", "fikit_table_carve", "fikit_identify", "fikit_measure",
           "fikit_measure_timed", "fikit_measure_dict", "fikit_measure_dict_timed", "fikit_measure_dict_ex", "fikit_table_finalize", "fikit_table_means", "fikit_table_predict", "fikit_resolve", "fikit_resolve_ex", "fikit_lookup", "fikit_fill",
           "fikit_simulate_batch", "fikit_simulate_stream_batch",
           "fikit_dict_union", "fikit_table_remap", "fikit_table_bias", "fikit_get_status", "fikit_strerror",
           "fikit_launch_count")


class FikitError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        super().__init__(f"libfikit: {what}: {_strerror(code)} ({code})")


class StrTabC(C.Structure):
    _fields_ = [("bytes", C.c_void_p), ("offsets", C.c_void_p), ("count", C.c_uint32)]


class TableC(C.Structure):
    _fields_ = [("kernel_id", C.c_void_p), ("task_id", C.c_void_p), ("sums", C.c_void_p), ("hist", C.c_void_p),
                ("ext", C.c_void_p), ("mean", C.c_void_p), ("n_rows", C.c_void_p), ("capacity", C.c_uint32)]


class StatusC(C.Structure):
    _fields_ = [("code", C.c_int32), ("flags", C.c_uint32), ("first_bad_index", C.c_uint64),
                ("n_rows_needed", C.c_uint64), ("n_overlap_gaps", C.c_uint64), ("schedule", C.c_uint32),
                ("n_task_buckets", C.c_uint32), ("first_missing_index", C.c_uint64)]


class FillParamsC(C.Structure):
    _fields_ = [("threshold_ns", C.c_uint64), ("feedback", C.c_uint32), ("flags", C.c_uint32)]


RESULT_DTYPE = np.dtype([("hp_jct", "<u8"), ("lp_jct", "<u8"), ("hp_delay", "<u8"), ("fill_work", "<u8"),
                         ("digest", "<u8"), ("n_fills", "<u4"), ("n_tail", "<u4")])

_lib = None


def lib():
    """Load libfikit.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        p, u32, u64, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_size_t
        L.fikit_ws_bytes.restype = sz
        L.fikit_ws_bytes.argtypes = [u32, u32, u32, u64]
        L.fikit_table_bytes.restype = sz
        L.fikit_table_bytes.argtypes = [u32]
        L.fikit_table_carve.argtypes = [p, u32, C.POINTER(TableC)]
        L.fikit_identify.argtypes = [p, u64, StrTabC, StrTabC, p, p, sz, p]
        L.fikit_measure.argtypes = [p, u64, p, StrTabC, StrTabC, C.POINTER(TableC), p, p, sz, p]
        L.fikit_measure_timed.argtypes = [p, u64, p, StrTabC, StrTabC, C.POINTER(TableC), p, p, sz, p, p, p]
        L.fikit_measure_dict.argtypes = [p, u64, p, StrTabC, StrTabC, p, p, u32, C.POINTER(TableC), p, p, sz, p]
        L.fikit_measure_dict_timed.argtypes = [p, u64, p, StrTabC, StrTabC, p, p, u32, C.POINTER(TableC), p, p, sz,
                                               p, p, p]
        L.fikit_measure_dict_ex.argtypes = [p, u64, p, StrTabC, StrTabC, p, p, u32, u32, C.POINTER(TableC), p, p, sz,
                                            p, p, p]
        L.fikit_table_finalize.argtypes = [C.POINTER(TableC), p, u64, p, sz, p]
        L.fikit_table_means.argtypes = [C.POINTER(TableC), p]
        L.fikit_table_predict.argtypes = [C.POINTER(TableC), u32, u32, p]
        L.fikit_resolve.argtypes = [p, u64, p, StrTabC, StrTabC, C.POINTER(TableC), p, p, p, p, sz, p]
        L.fikit_resolve_ex.argtypes = [p, u64, p, StrTabC, StrTabC, C.POINTER(TableC), p, p, p, u32, p, sz, p]
        L.fikit_lookup.argtypes = [C.POINTER(TableC), p, p, u64, p, p]
        L.fikit_fill.argtypes = [C.POINTER(TableC), p, p, p, p, p, p, p, u32, FillParamsC, p, p, p, p, p, p, sz, p]
        L.fikit_simulate_batch.argtypes = [C.POINTER(TableC), p, p, p, p, p, p, p, u32, FillParamsC, p, p, p, p, p,
                                           sz, p]
        L.fikit_simulate_stream_batch.argtypes = [C.POINTER(TableC), p, p, p, p, p, p, p, p, p, p, u32,
                                                  FillParamsC, p, p, p, p, p, sz, p]
        L.fikit_dict_union.argtypes = [p, p, p, u32, u32, u32, p, p, u32, p, p, p, sz, p]
        L.fikit_table_remap.argtypes = [C.POINTER(TableC), p, p, p, p, C.POINTER(TableC), p]
        L.fikit_table_bias.argtypes = [C.POINTER(TableC), p]
        L.fikit_get_status.argtypes = [p, C.POINTER(StatusC), p]
        L.fikit_strerror.restype = C.c_char_p
        L.fikit_strerror.argtypes = [C.c_int]
        L.fikit_launch_count.restype = u64
        _lib = L
    return _lib


def _strerror(code):
    try:
        return lib().fikit_strerror(code).decode()
    except Exception:
        return "?"


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_10359_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _chk(code, what):
    if code != OK:
        raise FikitError(code, what)


def launch_count() -> int:
    return int(lib().fikit_launch_count())


# ---------------------------------------------------------------------------
# device containers
# ---------------------------------------------------------------------------
@dataclass
class DevStrTab:
    data: object  # torch uint8
    offsets: object  # torch int32 (u32 bits)
    count: int

    def c(self):
        return StrTabC(_ptr(self.data), _ptr(self.offsets), self.count)


def strtab_to_device(tab, device="cuda") -> DevStrTab:
    """The bytes are zero-padded to a multiple of 16: the kernels read whole aligned 16-B blocks
    (include/fikit.h), so the padding keeps every byte they touch initialised."""
    torch = _torch()
    raw = np.ascontiguousarray(tab.data, dtype=np.uint8)
    pad = np.zeros(((raw.shape[0] + 16) // 16) * 16, dtype=np.uint8)
    pad[: raw.shape[0]] = raw
    data = torch.from_numpy(pad).to(device)
    offs = torch.from_numpy(np.ascontiguousarray(tab.offsets).view(np.int32)).to(device)
    return DevStrTab(data, offs, int(tab.count))


def records_to_device(rec: np.ndarray, device="cuda", pinned_src=None):
    """48-byte launch records -> a uint8 device tensor (16-B aligned)."""
    torch = _torch()
    assert rec.dtype.itemsize == 48
    host = torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8).reshape(-1))
    return host.to(device)


class Workspace:
    def __init__(self, capacity: int, n_names: int, n_sigs: int, device="cuda", extra: int = 0, n_records: int = 0):
        torch = _torch()
        self.capacity, self.n_names, self.n_sigs = capacity, n_names, n_sigs
        self.nbytes = int(lib().fikit_ws_bytes(capacity, n_names, n_sigs, n_records)) + int(extra)
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8, device=device)
        off = (-self.buf.data_ptr()) % 256
        self.t = self.buf[off:off + self.nbytes]

    def ptr(self):
        return _ptr(self.t)


class Table:
    """A statistic table of `capacity` rows in one device block (fikit_table_carve)."""

    def __init__(self, capacity: int, device="cuda"):
        torch = _torch()
        self.capacity = int(capacity)
        nb = int(lib().fikit_table_bytes(self.capacity))
        self.block = torch.zeros(nb + 256, dtype=torch.uint8, device=device)
        off = (-self.block.data_ptr()) % 256
        self.c = TableC()
        _chk(lib().fikit_table_carve(C.c_void_p(self.block.data_ptr() + off), self.capacity, C.byref(self.c)),
             "table_carve")
        base = self.block.data_ptr()
        cap = self.capacity

        def view(addr, n, dtype, esize):
            o = addr - base
            return self.block[o:o + n * esize].view(dtype)

        self.kernel_id = view(self.c.kernel_id, cap, torch.int64, 8)
        self.task_id = view(self.c.task_id, cap, torch.int32, 4)
        self.sums = view(self.c.sums, cap * 4, torch.int64, 8)
        self.hist = view(self.c.hist, cap * 64, torch.int32, 4)
        self.ext = view(self.c.ext, cap * 4, torch.int64, 8)
        self.mean = view(self.c.mean, cap * 2, torch.int64, 8)
        self.n_rows_t = view(self.c.n_rows, 1, torch.int32, 4)

    def zero(self):
        self.block.zero_()

    def sum_span(self):
        """int64 view over the SUM block and the histogram block when they are adjacent
        (fikit_table_carve: capacity a multiple of 8), else None.  Summing the u32 bins pairwise
        as u64 words is exact while every summed bin stays < 2^32 (R37)."""
        torch = _torch()
        if self.c.hist != self.c.sums + 32 * self.capacity:
            return None
        o = self.c.sums - self.block.data_ptr()
        return self.block[o:o + 288 * self.capacity].view(torch.int64)

    def n_rows(self) -> int:
        return int(self.n_rows_t.item()) & 0xFFFFFFFF

    def to_numpy(self) -> dict:
        """Host copy in the oracle's field names (cut to n_rows)."""
        n = min(self.n_rows(), self.capacity)
        u64 = lambda t: t.cpu().numpy().view(np.uint64)
        sums = u64(self.sums).reshape(-1, 4)[:n]
        ext = u64(self.ext).reshape(-1, 4)[:n]
        hist = self.hist.cpu().numpy().view(np.uint32).reshape(-1, 64)[:n]
        mean = u64(self.mean).reshape(-1, 2)[:n]
        return {
            "kernel_id": u64(self.kernel_id)[:n], "task_id": self.task_id.cpu().numpy().view(np.uint32)[:n],
            "dur_cnt": sums[:, 0], "dur_sum": sums[:, 1], "gap_cnt": sums[:, 2], "gap_sum": sums[:, 3],
            "dur_max": ext[:, 0], "dur_min": ~ext[:, 1], "gap_max": ext[:, 2], "gap_min": ~ext[:, 3],
            "dur_hist": hist[:, :32], "gap_hist": hist[:, 32:], "dur_mean": mean[:, 0], "gap_mean": mean[:, 1],
        }


# ---------------------------------------------------------------------------
# entry points (fikit_<name>)
# ---------------------------------------------------------------------------
def get_status(ws: Workspace, stream=None) -> dict:
    st = StatusC()
    lib().fikit_get_status(ws.ptr(), C.byref(st), _stream(stream))
    return {"code": st.code, "flags": st.flags, "first_bad_index": st.first_bad_index,
            "n_rows_needed": st.n_rows_needed, "n_overlap_gaps": st.n_overlap_gaps, "schedule": st.schedule,
            "n_task_buckets": st.n_task_buckets, "first_missing_index": st.first_missing_index}


def check(ws: Workspace, what="", stream=None) -> dict:
    st = get_status(ws, stream)
    if st["code"] != OK:
        raise FikitError(st["code"], f"{what} (first_bad_index={st['first_bad_index']}, "
                                     f"n_rows_needed={st['n_rows_needed']})")
    return st


def identify(recs, n: int, names: DevStrTab, sigs: DevStrTab, out_kid, ws: Workspace, stream=None):
    _chk(lib().fikit_identify(_ptr(recs), n, names.c(), sigs.c(), _ptr(out_kid), ws.ptr(), ws.nbytes,
                              _stream(stream)), "identify")


def measure(recs, n: int, names: DevStrTab, sigs: DevStrTab, table: Table, ws: Workspace, halo=None, out_row=None,
            stream=None, events=None, dictionary=None, reuse_plan: bool = False):
    """events: (start, stop) torch.cuda.Event pair recorded around the fused streaming kernel
    (fikit_measure_timed; the events must exist, i.e. have been recorded once).  dictionary:
    (kid int64 device tensor, task int32 device tensor, n) -> fikit_measure_dict_ex; reuse_plan:
    FIKIT_MEASURE_REUSE_PLAN (keep the previous dictionary call's string hashes and hot sets)."""
    if dictionary is not None:
        dk, dt, dn = dictionary[:3]
        flags = 1 if reuse_plan else 0  # FIKIT_MEASURE_REUSE_PLAN
        e0, e1 = (C.c_void_p(events[0].cuda_event), C.c_void_p(events[1].cuda_event)) if events else (None, None)
        _chk(lib().fikit_measure_dict_ex(_ptr(recs), n, _ptr(halo), names.c(), sigs.c(), _ptr(dk), _ptr(dt), int(dn),
                                         flags, C.byref(table.c), _ptr(out_row), ws.ptr(), ws.nbytes, _stream(stream),
                                         e0, e1), "measure_dict")
        return
    if events is None:
        _chk(lib().fikit_measure(_ptr(recs), n, _ptr(halo), names.c(), sigs.c(), C.byref(table.c), _ptr(out_row),
                                 ws.ptr(), ws.nbytes, _stream(stream)), "measure")
    else:
        e0, e1 = events
        _chk(lib().fikit_measure_timed(_ptr(recs), n, _ptr(halo), names.c(), sigs.c(), C.byref(table.c),
                                       _ptr(out_row), ws.ptr(), ws.nbytes, _stream(stream),
                                       C.c_void_p(e0.cuda_event), C.c_void_p(e1.cuda_event)), "measure_timed")


def table_finalize(table: Table, ws: Workspace, out_row=None, n: int = 0, stream=None):
    _chk(lib().fikit_table_finalize(C.byref(table.c), _ptr(out_row), n if out_row is not None else 0, ws.ptr(),
                                    ws.nbytes, _stream(stream)), "table_finalize")


def table_means(table: Table, stream=None):
    _chk(lib().fikit_table_means(C.byref(table.c), _stream(stream)), "table_means")


PREDICT_MEAN, PREDICT_PERCENTILE, PREDICT_EXTREMES = 0, 1, 2


def table_predict(table: Table, mode: int, pct: int = 90, stream=None):
    """fikit_table_predict: the replay's predictions from the table (0 means, 1 percentile pct, 2 extremes)."""
    _chk(lib().fikit_table_predict(C.byref(table.c), mode, pct, _stream(stream)), "table_predict")


def resolve(recs, n: int, names: DevStrTab, sigs: DevStrTab, table: Table, out_row, out_dur, out_gap, ws: Workspace,
            halo=None, stream=None, reuse_hashes: bool = False):
    """reuse_hashes: the workspace holds these string tables' hashes from the previous measure /
    resolve call on it (FIKIT_RESOLVE_REUSE_HASHES: no re-hashing)."""
    if reuse_hashes:
        _chk(lib().fikit_resolve_ex(_ptr(recs), n, _ptr(halo), names.c(), sigs.c(), C.byref(table.c), _ptr(out_row),
                                    _ptr(out_dur), _ptr(out_gap), 1, ws.ptr(), ws.nbytes, _stream(stream)),
             "resolve_ex")
        return
    _chk(lib().fikit_resolve(_ptr(recs), n, _ptr(halo), names.c(), sigs.c(), C.byref(table.c), _ptr(out_row),
                             _ptr(out_dur), _ptr(out_gap), ws.ptr(), ws.nbytes, _stream(stream)), "resolve")


def lookup(table: Table, kid, task, n: int, out_row, stream=None):
    _chk(lib().fikit_lookup(C.byref(table.c), _ptr(kid), _ptr(task), n, _ptr(out_row), _stream(stream)), "lookup")


def fill(table: Table, R0, deadline, pool_row, pool_dur, pool_level, pool_off, pool_len, G: int, picks, picks_off,
         n_picks, R_left, t_used, ws: Workspace, threshold_ns=100_000, feedback=1, stream=None):
    prm = FillParamsC(threshold_ns, feedback, 0)
    _chk(lib().fikit_fill(C.byref(table.c), _ptr(R0), _ptr(deadline), _ptr(pool_row), _ptr(pool_dur),
                          _ptr(pool_level), _ptr(pool_off), _ptr(pool_len), G, prm, _ptr(picks), _ptr(picks_off),
                          _ptr(n_picks), _ptr(R_left), _ptr(t_used), ws.ptr(), ws.nbytes, _stream(stream)), "fill")


def simulate_batch(table: Table, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, scenarios, S: int, out,
                   ws: Workspace, threshold_ns=100_000, feedback=1, fill_gap=None, lp_start=None, sched_off=None,
                   stream=None):
    prm = FillParamsC(threshold_ns, feedback, 0)
    _chk(lib().fikit_simulate_batch(C.byref(table.c), _ptr(hp_row), _ptr(hp_dur), _ptr(hp_gap), _ptr(lp_row),
                                    _ptr(lp_dur), _ptr(lp_level), _ptr(scenarios), S, prm, _ptr(out),
                                    _ptr(fill_gap), _ptr(lp_start), _ptr(sched_off), ws.ptr(), ws.nbytes,
                                    _stream(stream)), "simulate_batch")


def simulate_stream_batch(table: Table, hp_row, hp_dur, hp_gap, lp_row, lp_dur, lp_level, lp_stream, lp_think,
                          scenarios, S: int, out, ws: Workspace, threshold_ns=100_000, feedback=1, fill_gap=None,
                          lp_start=None, sched_off=None, stream=None, hp_arrival=None):
    """fikit_simulate_stream_batch: the STREAM model (LP kernel streams, R29-R32; hp_arrival: Case A)."""
    prm = FillParamsC(threshold_ns, feedback, 0)
    _chk(lib().fikit_simulate_stream_batch(C.byref(table.c), _ptr(hp_row), _ptr(hp_dur), _ptr(hp_gap), _ptr(lp_row),
                                           _ptr(lp_dur), _ptr(lp_level), _ptr(lp_stream), _ptr(lp_think),
                                           _ptr(hp_arrival), _ptr(scenarios), S, prm, _ptr(out), _ptr(fill_gap), _ptr(lp_start),
                                           _ptr(sched_off), ws.ptr(), ws.nbytes, _stream(stream)),
         "simulate_stream_batch")


def dict_union(all_kid, all_task, n_list, P: int, Kmax: int, self_rank: int, out_kid, out_task, cap_out: int, out_n,
               local_to_union, ws: Workspace, stream=None):
    _chk(lib().fikit_dict_union(_ptr(all_kid), _ptr(all_task), _ptr(n_list), P, Kmax, self_rank, _ptr(out_kid),
                                _ptr(out_task), cap_out, _ptr(out_n), _ptr(local_to_union), ws.ptr(), ws.nbytes,
                                _stream(stream)), "dict_union")


def table_remap(local: Table, local_to_union, union_kid, union_task, union_n, dense: Table, stream=None):
    _chk(lib().fikit_table_remap(C.byref(local.c), _ptr(local_to_union), _ptr(union_kid), _ptr(union_task),
                                 _ptr(union_n), C.byref(dense.c), _stream(stream)), "table_remap")


def table_bias(table: Table, stream=None):
    _chk(lib().fikit_table_bias(C.byref(table.c), _stream(stream)), "table_bias")
