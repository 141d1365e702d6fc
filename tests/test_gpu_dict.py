"""GPU parity of the dictionary-supplied measure mode (fikit_measure_dict, include/fikit.h;
SURVEY §8e "B200-native upgrade", repeated services keep their IDs) and of the merge it
enables (dist.merge_tables_dict: two all-reduces, no key exchange).

Expected values come from the oracle: the measured rows of a dictionary-mode table equal the
oracle's table rows placed at their dictionary positions, the other dictionary rows
are empty, E_DICT reports the first launch whose identity the dictionary lacks, and a merged
dictionary-mode table equals the unsharded oracle table."""
import numpy as np
import pytest

import fikit_synth as F
from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

FIELDS = ("dur_cnt", "dur_sum", "dur_min", "dur_max", "gap_cnt", "gap_sum", "gap_min", "gap_max", "dur_hist",
          "gap_hist", "dur_mean", "gap_mean")


@pytest.fixture(scope="module")
def fk():
    import paper_2311_10359_b200 as fk
    from paper_2311_10359_b200 import _build

    _build.build()
    return fk


def dict_tensors(keys):
    import torch

    kid = np.array([k for _, k in keys], dtype=np.uint64)
    task = np.array([t for t, _ in keys], dtype=np.uint32)
    return (torch.from_numpy(kid.view(np.int64)).cuda(), torch.from_numpy(task.view(np.int32)).cuda(), len(keys))


def oracle_keys(tab):
    return [(int(tab.task_id[r]), int(tab.kernel_id[r])) for r in range(tab.n_rows)]


def run_dict(fk, recs, names, sigs, keys, cap, halo=None, want_rows=False, ws=None, strtabs=None, reuse=False,
             dictionary=None):
    import torch

    from paper_2311_10359_b200 import (Table, Workspace, measure, records_to_device, strtab_to_device,
                                       table_finalize)

    n = recs.shape[0]
    d_recs = records_to_device(recs) if n else torch.zeros(48, dtype=torch.uint8, device="cuda")
    t = Table(cap)
    if ws is None:
        ws = Workspace(cap, max(1, names.count), max(1, sigs.count), n_records=n)
    rows = torch.empty(max(1, n), dtype=torch.int32, device="cuda") if want_rows else None
    h = records_to_device(halo.reshape(1)) if halo is not None else None
    dn, ds = strtabs if strtabs is not None else (strtab_to_device(names), strtab_to_device(sigs))
    measure(d_recs, n, dn, ds, t, ws, halo=h, out_row=rows,
            dictionary=dictionary if dictionary is not None else dict_tensors(keys), reuse_plan=reuse)
    st = fk.get_status(ws)
    table_finalize(t, ws, out_row=rows, n=n)
    return t, st, rows


def check_dict_table(got, keys, ref_tab):
    """got (Table.to_numpy) holds every dictionary key in order; the oracle's rows at their
    dictionary positions, empty rows elsewhere."""
    assert got["kernel_id"].shape[0] == len(keys)
    assert [(int(a), int(b)) for a, b in zip(got["task_id"], got["kernel_id"])] == keys
    pos = {k: j for j, k in enumerate(keys)}
    ref = ref_tab.head()
    at = np.array([pos[k] for k in oracle_keys(ref_tab)], dtype=np.int64)
    for f in FIELDS:
        assert np.array_equal(got[f][at], ref[f]), f
    empty = np.setdiff1d(np.arange(len(keys)), at)
    assert np.all(got["dur_cnt"][empty] == 0) and np.all(got["gap_cnt"][empty] == 0)
    assert np.all(got["dur_min"][empty] == 2**64 - 1) and np.all(got["dur_max"][empty] == 0)
    assert np.all(got["dur_hist"][empty] == 0) and np.all(got["dur_mean"][empty] == 0)


@pytest.mark.parametrize("seed,n,kw", [(1, 5000, {}), (2, 20000, {"overlap_frac": 0.2}), (3, 257, {}),
                                        (4, 70000, {"n_ids": 3000, "n_tasks": 5}), (5, 1, {})])
def test_measure_dict_parity(fk, orc, seed, n, kw):
    kw = {"n_tasks": 3, "n_ids": 200, "run_len_max": 40, **kw}
    tr = F.random_trace(seed, n, **kw)
    ref, st_ref, ref_rows = orc.measure(tr.records, tr.names, tr.sigs, capacity=1 << 16, want_rows=True)
    assert st_ref["code"] == 0
    rng = np.random.default_rng(seed)
    extra = {(int(rng.integers(0, 50)), int(rng.integers(1, 2**63))) for _ in range(37)}
    keys = sorted(set(oracle_keys(ref)) | extra)
    t, st, rows = run_dict(fk, tr.records, tr.names, tr.sigs, keys, cap=len(keys) + 5, want_rows=True)
    assert st["code"] == 0, st
    check_dict_table(t.to_numpy(), keys, ref)
    # out_row: each launch's dictionary position
    pos = {k: j for j, k in enumerate(keys)}
    exp = np.array([pos[k] for k in oracle_keys(ref)], dtype=np.uint32)[ref_rows]
    assert np.array_equal(rows.cpu().numpy().view(np.uint32)[:n], exp)


def test_measure_dict_zipf_hot_path(fk, orc):
    # a skewed multi-task trace: both hot-set schedules run against the supplied rows
    cfg = F.zipf_trace(n_runs=4000, threads=8)
    tr = cfg.trace
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=8192)
    keys = oracle_keys(ref)
    t, st, _ = run_dict(fk, tr.records, tr.names, tr.sigs, keys, cap=8192)
    assert st["code"] == 0, st
    check_dict_table(t.to_numpy(), keys, ref)


def test_measure_dict_missing_identity(fk, orc):
    tr = F.random_trace(11, 6000, n_tasks=2, n_ids=60, run_len_max=30)
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=1024)
    keys = oracle_keys(ref)
    kid, _ = orc.identify(tr.records, tr.names, tr.sigs)
    gone = keys[17]
    keys = [k for k in keys if k != gone]
    first = int(np.flatnonzero((tr.records["task_id"] == gone[0]) & (kid == gone[1]))[0])
    _, st, _ = run_dict(fk, tr.records, tr.names, tr.sigs, keys, cap=1024)
    assert st["code"] == fk.E_DICT and st["first_missing_index"] == first


def test_measure_dict_bad_order_and_args(fk):
    tr = F.random_trace(12, 500, n_tasks=2, n_ids=10)
    _, st, _ = run_dict(fk, tr.records, tr.names, tr.sigs, [(0, 5), (0, 5)], cap=8)  # not strictly increasing
    assert st["code"] == fk.E_ARG
    with pytest.raises(fk.FikitError):
        run_dict(fk, tr.records, tr.names, tr.sigs, [(0, k) for k in range(1, 20)], cap=8)  # dict_n > capacity


@pytest.mark.parametrize("P", [2, 3, 8])
def test_dict_merge_one_gpu(fk, orc, P):
    """P record shards (+ halo) measured against one dictionary; the rank tables reduced the way
    merge_tables_dict does (bias, SUM span, MAX ext, bias, means) equal the unsharded oracle."""
    import torch

    from paper_2311_10359_b200.dist import shard_range

    cfg = F.zipf_trace(n_runs=1500, threads=8)
    tr = cfg.trace
    N = tr.records.shape[0]
    ref, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=8192)
    keys = oracle_keys(ref)
    tabs = []
    for r in range(P):
        lo, hi = shard_range(N, r, P)
        t, st, _ = run_dict(fk, tr.records[lo:hi], tr.names, tr.sigs, keys, cap=8192,
                            halo=tr.records[hi] if hi < N else None)
        assert st["code"] == 0
        fk.table_bias(t)
        tabs.append(t)
    out = tabs[0]
    for t in tabs[1:]:  # what the SUM / MAX all-reduces compute
        out.sum_span().add_(t.sum_span())
        torch.maximum(out.ext, t.ext, out=out.ext)
    fk.table_bias(out)
    fk.table_means(out)
    check_dict_table(out.to_numpy(), keys, ref)


@pytest.mark.parametrize("kind", ["zipf", "resnet"])
def test_measure_dict_reuse_plan(fk, orc, kind):
    """FIKIT_MEASURE_REUSE_PLAN: a second trace of the same services measured with the first
    call's hot sets and string hashes gives the oracle's table for the second trace (Zipf:
    task-bucket schedule; ResNet-like: address order, the schedule kernels exit at once); a
    different dictionary is rejected (E_ARG)."""
    from paper_2311_10359_b200 import Workspace, strtab_to_device

    if kind == "zipf":
        cfg = F.zipf_trace(n_runs=3000, threads=8)
        run = 256
    else:
        cfg = F.resnet_trace(n_runs=3000)
        run = 300
    tr = cfg.trace
    a, b = tr.records[: run * 1500], tr.records[run * 1500:]
    ref_all, _, _ = orc.measure(tr.records, tr.names, tr.sigs, capacity=8192)
    keys = oracle_keys(ref_all)
    ref_b, _, _ = orc.measure(b, tr.names, tr.sigs, capacity=8192)
    ws = Workspace(8192, tr.names.count, tr.sigs.count, n_records=tr.records.shape[0])
    st_tabs = (strtab_to_device(tr.names), strtab_to_device(tr.sigs))
    dic = dict_tensors(keys)
    _, st, _ = run_dict(fk, a, tr.names, tr.sigs, keys, 8192, ws=ws, strtabs=st_tabs, dictionary=dic)
    assert st["code"] == 0
    t, st, _ = run_dict(fk, b, tr.names, tr.sigs, keys, 8192, ws=ws, strtabs=st_tabs, dictionary=dic, reuse=True)
    assert st["code"] == 0, st
    check_dict_table(t.to_numpy(), keys, ref_b)
    # a plan built on another dictionary
    other = keys[:-1]
    _, st, _ = run_dict(fk, b[: run * 10], tr.names, tr.sigs, other, 8192, ws=ws, strtabs=st_tabs, reuse=True)
    assert st["code"] == fk.E_ARG
    # reuse without a dictionary: a host-side argument error
    import ctypes as C

    t2 = fk.Table(8192)
    rc = fk.lib().fikit_measure_dict_ex(None, 0, None, st_tabs[0].c(), st_tabs[1].c(), None, None, 0, 1,
                                        C.byref(t2.c), None, ws.ptr(), ws.nbytes, None, None, None)
    assert rc == fk.E_ARG
    st = fk.get_status(ws)  # (the reused plan's schedule mode is the one the kind exercises)
    assert st["schedule"] == (1 if kind == "zipf" else 0) or st["code"] != 0
