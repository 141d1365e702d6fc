"""Oracle pins for kernel identification (readings R1, R2).

Pinned against published FNV-1a-64 and splitmix64 vectors, SURVEY §8c-5's
independently computed composite IDs, and the position/run
independence stated at P:239."""
import numpy as np
import pytest

import fikit_synth as F
from helpers import golden_lines


def _golden():
    for ln in golden_lines("hash_vectors.txt"):
        import shlex

        yield shlex.split(ln)


@pytest.mark.parametrize("row", list(_golden()), ids=lambda r: r[0] + ":" + r[1])
def test_hash_vectors(orc, row):
    kind = row[0]
    if kind == "fnv":
        assert orc.fnv1a64(row[1].encode()) == int(row[2], 16)
    elif kind == "mix":
        assert orc.mix64(int(row[1], 16)) == int(row[2], 16)
    else:
        grid = tuple(int(x) for x in row[3].split(","))
        block = tuple(int(x) for x in row[4].split(","))
        assert orc.kernel_id(row[1].encode(), row[2].encode(), grid, block) == int(row[5], 16)


def test_spec_equal_unequal(orc):
    # S:77 identical inputs -> equal IDs ; S:78 grid dim is part of the identity
    a = orc.kernel_id(b"vectorAdd", b"", (16, 1, 1), (256, 1, 1))
    assert a == orc.kernel_id(b"vectorAdd", b"", (16, 1, 1), (256, 1, 1))
    assert a != orc.kernel_id(b"vectorAdd", b"", (32, 1, 1), (256, 1, 1))
    # every field of the tuple matters (P:190 name + block + grid; R1 signature)
    variants = [(b"vectorAdd2", b"", (16, 1, 1), (256, 1, 1)), (b"vectorAdd", b"(int)", (16, 1, 1), (256, 1, 1)),
                (b"vectorAdd", b"", (16, 2, 1), (256, 1, 1)), (b"vectorAdd", b"", (16, 1, 2), (256, 1, 1)),
                (b"vectorAdd", b"", (16, 1, 1), (128, 1, 1)), (b"vectorAdd", b"", (16, 1, 1), (256, 2, 1)),
                (b"vectorAdd", b"", (16, 1, 1), (256, 1, 2))]
    ids = {orc.kernel_id(*v) for v in variants}
    assert len(ids) == len(variants) and a not in ids


def test_identify_position_and_run_independent(orc):
    # "The Kernel ID is independent of kernel's sequential index within a task [...] also
    # independent of index of t-th run"
    tr = F.random_trace(7, 400)
    kid, st = orc.identify(tr.records, tr.names, tr.sigs)
    assert st["code"] == 0
    perm = np.random.default_rng(0).permutation(400)
    r2 = tr.records[perm].copy()
    r2["run_id"] = np.arange(400)
    r2["start_ns"] = 0
    r2["end_ns"] = 5
    kid2, _ = orc.identify(r2, tr.names, tr.sigs)
    assert np.array_equal(kid2, kid[perm])
    # the ID of each record equals the ID of its tuple
    for i in range(0, 400, 37):
        r = tr.records[i]
        want = orc.kernel_id(tr.names.get(r["name_id"]), tr.sigs.get(r["sig_id"]),
                             (int(r["grid_x"]), int(r["grid_y"]), int(r["grid_z"])),
                             (int(r["block_x"]), int(r["block_y"]), int(r["block_z"])))
        assert kid[i] == want


def test_identify_interned_duplicates_share_id(orc):
    # two name_ids with identical bytes are the same kernel function (content hash, R2)
    names = F.StrTab.from_list([b"foo_kernel", b"bar", b"foo_kernel"])
    sigs = F.StrTab.from_list([b""])
    r = np.zeros(2, dtype=F.REC_DTYPE)
    r["name_id"] = [0, 2]
    for f in ("grid_x", "grid_y", "grid_z", "block_x", "block_y", "block_z"):
        r[f] = 1
    kid, st = orc.identify(r, names, sigs)
    assert st["code"] == 0 and kid[0] == kid[1]


@pytest.mark.parametrize("field,val", [("grid_x", 0), ("grid_y", 0), ("grid_z", 0), ("block_x", 0), ("block_y", 0),
                                       ("block_z", 0), ("name_id", 99), ("sig_id", 99), ("flags", 1)])
def test_identify_invalid(orc, field, val):
    # SPEC S:72-74 (zero dimension -> validation error), a1
    tr = F.random_trace(3, 50)
    rec = tr.records.copy()
    rec[field][17] = val
    rec[field][31] = val
    _, st = orc.identify(rec, tr.names, tr.sigs)
    assert st["code"] == orc.E_RECORD and st["first_bad_index"] == 17


def test_identify_empty_name(orc):
    names = F.StrTab.from_list([b"a", b""])
    r = np.zeros(1, dtype=F.REC_DTYPE)
    for f in ("grid_x", "grid_y", "grid_z", "block_x", "block_y", "block_z"):
        r[f] = 1
    _, st = orc.identify(r, names, F.StrTab.from_list([b""]))
    assert st["code"] == orc.E_NAME
