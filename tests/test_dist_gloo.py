"""Multi-process (world_size 2 and 3, gloo, CPU) test of the multi-GPU merge
plumbing in paper_2311_10359_b200/dist.py: record shards with a one-record
halo, all_gather of the row keys, dictionary union, remap, the order-biased
MAX reduction and the SUM reductions (the sums and the u32 histograms as one
u64 span, R37, or separately).  The per-rank tables come from the
oracle and the merge kernels are replaced by numpy doubles (there is no GPU
here); the merged table must equal the oracle's unsharded table bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fikit_synth as F

BIAS = np.int64(-(2**63))


class HostTable:
    """CPU tensors in libfikit's table layout (include/fikit.h fikit_table_t)."""

    def __init__(self, cap, span=True):
        self.capacity = cap
        self.kernel_id = torch.zeros(cap, dtype=torch.int64)
        self.task_id = torch.zeros(cap, dtype=torch.int32)
        # as fikit_table_carve lays them out: the SUM block, then the histograms (span=True)
        self._span = torch.zeros(cap * 36, dtype=torch.int64) if span else None
        self.sums = self._span[:cap * 4] if span else torch.zeros(cap * 4, dtype=torch.int64)
        self.hist = self._span[cap * 4:].view(torch.int32) if span else torch.zeros(cap * 64, dtype=torch.int32)
        self.ext = torch.zeros(cap * 4, dtype=torch.int64)
        self.mean = torch.zeros(cap * 2, dtype=torch.int64)
        self.n_rows_t = torch.zeros(1, dtype=torch.int32)

    def sum_span(self):
        return self._span

    def zero(self):
        for a in (self.kernel_id, self.task_id, self.sums, self.hist, self.ext, self.mean, self.n_rows_t):
            a.zero_()

    @staticmethod
    def from_oracle(tab, cap, span=True):
        t = HostTable(cap, span)
        n = tab.n_rows
        s = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64))
        t.kernel_id[:n] = s(tab.kernel_id[:n])
        t.task_id[:n] = torch.from_numpy(tab.task_id[:n].view(np.int32))
        t.sums.view(-1, 4)[:n] = s(np.stack([tab.dur_cnt, tab.dur_sum, tab.gap_cnt, tab.gap_sum], 1)[:n])
        t.hist.view(-1, 64)[:n] = torch.from_numpy(np.concatenate([tab.dur_hist, tab.gap_hist], 1)[:n].view(np.int32))
        t.ext.view(-1, 4)[:n] = s(np.stack([tab.dur_max, ~tab.dur_min, tab.gap_max, ~tab.gap_min], 1)[:n])
        t.mean.view(-1, 2)[:n] = s(np.stack([tab.dur_mean, tab.gap_mean], 1)[:n])
        t.n_rows_t[0] = n
        return t


class NumpyOps:
    """Host doubles of fikit_dict_union / table_remap / table_bias / table_means."""

    def dict_union(self, all_kid, all_task, n_all, P, Kmax, rank, ukid, utask, cap_out, un, l2u):
        keys = set()
        for r in range(P):
            for j in range(int(n_all[r])):
                keys.add((int(all_task[r, j]) & 0xFFFFFFFF, int(all_kid[r, j]) & 0xFFFFFFFFFFFFFFFF))
        u = sorted(keys)
        pos = {k: i for i, k in enumerate(u)}
        for i, (t, k) in enumerate(u):
            ukid[i] = int(np.uint64(k).view(np.int64))
            utask[i] = int(np.uint32(t).view(np.int32))
        un[0] = len(u)
        for j in range(int(n_all[rank])):
            l2u[j] = pos[(int(all_task[rank, j]) & 0xFFFFFFFF, int(all_kid[rank, j]) & 0xFFFFFFFFFFFFFFFF)]

    def table_remap(self, local, l2u, ukid, utask, un, dense):
        U = int(un[0])
        dense.n_rows_t[0] = U
        dense.kernel_id[:U] = ukid[:U]
        dense.task_id[:U] = utask[:U]
        for i in range(int(local.n_rows_t[0])):
            d = int(l2u[i])
            dense.sums.view(-1, 4)[d] = local.sums.view(-1, 4)[i]
            dense.hist.view(-1, 64)[d] = local.hist.view(-1, 64)[i]
            dense.ext.view(-1, 4)[d] = local.ext.view(-1, 4)[i]

    def table_bias(self, t):
        t.ext ^= torch.tensor(int(BIAS), dtype=torch.int64)

    def table_means(self, t):
        n = int(t.n_rows_t[0])
        h = t.hist.view(-1, 64)[:n].numpy().view(np.uint32).astype(np.uint64)
        s = t.sums.view(-1, 4)[:n].numpy().view(np.uint64)
        dc, gc = h[:, :32].sum(1), h[:, 32:].sum(1)
        t.sums.view(-1, 4)[:n, 0] = torch.from_numpy(dc.view(np.int64))
        t.sums.view(-1, 4)[:n, 2] = torch.from_numpy(gc.view(np.int64))

        def mean(sm, c):
            out = np.zeros_like(sm)
            nz = c > 0
            q, r = sm[nz] // c[nz], sm[nz] % c[nz]
            out[nz] = q + (2 * r >= c[nz])
            return out

        t.mean.view(-1, 2)[:n, 0] = torch.from_numpy(mean(s[:, 1], dc).view(np.int64))
        t.mean.view(-1, 2)[:n, 1] = torch.from_numpy(mean(s[:, 3], gc).view(np.int64))


def _worker(rank, world, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2311_10359_b200.dist import merge_tables, shard_range

        tr = F.random_trace(seed, 2500, n_tasks=3, n_ids=70, run_len_max=60, overlap_frac=0.05, big_frac=0.02)
        N = tr.records.shape[0]
        lo, hi = shard_range(N, rank, world)
        halo = tr.records[hi] if hi < N else None
        tab, st, _ = oracle.measure(tr.records[lo:hi], tr.names, tr.sigs, capacity=512, halo=halo)
        span = world != 3  # 3 ranks: separate SUM reductions of the sums and the histograms
        local = HostTable.from_oracle(tab, 512, span)
        dense = HostTable(512, span)
        merge_tables(local, dense, NumpyOps())
        full, _, _ = oracle.measure(tr.records, tr.names, tr.sigs, capacity=512)
        ref = HostTable.from_oracle(full, 512)
        n = full.n_rows
        ok = int(dense.n_rows_t[0]) == n
        for a in ("kernel_id", "task_id", "sums", "hist", "ext", "mean"):
            ok &= bool(torch.equal(getattr(dense, a), getattr(ref, a)))
        q.put((rank, ok, int(dense.n_rows_t[0]), n))
    finally:
        dist.destroy_process_group()


def dict_table(tab, keys, cap):
    """The host double of fikit_measure_dict + finalize: row j = dictionary key j, holding the
    shard table's statistics for that key (an all-zero row if the shard never saw it)."""
    t = HostTable(cap)
    pos = {k: j for j, k in enumerate(keys)}
    src = HostTable.from_oracle(tab, cap)
    for r in range(tab.n_rows):
        j = pos[(int(tab.task_id[r]), int(tab.kernel_id[r]))]
        t.sums.view(-1, 4)[j] = src.sums.view(-1, 4)[r]
        t.hist.view(-1, 64)[j] = src.hist.view(-1, 64)[r]
        t.ext.view(-1, 4)[j] = src.ext.view(-1, 4)[r]
    for j, (tk, kd) in enumerate(keys):
        t.kernel_id[j] = int(np.uint64(kd).view(np.int64))
        t.task_id[j] = int(np.uint32(tk).view(np.int32))
    t.n_rows_t[0] = len(keys)
    return t


def _worker_dict(rank, world, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2311_10359_b200.dist import merge_tables_dict, shard_range

        tr = F.random_trace(seed, 2500, n_tasks=3, n_ids=70, run_len_max=60, overlap_frac=0.05, big_frac=0.02)
        N = tr.records.shape[0]
        full, _, _ = oracle.measure(tr.records, tr.names, tr.sigs, capacity=512)
        # the dictionary: the whole trace's keys plus keys no rank sees (rows that stay empty)
        keys = sorted({(int(full.task_id[r]), int(full.kernel_id[r])) for r in range(full.n_rows)}
                      | {(7, 12345), (0, 1), (2, 2**64 - 1)})
        lo, hi = shard_range(N, rank, world)
        halo = tr.records[hi] if hi < N else None
        tab, st, _ = oracle.measure(tr.records[lo:hi], tr.names, tr.sigs, capacity=512, halo=halo)
        local = dict_table(tab, keys, 512)
        merge_tables_dict(local, NumpyOps())
        ref = dict_table(full, keys, 512)
        NumpyOps().table_means(ref)
        ok = int(local.n_rows_t[0]) == len(keys)
        for a in ("kernel_id", "task_id", "sums", "hist", "ext", "mean"):
            ok &= bool(torch.equal(getattr(local, a), getattr(ref, a)))
        # the rows the trace has equal the oracle's unsharded table
        pos = [keys.index((int(full.task_id[r]), int(full.kernel_id[r]))) for r in range(full.n_rows)]
        o = HostTable.from_oracle(full, 512)
        ok &= bool(torch.equal(local.sums.view(-1, 4)[pos], o.sums.view(-1, 4)[:full.n_rows]))
        ok &= bool(torch.equal(local.mean.view(-1, 2)[pos], o.mean.view(-1, 2)[:full.n_rows]))
        ok &= bool(torch.equal(local.ext.view(-1, 4)[pos], o.ext.view(-1, 4)[:full.n_rows]))
        q.put((rank, ok, int(local.n_rows_t[0]), len(keys)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,seed", [(2, 1), (3, 2)])
def test_merge_gloo(world, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
    for rank, ok, got_n, n in res:
        assert ok, f"rank {rank}: merged table differs from the unsharded oracle table ({got_n} vs {n} rows)"


@pytest.mark.parametrize("world,seed", [(2, 3), (3, 4)])
def test_merge_dict_gloo(world, seed):
    # dictionary-supplied mode (fikit_measure_dict): the merge is the two all-reduces alone
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dict, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
    for rank, ok, got_n, n in res:
        assert ok, f"rank {rank}: dictionary-mode merge differs from the oracle ({got_n} vs {n} rows)"


def test_shard_ranges_cover():
    from paper_2311_10359_b200.dist import scenario_shard, shard_range

    for n in (0, 1, 7, 100_000_000):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n and all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
    s = np.concatenate([scenario_shard(1000, r, 8) for r in range(8)])
    assert np.array_equal(np.sort(s), np.arange(1000))
