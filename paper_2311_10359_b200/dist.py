"""Multi-GPU plumbing: record shards with a one-record halo, and
the merge of per-rank statistic tables into one identical table on every rank.

One process per GPU, torch.distributed (NCCL on GPUs; gloo works for the
host-side tests).  The arithmetic of the merge -- dictionary union, row
remap, order-bias of the MAX block, counts and means -- runs in libfikit's
kernels (`LibOps`); this module only sequences them around the collectives:

    all_gather(n_rows) ; all_gather(kernel_id) ; all_gather(task_id)
    fikit_dict_union -> identical sorted union on every rank + local->union map
    fikit_table_remap (dense table, zeroed) ; fikit_table_bias
    all_reduce SUM(sums u64 + hist u32 pairs as u64: one span, R37) ; all_reduce MAX(ext, biased)
    fikit_table_bias ; fikit_table_means

With a dictionary supplied to every rank (fikit_measure_dict: the rows are pre-assigned in
global canonical order), `merge_tables_dict` needs only the two all-reduces.

Integer sum / min / max are associative and commutative and the halo gives
every boundary gap exactly once, so the merged table equals the 1-GPU table
bit for bit.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous record shard [lo, hi) of rank `rank`; the halo is record hi (if hi < n)."""
    return n * rank // world, n * (rank + 1) // world


class LibOps:
    """The CUDA implementations (libfikit.so)."""

    def __init__(self, ws, stream=None):
        self.ws = ws
        self.stream = stream

    def dict_union(self, all_kid, all_task, n_all, P, Kmax, rank, ukid, utask, cap_out, un, l2u):
        from . import dict_union

        dict_union(all_kid, all_task, n_all, P, Kmax, rank, ukid, utask, cap_out, un, l2u, self.ws, self.stream)

    def table_remap(self, local, l2u, ukid, utask, un, dense):
        from . import table_remap

        table_remap(local, l2u, ukid, utask, un, dense, self.stream)

    def table_bias(self, t):
        from . import table_bias

        table_bias(t, self.stream)

    def table_means(self, t):
        from . import table_means

        table_means(t, self.stream)


def merge_tables(local, dense, ops, group=None):
    """local: this rank's finalized table; dense: a table of capacity >= the
    union (overwritten).  Returns the union size tensor (device, int32[1])."""
    import torch
    import torch.distributed as dist

    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = local.kernel_id.device
    cap = local.capacity
    # the gathered lists land rank after rank in one tensor each (no stacking copies)
    n_all = torch.empty(P, dtype=local.n_rows_t.dtype, device=dev)
    dist.all_gather_into_tensor(n_all, local.n_rows_t, group=group)
    all_kid = torch.empty(P * cap, dtype=local.kernel_id.dtype, device=dev)
    dist.all_gather_into_tensor(all_kid, local.kernel_id, group=group)
    all_task = torch.empty(P * cap, dtype=local.task_id.dtype, device=dev)
    dist.all_gather_into_tensor(all_task, local.task_id, group=group)
    all_kid, all_task = all_kid.view(P, cap), all_task.view(P, cap)
    ukid = torch.empty(dense.capacity, dtype=torch.int64, device=dev)
    utask = torch.empty(dense.capacity, dtype=torch.int32, device=dev)
    un = torch.zeros(1, dtype=torch.int32, device=dev)
    l2u = torch.empty(cap, dtype=torch.int32, device=dev)
    dense.zero()
    ops.dict_union(all_kid, all_task, n_all, P, cap, r, ukid, utask, dense.capacity, un, l2u)
    ops.table_remap(local, l2u, ukid, utask, un, dense)
    ops.table_bias(dense)
    span = dense.sum_span() if hasattr(dense, "sum_span") else None
    if span is not None:  # sums and hist adjacent: one SUM over both (R37)
        dist.all_reduce(span, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(dense.sums, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(dense.hist, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(dense.ext, op=dist.ReduceOp.MAX, group=group)
    ops.table_bias(dense)
    ops.table_means(dense)
    return un


def merge_tables_dict(local, ops, group=None):
    """In place: tables measured against ONE dictionary on every rank (fikit_measure_dict +
    fikit_table_finalize: row j = dictionary key j everywhere, SURVEY §8e "dictionary supplied",
    repeated services keep their IDs).  The rows already line up, so the merge is the two
    all-reduces alone -- no key gathers, no union, no remap:

        fikit_table_bias ; all_reduce SUM(sums u64 + hist u32 pairs: one span, R37) ;
        all_reduce MAX(ext, biased) ; fikit_table_bias ; fikit_table_means

    Bytes per rank: 288 per row (SUM span) + 32 per row (MAX block)."""
    import torch.distributed as dist

    ops.table_bias(local)
    span = local.sum_span() if hasattr(local, "sum_span") else None
    if span is not None:
        dist.all_reduce(span, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(local.sums, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(local.hist, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(local.ext, op=dist.ReduceOp.MAX, group=group)
    ops.table_bias(local)
    ops.table_means(local)
    return local


def scenario_shard(S: int, rank: int, world: int):
    """Scenario s -> rank s mod world (cost-interleaved)."""
    import numpy as np

    return np.arange(rank, S, world, dtype=np.int64)
