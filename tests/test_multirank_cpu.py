"""CPU, world_size 2 (gloo): the multi-GPU decomposition of the predictor.

Each rank takes the nnz-balanced row shard that the product's
spnnz_gpu_partition_rows assigns it (the same call spnnz_gpu_load makes),
computes its local FLOP / sampled FLOP / sampled NNZ for the sample draws
that fall in its rows (the CPU oracle stands in for the kernels here; the
GPU side of the same split is test_gpu_parity.py::test_detached_shards...),
all-reduces {F, f*, z*} once -- the one exchange the GPU path does with NCCL
-- and finishes with the product's scalar tail and ceil view.  Rank 0 checks
the concatenation against the single-process result, bit for bit.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(m, lo, hi):
    from paper_2207_13848_b200.spnnz import CsrMatrix
    rpt = m.rpt[lo:hi + 1] - m.rpt[lo]
    return CsrMatrix(hi - lo, m.cols, rpt, m.col[m.rpt[lo]:m.rpt[hi]])


def _worker(rank, world, port, cfg, results):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_2207_13848_b200 import capi, gen, spnnz
        O = Oracle(threads=1)
        a, b, seed, frac, cap = cfg
        a = gen.rmat(*a) if isinstance(a, tuple) else a
        b = a if b is None else b
        bounds = np.zeros(world + 1, np.int32)
        capi.check(capi.lib().spnnz_gpu_partition_rows(a.rpt.ctypes.data, a.rows, world,
                                                        bounds.ctypes.data))
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        mine = _slice(a, lo, hi)
        flop, F, mx = O.compute_flop(mine, b)
        rows, n, p = O.make_sample_plan(a.rows, seed, frac, cap)  # every rank draws all
        own = rows[(rows >= lo) & (rows < hi)] - lo                 # keeps its own draws
        fs = O.sampled_flop(flop, own) if len(own) else 0
        zs = O.sampled_symbolic(mine, b, flop, mx, own)[1] if len(own) else 0
        # the single exchange, as capi.cpp allreduce_totals does it: each rank
        # fills its own row of a world x 8 table (slots F, f*, z*, Z, max),
        # one SUM all-reduce gathers the rows, sums and the max are local
        table = torch.zeros(world, 8, dtype=torch.int64)
        table[rank, :5] = torch.tensor([F, fs, zs, 0, mx])
        dist.all_reduce(table)
        F, fs, zs = (int(x) for x in table[:, :3].sum(0))
        m = table[:, 4].max()
        pp = spnnz.predict_proposed(spnnz.SampleStats(fs, zs), F)
        z1 = spnnz.predict_reference(spnnz.SampleStats(fs, zs), spnnz.SamplePlan(p=p))
        ceil = O.predict_row_structure_ceil(flop, pp.predicted_cr)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, ceil, flop))
        if rank == 0:
            results.put((F, int(m), fs, zs, pp.predicted_cr, pp.z2_star, z1, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cap", [-1, 300])
def test_two_rank_prediction_equals_single(cap):
    import torch.multiprocessing as mp
    from oracle.pyoracle import Oracle
    from paper_2207_13848_b200 import gen
    cfg = ((14, 16 << 14, 0.57, 0.19, 0.19, 2), None, 7, 0.01, cap)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = mp.start_processes(_worker, args=(2, port, cfg, q), nprocs=2, join=False,
                               start_method="spawn")
    F, mx, fs, zs, cr, z2, z1, parts = q.get()  # before join: the result exceeds a pipe buffer
    while not procs.join():
        pass
    a = gen.rmat(*cfg[0])
    rep, flop, ceil, _ = Oracle().run_prediction(a, a, cfg[2], cfg[3], cap)
    assert (F, mx, fs, zs) == (rep.total_flop, rep.max_flop_row, rep.sampled_flop, rep.sampled_nnz)
    assert (cr, z2, z1) == (rep.predicted_cr, rep.z2_star, rep.z1_star)
    parts.sort(key=lambda x: x[0])
    assert parts[0][0] == 0 and parts[-1][1] == a.rows
    assert all(parts[i][1] == parts[i + 1][0] for i in range(len(parts) - 1))
    assert (np.concatenate([p[2] for p in parts]) == ceil).all()
    assert (np.concatenate([p[3] for p in parts]) == flop).all()
    # the shards are balanced on nnz + rows (within one row's worth)
    work = [int(a.rpt[p[1]] - a.rpt[p[0]]) + (p[1] - p[0]) for p in parts]
    assert abs(work[0] - work[1]) <= int(np.diff(a.rpt).max()) + 2


def flop_window(item_flop, rank, world):
    """The FLOP-balanced share of a sample list that rank counts when every
    rank holds all of A (C = A*A; csrc/flop.cu k_flop_window): items whose
    exclusive FLOP prefix lies in [T_r, T_{r+1}), T_r = floor(total r / W),
    the last rank taking the rest."""
    total = int(item_flop.sum())
    t = [(total // world) * r + (total % world) * r // world for r in range(world + 1)]
    pre = np.concatenate([[0], np.cumsum(item_flop)[:-1]]) if len(item_flop) else np.zeros(0, np.int64)
    lo = 0 if rank == 0 else int((pre < t[rank]).sum())
    hi = len(item_flop) if rank == world - 1 else int((pre < t[rank + 1]).sum())
    return lo, hi


def _worker_window(rank, world, port, cfg, results):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_2207_13848_b200 import capi, gen
        O = Oracle(threads=1)
        a = gen.rmat(*cfg[0])
        seed, frac, cap = cfg[1:]
        bounds = np.zeros(world + 1, np.int32)
        capi.check(capi.lib().spnnz_gpu_partition_rows(a.rpt.ctypes.data, a.rows, world,
                                                        bounds.ctypes.data))
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        F = int(O.compute_flop(_slice(a, lo, hi), a)[0].sum())      # local FLOP pass
        full, _, mx = O.compute_flop(a, a)                            # every rank holds all of A
        rows, n, p = O.make_sample_plan(a.rows, seed, frac, cap)
        item = full[rows.astype(np.int64)]                            # sampled rows' FLOP
        wlo, whi = flop_window(item, rank, world)
        mine = rows[wlo:whi]
        fs = int(item[wlo:whi].sum())
        zs = O.sampled_symbolic(a, a, full, mx, mine)[1] if len(mine) else 0
        t = torch.tensor([F, fs, zs], dtype=torch.int64)
        dist.all_reduce(t)
        parts = [None] * world
        dist.all_gather_object(parts, (wlo, whi, int(item[wlo:whi].sum())))
        if rank == 0:
            results.put((tuple(int(x) for x in t), parts, int(item.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_flop_balanced_sample_split_equals_single(world):
    """C = A*A on several ranks: the sample list is split into contiguous,
    FLOP-balanced windows; the windows tile the list and the all-reduced
    {F, f*, z*} equal the single-process values."""
    import torch.multiprocessing as mp
    from oracle.pyoracle import Oracle
    from paper_2207_13848_b200 import gen
    cfg = ((14, 16 << 14, 0.57, 0.19, 0.19, 2), 7, 0.02, -1)
    q = mp.get_context("spawn").SimpleQueue()
    procs = mp.start_processes(_worker_window, args=(world, _free_port(), cfg, q), nprocs=world,
                               join=False, start_method="spawn")
    tot, parts, fsum = q.get()
    while not procs.join():
        pass
    a = gen.rmat(*cfg[0])
    rep = Oracle().run_prediction(a, a, cfg[1], cfg[2], cfg[3])[0]
    assert tot == (rep.total_flop, rep.sampled_flop, rep.sampled_nnz)
    parts.sort()
    assert parts[0][0] == 0 and parts[-1][1] == rep.sample_num
    assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
    # balanced: every window within one row's FLOP of its share
    assert max(abs(f - fsum / world) for _, _, f in parts) <= rep.max_flop_row + 1
