"""COLS mode: right-hand sides are independent, F-hat is
replicated, no data-path collective.  What bench.py does across ranks --
the per-rank sun azimuth offsets and RHS seeds, and the timing reductions
(max of the time over ranks, sum of the work) -- checked with a world-size-2
gloo job on CPU."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t_ms = [12.5, 20.0][rank]
    work = [100, 140][rank]
    t, w = bench.reduce_time_work(t_ms, work, dist, torch.device("cpu"))
    t2, w2 = bench.reduce_time_work(t_ms, work, dist, torch.device("cpu"), sum_work=False)
    out[rank] = (t, w, t2, w2)
    dist.barrier()
    dist.destroy_process_group()


def test_cols_reductions_max_time_sum_work():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        t, w, t2, w2 = out[r]
        assert t == 20.0 and w == 240.0          # COLS: max time over ranks, summed work
        assert t2 == 20.0 and w2 == [100, 140][r]  # ROWS: one shared solve, work not summed


def test_cols_rank_offsets_partition_the_suns():
    """cfg2 COLS: rank g's 64 suns are offset by 2 pi g / (64 G) in azimuth, so
    the G batches interleave without duplicates; terrain RHS seeds differ."""
    import scenegen as sg
    G = 4
    phis = []
    for g in range(G):
        phase = 2 * math.pi / bench.NRHS * g / G
        s = sg.sun_dirs(bench.ELEV, bench.NRHS, phase)
        phis.append(np.arctan2(s[:, 1], s[:, 0]) % (2 * math.pi))
    allp = np.sort(np.concatenate(phis))
    d = np.diff(np.concatenate([allp, [allp[0] + 2 * math.pi]]))
    assert np.allclose(d, 2 * math.pi / (bench.NRHS * G))
    X0, X1 = sg.random_rhs(100, 2, seed=3), sg.random_rhs(100, 2, seed=4)
    assert not np.allclose(X0, X1)
