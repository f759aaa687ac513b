"""Tensor-parallel orchestration (BASELINE cfg5) on CPU ranks with gloo,
world size 2: the real TensorParallelLoRA (buffer shapes, rank-major
all-gather, shard bookkeeping) with the two kernel halves replaced by a
numpy restatement of their C-ABI contract (include/plora.h, tensor-parallel
decode), checked against the dense y += (x·Aᵀ)·Bᵀ of PAPER.md:64-69."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_20210_b200.tp import TensorParallelLoRA

RANKS = [4, 8, 2, 6]          # divisible by the TP size
D_IN, D_OUT, T = 16, 12, 7
TA = np.array([0, 1, 2, 3, 0, -1, 1], dtype=np.int32)


def _weights():
    rng = np.random.default_rng(7)
    A = [rng.standard_normal((r, D_IN)) for r in RANKS]
    B = [rng.standard_normal((D_OUT, r)) for r in RANKS]
    x = rng.standard_normal((T, D_IN))
    y0 = rng.standard_normal((T, D_OUT))
    return A, B, x, y0


def _dense(A, B, x, y0, scale):
    y = y0.copy()
    for t, a in enumerate(TA):
        if a >= 0:
            y[t] += scale * (x[t] @ A[a].T) @ B[a].T
    return y


def _emulated_halves(A, B):
    def shrink(plan, layer, proj, tp_rank, tp_size, x, v_part):
        xv = x.numpy()
        for t, a in enumerate(TA):
            if a < 0:
                continue
            rs = RANKS[a] // tp_size
            for j in range(rs):
                v_part[t, j] = float(xv[t] @ A[a][tp_rank * rs + j])
        return v_part

    def expand(plan, layer, proj, tp_rank, tp_size, vg, y_shard, scale):
        ncols = D_OUT // tp_size
        c0 = tp_rank * ncols
        for t, a in enumerate(TA):
            if a < 0:
                continue
            r, rs = RANKS[a], RANKS[a] // tp_size
            v = np.array([vg[jj // rs, t, jj % rs].item() for jj in range(r)])
            y_shard[t] += torch.from_numpy(scale * (B[a][c0:c0 + ncols] @ v))
        return y_shard

    return shrink, expand


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B, x, y0 = _weights()
        shrink, expand = _emulated_halves(A, B)
        tp = TensorParallelLoRA(None, rank, world, group=None, shrink=shrink, expand=expand,
                                shard_rows=max(RANKS) // world, n_tokens=T,
                                device=torch.device("cpu"))
        ncols = D_OUT // world
        y_shard = torch.from_numpy(y0[:, rank * ncols:(rank + 1) * ncols].copy())
        tp(0, 0, torch.from_numpy(x), y_shard, scale=0.5)
        ref = _dense(A, B, x, y0, 0.5)[:, rank * ncols:(rank + 1) * ncols]
        q.put((rank, float(np.abs(y_shard.numpy() - ref).max())))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tp_world2_gloo_matches_dense():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    errs = dict(q.get() for _ in range(2))
    assert set(errs) == {0, 1}
    assert max(errs.values()) < 1e-5, errs  # v travels in fp32


def test_tp_validates_rank_arguments():
    with pytest.raises(Exception):
        TensorParallelLoRA(None, 2, 2, shard_rows=1, n_tokens=1, device=torch.device("cpu"))
