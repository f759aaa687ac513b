"""Request-sharded data parallelism (BASELINE configs[3]) on CPU
ranks with gloo, world size 2: adapter key k is served by rank k mod N
(serving.owner_of / shard_keys), every rank builds its own page pool over
its shard only, routes the requests of the batch to their owners, and
applies the paged LoRA to its tokens (here the CPU oracle stands in for the
rank's GPU); the union of the ranks' outputs equals a single-process run,
and the step time is the max over ranks (the bench's reduction)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lora as OL
from paper_2512_20210_b200.lora import ModelShape
from paper_2512_20210_b200.memory import AllocStatus, PagePool
from paper_2512_20210_b200.serving import owner_of, shard_keys

SHAPE = ModelShape(2, (64, 64), (32, 32))
RANKS = [4, 8, 2, 6, 3, 5, 7, 1]
PAGE = 256
T = 40


def _data():
    rng = np.random.default_rng(11)
    images = []
    for a, r in enumerate(RANKS):
        n = SHAPE.adapter_bytes(r) // 2
        v = (rng.standard_normal(n) * 0.1).astype(np.float32)
        images.append(OL.f32_to_bf16_bits(v))
    ta = rng.integers(0, len(RANKS), size=T).astype(np.int32)
    x = OL.f32_to_bf16_bits(rng.standard_normal((T, 64)).astype(np.float32))
    y0 = OL.f32_to_bf16_bits(rng.standard_normal((T, 32)).astype(np.float32))
    return images, ta, x, y0


def _apply(keys, images, ta_global, x, y0, layer, proj):
    """One rank's pool (its keys only, churned) and its tokens' LoRA."""
    sizes = {a: SHAPE.adapter_bytes(RANKS[a]) for a in keys}
    pool = PagePool(PAGE, sum(-(-s // PAGE) for s in sizes.values()) * 2)
    for a in keys:
        assert pool.alloc(a, sizes[a]) == AllocStatus.ok
    for a in keys[::2]:
        pool.free(a)
    for a in keys[::2]:
        assert pool.alloc(a, sizes[a]) == AllocStatus.ok
    pool.check_invariants()
    arena = np.zeros(pool.total_pages() * PAGE, np.uint8)
    for a in keys:
        OL.scatter_pages(arena, PAGE, pool.table(a), images[a])
    mine = np.array([a in keys for a in ta_global])
    ta = np.where(mine, ta_global, -1).astype(np.int32)  # other ranks' tokens: no LoRA here
    y = y0.copy()
    m = OL.model(2, SHAPE.d_in, SHAPE.d_out, 2)
    OL.paged_lora_apply(m, arena, PAGE, {a: pool.table(a) for a in keys},
                        {a: RANKS[a] for a in keys}, layer, proj, x, y, ta)
    return y, mine, {a: pool.table(a) for a in keys}


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    images, ta, x, y0 = _data()
    keys = shard_keys(len(RANKS), rank, world)
    assert all(owner_of(a, world) == rank for a in keys)
    y, mine, tables = _apply(keys, images, ta, x, y0, 1, 0)
    # disjoint shards: each key is owned once, and every token has exactly one owner
    owned = torch.zeros(len(RANKS), dtype=torch.int32)
    owned[keys] = 1
    dist.all_reduce(owned)
    served = torch.from_numpy(mine.astype(np.int32))
    dist.all_reduce(served)
    # the max-over-ranks step time (bench.py: all_reduce MAX)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # gather every rank's rows of its own tokens
    rows = torch.from_numpy(np.where(mine[:, None], y, 0).astype(np.int32))
    dist.all_reduce(rows)
    if rank == 0:
        out.put((owned.tolist(), served.tolist(), t.item(), rows.numpy().astype(np.uint16)))
    dist.barrier()
    dist.destroy_process_group()


def test_request_sharding_world2_matches_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    owned, served, tmax, rows = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert owned == [1] * len(RANKS)
    assert served == [1] * T
    assert tmax == 2.0
    images, ta, x, y0 = _data()
    y_single, _, _ = _apply(list(range(len(RANKS))), images, ta, x, y0, 1, 0)
    assert np.array_equal(rows, y_single)  # bit-identical: same per-token arithmetic


@pytest.mark.gpu
def test_bench_multirank_path_on_one_gpu(tmp_path):
    """bench.py's N > 1 path (torchrun, one process per rank, barrier +
    max-over-ranks timing, whole-job value) end to end, with two ranks sharing
    the one GPU of this box over gloo (PLORA_BENCH_BACKEND; the numbers mean
    nothing here, the multi-GPU driver run uses NCCL on N GPUs)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PLORA_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--gpus", "2",
                          "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["config"]["parallelism"] == "request-sharded x2 (no collective)"
