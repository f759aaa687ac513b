"""GPU parity of the paged LoRA forward op (BGMV decode path) against the CPU
oracle (oracle/lora_oracle.c) on identical inputs, page tables and adapter
assignment; page tables come from the bit-exact pool (pinned to the reference
PagePool in test_pagepool.py and here against tests/golden)."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from lora_harness import BGMV_BF16_LAUNCHES, TOL_BF16, TOL_F32, Setup, rel_err, to_np_bits
from oracle import lora as OL
from paper_2512_20210_b200 import (AllocStatus, PagePool, ValidationError, synth)
from paper_2512_20210_b200.lora import (AdapterStore, BatchPlan, ModelShape, bgmv,
                                        kernel_launch_count)

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _run(setup, layer, proj, ta, scale=1.0, salt=0, x_pad=0, y_pad=0):
    cfg = setup.cfg
    T = len(ta)
    din, dout = cfg.shape.d_in[proj], cfg.shape.d_out[proj]
    x = synth.activations(T, din + x_pad, cfg.shape.dtype, "x", salt=salt)[:, :din]
    y0 = synth.activations(T, dout + y_pad, cfg.shape.dtype, "y", salt=salt)[:, :dout]
    xd = torch.empty(T, din + x_pad, dtype=cfg.shape.dtype, device="cuda")[:, :din]
    yd = torch.empty(T, dout + y_pad, dtype=cfg.shape.dtype, device="cuda")[:, :dout]
    xd.copy_(x)
    yd.copy_(y0)
    plan = BatchPlan(setup.store, ta)
    bgmv(plan, layer, proj, xd, yd, scale)
    torch.cuda.synchronize()
    ref = setup.oracle(layer, proj, x.contiguous(), y0.contiguous(), ta, scale=scale)
    return yd, ref


def test_store_readback_bit_exact(cuda):
    for mode in (0, 1):  # copy engines, SM page-scatter kernel over mapped pinned memory
        cfg = synth.cfg1(n_layers=2)
        s = Setup(cfg, copy_mode=mode)
        for a in range(cfg.n_adapters):
            got = s.store.read_pages(a, cfg.shape.adapter_bytes(cfg.ranks[a]))
            assert torch.equal(got, s.images[a].view(torch.uint8)), (mode, a)


def test_small_golden_vectors(cuda):
    """tests/golden/lora_small.npz: odd ranks, 64-byte pages, -1 tokens."""
    z = np.load(os.path.join(GOLDEN, "lora_small.npz"))
    for dt, dtype, tol in (("bf16", torch.bfloat16, TOL_BF16), ("f32", torch.float32, TOL_F32)):
        ranks = [int(r) for r in z[f"{dt}_ranks"]]
        page, total = (int(v) for v in z[f"{dt}_page"])
        shape = ModelShape(2, (64, 128), (64, 32), dtype)
        pool = PagePool(page, total)
        sizes = [shape.adapter_bytes(r) for r in ranks]
        for a, sz in enumerate(sizes):
            assert pool.alloc(a, sz) == AllocStatus.ok
        for a in range(0, len(ranks), 2):
            pool.free(a)
        for a in range(0, len(ranks), 2):
            assert pool.alloc(a, sizes[a]) == AllocStatus.ok
        store = AdapterStore(pool, shape, len(ranks))
        for a, r in enumerate(ranks):
            assert pool.table(a) == list(z[f"{dt}_table{a}"])  # reference tables
            store.register(a, r)
            img = torch.from_numpy(z[f"{dt}_img{a}"].view(np.uint8).copy())
            store.write_pages(a, img)
            store.publish(a)
        ta = z[f"{dt}_tokens"]
        plan = BatchPlan(store, ta)
        for layer in range(2):
            for proj in range(2):
                x = z[f"{dt}_x_{layer}_{proj}"]
                y0 = z[f"{dt}_y0_{layer}_{proj}"]
                tx = torch.from_numpy(x.view(np.int16) if dt == "bf16" else x)
                ty = torch.from_numpy(y0.view(np.int16).copy() if dt == "bf16" else y0.copy())
                if dt == "bf16":
                    tx, ty = tx.view(torch.bfloat16), ty.view(torch.bfloat16)
                xd, yd = tx.cuda(), ty.cuda()
                bgmv(plan, layer, proj, xd, yd, 0.5)
                torch.cuda.synchronize()
                err = rel_err(yd, z[f"{dt}_y_{layer}_{proj}_v0"])
                assert err <= tol, (dt, layer, proj, err)
                # rows of tokens with no adapter are untouched bit for bit
                none = ta < 0
                assert np.array_equal(to_np_bits(yd)[none], y0[none])


def test_cfg1_parity_and_checksum(cuda):
    """BASELINE config 1 at full size (32 layers), four (layer, proj) calls; the
    oracle itself is pinned by tests/golden/cfg1_checksums.json."""
    with open(os.path.join(GOLDEN, "cfg1_checksums.json")) as f:
        g = json.load(f)
    cfg = synth.cfg1()
    s = Setup(cfg)
    tables = np.concatenate([np.asarray(s.pool.table(a), np.uint32) for a in range(16)])
    assert hashlib.sha256(tables.tobytes()).hexdigest() == g["tables_sha256"]
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    for call in g["calls"]:
        layer, proj = call["layer"], call["proj"]
        yd, ref = _run(s, layer, proj, ta, salt=layer * 2 + proj)
        assert hashlib.sha256(ref.tobytes()).hexdigest() == call["y_sha256"]
        err = rel_err(yd, ref)
        assert err <= TOL_BF16, (layer, proj, err)


@pytest.mark.parametrize("page_bytes", [2048, 2 << 20])
def test_cfg2_per_call_parity(cuda, page_bytes):
    """BASELINE config 2 call shape (256 tokens, 128 adapters, r in {8..64});
    two layers instead of 32 — the kernel sees identical per-call work."""
    cfg = synth.cfg2(n_layers=2, page_bytes=page_bytes)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    for layer, proj in ((0, 0), (1, 1)):
        yd, ref = _run(s, layer, proj, ta, salt=7 + layer)
        err = rel_err(yd, ref)
        assert err <= TOL_BF16, (page_bytes, layer, proj, err)


def test_fp32_accumulate_mode(cuda):
    cfg = synth.DecodeConfig("f32", ModelShape(2, (512, 256), (256, 1024), torch.float32),
                             [4, 8, 16, 32, 64, 128, 3, 7], 3, 1024)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    for layer, proj in ((0, 0), (1, 1), (1, 0)):
        yd, ref = _run(s, layer, proj, ta, scale=0.75, salt=layer)
        err = rel_err(yd, ref)
        assert err <= TOL_F32, (layer, proj, err)


def test_edge_cases(cuda):
    shape = ModelShape(3, (64, 256), (128, 64), torch.bfloat16)
    ranks = [1, 5, 12, 33, 100, 128, 200, 2]
    cfg = synth.DecodeConfig("edge", shape, ranks, 1, 16)  # 16-byte pages
    s = Setup(cfg)
    # many tokens for one adapter (> token chunk), unordered, with -1s and repeats
    rng = np.random.default_rng(3)
    ta = rng.integers(-1, len(ranks), size=71).astype(np.int32)
    ta[:20] = 4
    for layer, proj in ((0, 0), (2, 1), (1, 1)):
        yd, ref = _run(s, layer, proj, ta, scale=-1.25, salt=layer, x_pad=24, y_pad=8)
        assert rel_err(yd, ref) <= TOL_BF16
    # single token
    yd, ref = _run(s, 1, 0, np.asarray([6], np.int32))
    assert rel_err(yd, ref) <= TOL_BF16
    # empty batch and all-(-1) batch leave y untouched
    for ta in (np.zeros(0, np.int32), np.full(9, -1, np.int32)):
        plan = BatchPlan(s.store, ta)
        y = torch.randn(max(len(ta), 1), 128, device="cuda").to(torch.bfloat16)
        y0 = y.clone()
        bgmv(plan, 0, 0, torch.randn(max(len(ta), 1), 64, device="cuda").to(torch.bfloat16), y)
        torch.cuda.synchronize()
        assert torch.equal(y, y0)


@pytest.mark.parametrize("page_bytes", [256, 512])
def test_small_pages_wide_rows(cuda, page_bytes):
    """Llama-7B row widths on pages smaller than a CTA's 2 KiB row slice (the
    generic piece path; 72 / 40 page pieces per 8 A rows, past the 32 the
    lookahead covers: the producer's synchronous small-page loop), ranks 3..64
    with partial chunks."""
    shape = ModelShape(2, (4096, 4096), (4096, 4096), torch.bfloat16)
    ranks = [8, 16, 64, 3, 13]
    cfg = synth.DecodeConfig("smallpage", shape, ranks, 2, page_bytes)
    s = Setup(cfg)
    ta = synth.token_assignment(len(ranks), 2)
    for layer, proj in ((0, 1), (1, 0)):
        yd, ref = _run(s, layer, proj, ta, scale=0.5, salt=layer)
        assert rel_err(yd, ref) <= TOL_BF16, (page_bytes, layer, proj)


def test_errors_are_loud(cuda):
    cfg = synth.cfg1(n_layers=1)
    s = Setup(cfg)
    s.store.retire(3)
    with pytest.raises(ValidationError, match="not resident"):
        BatchPlan(s.store, [0, 3])
    plan = BatchPlan(s.store, [0, 1])
    x = torch.zeros(2, 4096, device="cuda", dtype=torch.bfloat16)
    y = torch.zeros(2, 4096, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValidationError):
        bgmv(plan, 5, 0, x, y)  # layer out of range
    with pytest.raises(ValidationError):
        bgmv(plan, 0, 0, x.float(), y)  # dtype mismatch
    with pytest.raises(ValidationError):
        bgmv(plan, 0, 0, x[:, :2048], y)  # width mismatch


def test_compaction_relocations_preserve_results(cuda):
    cfg = synth.cfg1(n_layers=2)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    before, _ = _run(s, 1, 1, ta, salt=3)
    # evict a few adapters, compact, move pages on device, republish
    for a in (1, 4, 9):
        s.store.retire(a)
        s.pool.free(a)
    moved = s.pool.compact()
    assert moved > 0
    relocs = s.pool.last_relocations()
    s.store.apply_relocations(relocs)
    s.pool.check_invariants()
    live = [a for a in range(cfg.n_adapters) if a not in (1, 4, 9)]
    ta2 = np.asarray([a if a in live else -1 for a in ta], np.int32)
    x = synth.activations(len(ta), 4096, cfg.shape.dtype, "x", salt=3).cuda()
    y = synth.activations(len(ta), 4096, cfg.shape.dtype, "y", salt=3).cuda()
    bgmv(BatchPlan(s.store, ta2), 1, 1, x, y)
    torch.cuda.synchronize()
    keep = ta2 >= 0
    assert torch.equal(y[torch.from_numpy(keep).cuda()], before[torch.from_numpy(keep).cuda()])
    for a in live:  # device bytes followed their pages
        got = s.store.read_pages(a, cfg.shape.adapter_bytes(cfg.ranks[a]))
        assert torch.equal(got, s.images[a].view(torch.uint8))


def test_graph_capture_and_determinism(cuda):
    cfg = synth.cfg2(n_layers=2)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    plan = BatchPlan(s.store, ta)
    x = synth.activations(len(ta), 4096, cfg.shape.dtype, "x").cuda()
    y0 = synth.activations(len(ta), 4096, cfg.shape.dtype, "y").cuda()
    y_eager = y0.clone()
    for layer in range(2):
        for proj in range(2):
            bgmv(plan, layer, proj, x, y_eager)
    torch.cuda.synchronize()
    y_graph = y0.clone()
    stream = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for layer in range(2):
                for proj in range(2):
                    bgmv(plan, layer, proj, x, y_graph, stream=stream.cuda_stream)
    y_graph.copy_(y0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_graph, y_eager)  # same unit decomposition -> bit-identical
    y_graph.copy_(y0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_graph, y_eager)


def test_linearity_property_full_cfg2(cuda):
    """Size-independent property at BASELINE config 2 full size (32 layers):
    zero x leaves y bit-identical; Δy(scale=2) ≈ 2·Δy(scale=1)."""
    cfg = synth.cfg2()
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        img = synth.adapter_image(cfg.shape, r, a, device="cuda")
        store.write_pages(a, img.view(torch.uint8).cpu())
        store.publish(a)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    plan = BatchPlan(store, ta)
    n0 = kernel_launch_count()
    x = torch.zeros(256, 4096, device="cuda", dtype=torch.bfloat16)
    y = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
    y0 = y.clone()
    bgmv(plan, 31, 1, x, y)
    torch.cuda.synchronize()
    assert torch.equal(y, y0)
    x = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
    yz = torch.zeros(256, 4096, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    y1, y2 = yz.clone(), yz.clone()
    bgmv(plan, 20, 0, x, y1, 1.0)
    bgmv(plan, 20, 0, x, y2, 2.0)
    torch.cuda.synchronize()
    d = (y2.float() - 2 * y1.float()).abs().max().item()
    assert d <= 2e-2 * y2.float().abs().max().item()
    assert kernel_launch_count() - n0 == 3 * BGMV_BF16_LAUNCHES  # shrink + expand per call


def test_ring_stress_random_ranks(cuda):
    """Many units per CTA (every ring slot, wrap-around phases), ranks 1..256,
    1..5 tokens per adapter, two projection shapes."""
    rng = np.random.default_rng(11)
    shape = ModelShape(1, (4096, 2048), (1024, 4096), torch.bfloat16)
    ranks = [int(r) for r in rng.integers(1, 257, size=300)]
    cfg = synth.DecodeConfig("stress", shape, ranks, 1, 2048)
    s = Setup(cfg)
    ta = np.concatenate([np.full(int(rng.integers(1, 6)), a, np.int32) for a in range(300)])
    rng.shuffle(ta)
    for proj in (0, 1):
        yd, ref = _run(s, 0, proj, ta, scale=0.5, salt=proj)
        assert rel_err(yd, ref) <= TOL_BF16, proj


@pytest.mark.parametrize("page_bytes", [2048, 2097152])
def test_bgmv_layer_fused_equals_per_projection(cuda, page_bytes):
    """plora_bgmv_layer (q and v of a layer in one launch) computes exactly
    what two plora_bgmv calls do: same chunks, same partial sums, same order."""
    from paper_2512_20210_b200.lora import bgmv_layer
    cfg = synth.cfg2(n_layers=2, page_bytes=page_bytes)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    x = synth.activations(T, 4096, torch.bfloat16, "x").cuda()
    y0 = [synth.activations(T, 4096, torch.bfloat16, "y", salt=p).cuda() for p in range(2)]
    plan = BatchPlan(s.store, ta)
    sep = [y.clone() for y in y0]
    for p in range(2):
        bgmv(plan, 1, p, x, sep[p], 0.75)
    fused = [y.clone() for y in y0]
    n0 = kernel_launch_count()
    bgmv_layer(plan, 1, x, fused, 0.75)
    torch.cuda.synchronize()
    assert kernel_launch_count() - n0 == BGMV_BF16_LAUNCHES  # both projections in one shrink + one expand
    for p in range(2):
        assert torch.equal(fused[p], sep[p])
    ref = s.oracle(1, 1, x.cpu(), y0[1].cpu(), ta, scale=0.75)
    assert rel_err(fused[1], ref) <= TOL_BF16


@pytest.mark.parametrize("page_bytes", [2048, 256])
def test_bgmv_layers_multi_layer_launch_bit_identical(cuda, page_bytes):
    """plora_bgmv_layers (several layers per launch) computes what per-layer
    bgmv_layer calls do, on strided per-layer views, and matches the oracle:
    the default warp-item op (one shrink + one expand launch for all layers;
    within one bf16 ulp of the per-layer calls, whose widest adapters' expand
    items are split pairs), the cluster kernel (impl 2: its chunk lists
    repeated per layer; bit for bit) and the round-2 hybrid pair (impl 3:
    clusters + a streaming share)."""
    from paper_2512_20210_b200.lora import bgmv_layer, bgmv_layers
    from paper_2512_20210_b200 import _native as N
    cfg = synth.cfg2(n_layers=4, page_bytes=page_bytes)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(3, T, 4096, device="cuda", generator=g).to(torch.bfloat16)
    y0 = torch.randn(3, 2, T, 4096, device="cuda", generator=g).to(torch.bfloat16)

    def per_layer(plan):
        ref = y0.clone()
        for i in range(3):
            bgmv_layer(plan, 1 + i, x[i], [ref[i, 0], ref[i, 1]], 0.5)
        return ref

    outs = {}
    for impl, launches in ((0, BGMV_BF16_LAUNCHES), (2, 1), (3, 2)):
        N.check(N.lib().plora_debug_set_bgmv_impl(impl))
        try:
            plan = BatchPlan(s.store, ta)
            got = y0.clone()
            n0 = kernel_launch_count()
            bgmv_layers(plan, 1, x, [got[:, 0], got[:, 1]], 0.5)
            torch.cuda.synchronize()
            assert kernel_launch_count() - n0 == launches, impl
            if impl == 2:
                assert torch.equal(got, per_layer(plan)), impl
            elif impl == 0:
                # single-layer calls split the rank-64 adapters' expand items over two warps (another
                # fp32 summation order of their rows): at most one bf16 ulp of y apart, mostly identical
                ref = per_layer(plan)
                d = (got.float() - ref.float()).abs()
                # (<= one ulp of y, or of the delta's fp32 rounding where y0 + delta cancels)
                assert (d <= ref.float().abs() * 2.0 ** -7 + ref.float().abs().max() * 2.0 ** -12).all(), impl
                assert (d > 0).float().mean().item() < 0.05, impl
            again = y0.clone()
            bgmv_layers(plan, 1, x, [again[:, 0], again[:, 1]], 0.5)
            torch.cuda.synchronize()
            assert torch.equal(got, again), impl  # deterministic
            outs[impl] = got
        finally:
            N.check(N.lib().plora_debug_set_bgmv_impl(0))
    for i in range(3):
        for p in range(2):
            o = s.oracle(1 + i, p, x[i].cpu(), y0[i, p].cpu(), ta, scale=0.5)
            for impl, got in outs.items():
                assert rel_err(got[i, p], o) <= TOL_BF16, (impl, i, p)


@pytest.mark.parametrize("tokens_per_adapter", [2, 6])
def test_streaming_kernel_parity(cuda, tokens_per_adapter):
    """The alternative streaming decode kernel (bgmv_stream.cu, selected with
    plora_debug_set_bgmv_impl(1)): per-call, per-layer and multi-layer
    launches against the oracle, 4- and 8-token jobs."""
    from paper_2512_20210_b200 import _native as N
    from paper_2512_20210_b200.lora import bgmv_layer, bgmv_layers
    cfg = synth.cfg2(n_layers=3)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, tokens_per_adapter)
    T = len(ta)
    x = synth.activations(T, 4096, torch.bfloat16, "x", salt=4)
    y0 = synth.activations(T, 4096, torch.bfloat16, "y", salt=4)
    N.check(N.lib().plora_debug_set_bgmv_impl(1))
    try:
        plan = BatchPlan(s.store, ta)
        yd = y0.cuda()
        bgmv(plan, 2, 1, x.cuda(), yd, 0.5)
        torch.cuda.synchronize()
        assert rel_err(yd, s.oracle(2, 1, x, y0, ta, scale=0.5)) <= TOL_BF16
        xl = x.cuda().unsqueeze(0).repeat(2, 1, 1)
        yl = y0.cuda().view(1, 1, T, 4096).repeat(2, 2, 1, 1)
        ref = yl.clone()
        for i in range(2):
            bgmv_layer(plan, 1 + i, xl[i], [ref[i, 0], ref[i, 1]])
        bgmv_layers(plan, 1, xl, [yl[:, 0], yl[:, 1]])
        torch.cuda.synchronize()
        assert torch.equal(yl, ref)
        assert rel_err(yl[1, 0], s.oracle(2, 0, x, y0, ta)) <= TOL_BF16
    finally:
        N.check(N.lib().plora_debug_set_bgmv_impl(0))


@pytest.mark.parametrize("page_bytes", [256, 2048])
def test_warp_items_token_counts_and_odd_widths(cuda, page_bytes):
    """The default warp-item op (bgmv_warp.cu): adapters with 1..7 tokens
    (jobs of 1-4 tokens: the four shrink / expand bodies, and a 5-7-token
    adapter split evenly over two jobs), widths that are not multiples of 256
    (partial 512-byte chunks) or of the expand block, ranks 1..80, 256-byte
    pages (page entries by table loads) and 2 KiB pages (by shuffle); -1
    tokens untouched; bgmv and bgmv_layer agree bit for bit."""
    from paper_2512_20210_b200.lora import bgmv_layer
    shape = ModelShape(3, (1000, 1000), (520, 1048), torch.bfloat16)
    ranks = [1, 5, 16, 33, 64, 80, 8, 24]
    s = Setup(synth.DecodeConfig("warp_edge", shape, ranks, 1, page_bytes))
    rng = np.random.default_rng(7)
    ta = np.concatenate([np.full(1 + a % 7, a, np.int32) for a in range(len(ranks))] + [np.full(5, -1, np.int32)])
    rng.shuffle(ta)
    T = len(ta)
    x = synth.activations(T, 1000, torch.bfloat16, "x", salt=3)
    y0 = [synth.activations(T, shape.d_out[p], torch.bfloat16, "y", salt=3 + p) for p in range(2)]
    plan = BatchPlan(s.store, ta)
    ys = [y.cuda() for y in y0]
    bgmv_layer(plan, 2, x.cuda(), ys, 0.5)
    sep = [y.cuda() for y in y0]
    for p in range(2):
        bgmv(plan, 2, p, x.cuda(), sep[p], 0.5)
    torch.cuda.synchronize()
    for p in range(2):
        assert torch.equal(ys[p], sep[p]), p
        ref = s.oracle(2, p, x, y0[p], ta, scale=0.5)
        assert rel_err(ys[p], ref) <= TOL_BF16, p
        none = ta < 0
        assert np.array_equal(to_np_bits(ys[p])[none], to_np_bits(y0[p])[none])
