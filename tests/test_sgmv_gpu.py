"""GPU parity of the tcgen05 prefill path (SGMV) against the CPU oracle in its
SGMV rounding mode (v = x·Aᵀ rounded to bf16 before the expand), plus
full-size BASELINE config-3 properties."""
import numpy as np
import pytest
import torch

from lora_harness import TOL_BF16, Setup, rel_err, to_np_bits
from paper_2512_20210_b200 import synth
from paper_2512_20210_b200.lora import (AdapterStore, BatchPlan, ModelShape, bgmv, sgmv,
                                        kernel_launch_count, sgmv_layer)

pytestmark = pytest.mark.gpu


def _sgmv_vs_oracle(s, ta, layer, proj, scale=1.0, salt=0):
    shape = s.cfg.shape
    T = len(ta)
    x = synth.activations(T, shape.d_in[proj], shape.dtype, "x", salt=salt)
    y0 = synth.activations(T, shape.d_out[proj], shape.dtype, "y", salt=salt)
    xd, yd = x.cuda(), y0.cuda()
    plan = BatchPlan(s.store, ta)
    n0 = kernel_launch_count()
    sgmv(plan, layer, proj, xd, yd, scale)
    torch.cuda.synchronize()
    ranks = [s.store.rank(a) for a in set(int(v) for v in ta) if a >= 0]
    tc = (shape.dtype == torch.bfloat16 and max(ranks, default=0) <= 128
          and shape.d_in[proj] % 64 == 0 and shape.d_out[proj] % 128 == 0)
    # tcgen05 shrink + split reduction + expand; else the BGMV path
    # (shrink + expand launches, bf16 and fp32 alike)
    expect = 3 if tc else 2
    assert kernel_launch_count() - n0 == expect
    ref = s.oracle(layer, proj, x, y0, ta, scale=scale, v_bf16=shape.dtype == torch.bfloat16)
    return yd, ref, y0


def test_sgmv_mixed_ranks_partial_tiles(cuda):
    """Runs of 1..300 tokens, ranks 3..128 (padded to 16 in smem), -1 gaps."""
    shape = ModelShape(2, (4096, 1024), (4096, 2048), torch.bfloat16)
    ranks = [16, 64, 128, 8, 3, 100, 32, 1]
    cfg = synth.DecodeConfig("sgmv", shape, ranks, 1, 2048)
    s = Setup(cfg)
    runs = [(0, 300), (1, 130), (-1, 5), (2, 128), (3, 1), (4, 77), (5, 129), (-1, 2), (6, 64),
            (7, 9), (2, 40)]
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in runs])
    for layer, proj in ((0, 0), (1, 1)):
        yd, ref, y0 = _sgmv_vs_oracle(s, ta, layer, proj, scale=0.5, salt=layer)
        assert rel_err(yd, ref) <= TOL_BF16, (layer, proj)
        none = ta < 0
        assert np.array_equal(to_np_bits(yd)[none], to_np_bits(y0)[none])


def test_sgmv_cfg3_shape_parity(cuda):
    """BASELINE config 3 call shape at reduced token count (6 segments × 512)."""
    cfg = synth.cfg3(n_layers=2, n_segments=6)
    s = Setup(cfg)
    ta = synth.segment_assignment(6, 512)
    yd, ref, _ = _sgmv_vs_oracle(s, ta, 1, 0, salt=11)
    assert rel_err(yd, ref) <= TOL_BF16


def test_sgmv_full_cfg3_properties(cuda):
    """Full BASELINE config 3 (32 × 512 tokens, r in {16,64,128}, 32 layers):
    SGMV agrees with the BGMV path (independent arithmetic: CUDA cores, fp32
    intermediate) within the bf16 tolerance; zero x leaves y untouched."""
    cfg = synth.cfg3()
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    ta = synth.segment_assignment(32, 512)
    plan = BatchPlan(store, ta)
    x = torch.randn(len(ta), 4096, device="cuda").to(torch.bfloat16)
    y0 = torch.randn(len(ta), 4096, device="cuda").to(torch.bfloat16)
    ys, yb = y0.clone(), y0.clone()
    sgmv(plan, 30, 1, x, ys)
    bgmv(plan, 30, 1, x, yb)
    torch.cuda.synchronize()
    err = (ys.float() - yb.float()).abs().max().item() / yb.float().abs().max().item()
    assert err <= TOL_BF16, err
    yz = y0.clone()
    sgmv(plan, 3, 0, torch.zeros_like(x), yz)
    torch.cuda.synchronize()
    assert torch.equal(yz, y0)


def test_sgmv_fp32_store_routes_to_exact_path(cuda):
    shape = ModelShape(1, (256,), (512,), torch.float32)
    cfg = synth.DecodeConfig("f32", shape, [16, 64], 40, 1024)
    s = Setup(cfg)
    ta = np.repeat(np.arange(2, dtype=np.int32), 40)
    yd, ref, _ = _sgmv_vs_oracle(s, ta, 0, 0)
    assert rel_err(yd, ref) <= 1e-5


def test_sgmv_layer_matches_oracle_per_projection(cuda):
    """plora_sgmv_layer (both projections from one x chunk, one expand launch)
    against the oracle for each projection: runs with partial tiles and -1
    gaps, ranks 1..128."""
    shape = ModelShape(2, (4096, 4096), (2048, 2048), torch.bfloat16)
    ranks = [16, 64, 128, 8, 3, 100, 32, 1]
    cfg = synth.DecodeConfig("sgmv_layer", shape, ranks, 1, 2048)
    s = Setup(cfg)
    runs = [(0, 300), (1, 130), (-1, 5), (2, 128), (3, 1), (4, 77), (5, 129), (-1, 2), (6, 64),
            (7, 9), (2, 40)]
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in runs])
    T = len(ta)
    x = synth.activations(T, 4096, shape.dtype, "x", salt=5)
    y0 = [synth.activations(T, 2048, shape.dtype, "y", salt=5 + p) for p in range(2)]
    ys = [y.cuda() for y in y0]
    plan = BatchPlan(s.store, ta)
    n0 = kernel_launch_count()
    sgmv_layer(plan, 1, x.cuda(), ys, 0.5)
    torch.cuda.synchronize()
    assert kernel_launch_count() - n0 == 3  # joint shrink + reduction + expand
    for p in range(2):
        ref = s.oracle(1, p, x, y0[p], ta, scale=0.5, v_bf16=True)
        assert rel_err(ys[p], ref) <= TOL_BF16, p
        none = ta < 0
        assert np.array_equal(to_np_bits(ys[p])[none], to_np_bits(y0[p])[none])


def test_sgmv_layer_cfg3_agrees_with_per_projection(cuda):
    """BASELINE config 3 call shape (6 segments × 512): the joint launch agrees
    with two plora_sgmv calls within the bf16 tolerance."""
    cfg = synth.cfg3(n_layers=2, n_segments=6)
    s = Setup(cfg)
    ta = synth.segment_assignment(6, 512)
    plan = BatchPlan(s.store, ta)
    x = torch.randn(len(ta), 4096, device="cuda").to(torch.bfloat16)
    y0 = torch.randn(len(ta), 4096, device="cuda").to(torch.bfloat16)
    a = [y0.clone(), y0.clone()]
    b = [y0.clone(), y0.clone()]
    sgmv_layer(plan, 1, x, a)
    for p in range(2):
        sgmv(plan, 1, p, x, b[p])
    torch.cuda.synchronize()
    for p in range(2):
        err = (a[p].float() - b[p].float()).abs().max().item() / b[p].float().abs().max().item()
        assert err <= TOL_BF16, (p, err)


@pytest.mark.parametrize("page_bytes", [64, 256])
def test_sgmv_small_pages(cuda, page_bytes):
    """Pages smaller than a row segment of a K chunk / column block: the
    gathers translate every 16-byte piece (64 B) or every 128-byte segment
    (256 B) through the page table; per-projection and per-layer paths."""
    shape = ModelShape(2, (1024, 1024), (1024, 1024), torch.bfloat16)
    ranks = [16, 64, 128, 5]
    cfg = synth.DecodeConfig("sgmv_smallpage", shape, ranks, 1, page_bytes)
    s = Setup(cfg)
    runs = [(0, 200), (1, 128), (-1, 3), (2, 150), (3, 20)]
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in runs])
    yd, ref, _ = _sgmv_vs_oracle(s, ta, 1, 0, scale=0.5, salt=2)
    assert rel_err(yd, ref) <= TOL_BF16
    T = len(ta)
    x = synth.activations(T, 1024, shape.dtype, "x", salt=3)
    y0 = [synth.activations(T, 1024, shape.dtype, "y", salt=3 + p) for p in range(2)]
    ys = [y.cuda() for y in y0]
    sgmv_layer(BatchPlan(s.store, ta), 0, x.cuda(), ys)
    torch.cuda.synchronize()
    for p in range(2):
        ref = s.oracle(0, p, x, y0[p], ta, v_bf16=True)
        assert rel_err(ys[p], ref) <= TOL_BF16, p


@pytest.mark.parametrize("page_bytes", [64, 256, 2048])
def test_sgmv_persistent_expand_bit_identical(cuda, page_bytes):
    """The persistent expand (plora_debug_set_sgmv_flags bit 20, a measured
    alternative) gives the tiled expand's y bit for bit: mixed ranks incl. a
    rank with gather4 tail/padding rows (5), partial tiles, adapter-less
    tokens, gather4 (>= 256 B pages) and cp.async (64 B) modes."""
    from paper_2512_20210_b200 import _native as N
    shape = ModelShape(2, (1024, 1024), (1024, 1024), torch.bfloat16)
    cfg = synth.DecodeConfig("sgmv_persist", shape, [16, 64, 128, 5], 1, page_bytes)
    s = Setup(cfg)
    runs = [(0, 200), (1, 128), (-1, 3), (2, 150), (3, 20), (2, 300)]
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in runs])
    T = len(ta)
    x = synth.activations(T, 1024, shape.dtype, "x", salt=5).cuda()
    y0 = [synth.activations(T, 1024, shape.dtype, "y", salt=6 + p).cuda() for p in range(2)]
    plan = BatchPlan(s.store, ta)
    outs = []
    try:
        for flags in (0, 1 << 20):
            N.check(N.lib().plora_debug_set_sgmv_flags(flags))
            ys = [y.clone() for y in y0]
            sgmv_layer(plan, 1, x, ys, scale=0.75)
            torch.cuda.synchronize()
            outs.append(ys)
    finally:
        N.check(N.lib().plora_debug_set_sgmv_flags(0))
    for p in range(2):
        assert torch.equal(outs[0][p], outs[1][p]), p
        assert not torch.equal(outs[0][p], y0[p])
