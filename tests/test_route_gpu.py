"""Decode batches with many-token adapters (VERDICT r01 missing #5): adapters
with >= N tokens (default 160; 16 here) leave the decode kernels for the tensor-core SGMV path on a
child plan (their x rows gathered, deltas added back), run concurrently with
the decode kernels over the other adapters.  The reference batches any number
of requests per adapter into a decode step (src/engine.cpp:499-511).

Checked against the CPU oracle (delta-only bound), against the unrouted
decode kernels, through every decode entry point (plora_bgmv, plora_bgmv_layer,
plora_bgmv_layers, CUDA-graph replay) and with every adapter routed."""
import ctypes as C

import numpy as np
import pytest
import torch

from lora_harness import TOL_BF16, Setup, delta_rel_err, rel_err
from paper_2512_20210_b200 import _native as N, synth
from paper_2512_20210_b200.lora import BatchPlan, ModelShape, bgmv, bgmv_layer, bgmv_layers
from test_parity_full_gpu import skewed_assignment

pytestmark = pytest.mark.gpu


def routed(plan):
    n = C.c_uint32()
    N.check(N.lib().plora_debug_plan_routed(plan.handle, C.byref(n)))
    return n.value


def set_route(n):
    N.check(N.lib().plora_debug_set_route_tokens(n))


@pytest.fixture(scope="module")
def skew(cuda):
    shape = ModelShape(3, (4096, 4096), (4096, 4096), torch.bfloat16)
    ranks = [(8, 16, 32, 64, 128)[a % 5] for a in range(128)]
    s = Setup.on_device(synth.DecodeConfig("skew", shape, ranks, 1, 2048))
    yield s
    set_route(160)  # the library default
    del s


def _xy(T, salt, zero_y=True, n_out=2, layers=None):
    shp = (T, 4096) if layers is None else (layers, T, 4096)
    g = torch.Generator().manual_seed(salt)
    x = (torch.randn(shp, generator=g) * 0.5).to(torch.bfloat16)
    ys = [torch.zeros(shp, dtype=torch.bfloat16) if zero_y else
          torch.randn(shp, generator=g).to(torch.bfloat16) for _ in range(n_out)]
    return x, ys


def test_routed_bgmv_matches_oracle_and_unrouted(skew):
    s = skew
    ta = skewed_assignment(seed=29, hot=80)
    counts = np.bincount(ta, minlength=128)
    T = len(ta)
    set_route(16)
    plan = BatchPlan(s.store, ta)
    assert routed(plan) == int(counts[counts >= 16].sum()) > 0
    set_route(0)
    plain = BatchPlan(s.store, ta)
    assert routed(plain) == 0
    set_route(16)
    for layer, proj, zero_y in ((0, 0, True), (2, 1, False)):
        x, (y0,) = _xy(T, 100 + layer, zero_y=zero_y, n_out=1)
        ya, yb = y0.cuda(), y0.cuda()
        bgmv(plan, layer, proj, x.cuda(), ya, 0.5)
        bgmv(plain, layer, proj, x.cuda(), yb, 0.5)
        torch.cuda.synchronize()
        ref = s.oracle(layer, proj, x, y0, ta, scale=0.5, nthreads=32)
        if zero_y:  # (with y0 != 0 the routed rows' extra bf16 rounding of the delta is ~1 ulp of y)
            assert delta_rel_err(ya, ref, y0) <= TOL_BF16, (layer, proj)
        assert rel_err(ya, ref) <= TOL_BF16
        # routed rows carry bf16 v and one bf16 rounding of the delta (SGMV);
        # the other rows are the same decode kernels' results, bit for bit
        hot = torch.from_numpy(np.isin(ta, np.nonzero(counts >= 16)[0])).cuda()
        assert torch.equal(ya[~hot], yb[~hot])
        d = (ya[hot].float() - yb[hot].float()).abs().max().item()
        assert d <= 2e-2 * max(yb[hot].float().abs().max().item(), 1e-6)


def test_routed_layer_and_multi_layer_launch(skew):
    s = skew
    ta = skewed_assignment(seed=31, hot=64)
    T = len(ta)
    set_route(16)
    plan = BatchPlan(s.store, ta)
    assert routed(plan) > 0
    x, y0 = _xy(T, 7, zero_y=True, layers=3)
    xd = x.cuda()
    per = [y.cuda() for y in y0]
    for l in range(3):
        bgmv_layer(plan, l, xd[l], [per[0][l], per[1][l]], 0.75)
    multi = [y.cuda() for y in y0]
    bgmv_layers(plan, 0, xd, multi, 0.75)
    torch.cuda.synchronize()
    for p in range(2):
        # routed rows: same SGMV kernels, same order of sums; decode rows: the single-layer calls split
        # the widest adapters' expand items over two warps (another fp32 order, <= 1 bf16 ulp apart)
        d = (per[p].float() - multi[p].float()).abs()
        assert (d <= multi[p].float().abs() * 2.0 ** -7 + multi[p].float().abs().max() * 2.0 ** -12).all(), p
        assert (d > 0).float().mean().item() < 0.05, p
        ref = s.oracle(2, p, x[2], y0[p][2], ta, scale=0.75, nthreads=32)
        assert delta_rel_err(multi[p][2], ref, y0[p][2]) <= TOL_BF16, p


@pytest.mark.parametrize("impl", [0, 3])
def test_routed_hot_adapter_with_hybrid_rest_and_graph(skew, impl):
    """One hot adapter, every other adapter <= 4 tokens: the hot one is routed
    and the rest runs the default warp-item op (impl 0) or the hybrid decode
    pair (impl 3); the whole step replays from a CUDA graph."""
    s = skew
    rng = np.random.default_rng(5)
    ta = np.concatenate([np.full(48, 3, np.int32), np.repeat(np.arange(4, 128, dtype=np.int32), 2)])
    rng.shuffle(ta)
    T = len(ta)
    set_route(16)
    N.check(N.lib().plora_debug_set_bgmv_impl(impl))
    try:
        plan = BatchPlan(s.store, ta)
        assert routed(plan) == 48
        hyb = (C.c_double * 4)()
        N.check(N.lib().plora_debug_plan_hybrid(plan.handle, hyb))
        assert (hyb[0] > 0) == (impl == 3)  # the hybrid streaming share runs beside the clusters
        x, y0 = _xy(T, 9, zero_y=False, layers=3)
        xd = x.cuda()
        eager = [y.cuda() for y in y0]
        bgmv_layers(plan, 0, xd, eager)
        ys = [y.cuda() for y in y0]
        bgmv_layers(plan, 0, xd, [torch.empty_like(y) for y in ys])  # warm (outside capture)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            bgmv_layers(plan, 0, xd, ys)
        for p in range(2):
            ys[p].copy_(y0[p].cuda())
        gr.replay()
        torch.cuda.synchronize()
    finally:
        N.check(N.lib().plora_debug_set_bgmv_impl(0))
    for p in range(2):
        assert torch.equal(ys[p], eager[p]), p
        ref = s.oracle(1, p, x[1], y0[p][1], ta, nthreads=32)
        assert rel_err(eager[p][1], ref) <= TOL_BF16, p


def test_every_adapter_routed(skew):
    s = skew
    ta = np.repeat(np.arange(0, 10, dtype=np.int32), 20)
    np.random.default_rng(2).shuffle(ta)
    T = len(ta)
    set_route(16)
    plan = BatchPlan(s.store, ta)
    assert routed(plan) == T
    x, y0 = _xy(T, 11, zero_y=True)
    ys = [y.cuda() for y in y0]
    bgmv_layer(plan, 1, x.cuda(), ys, 0.5)
    torch.cuda.synchronize()
    for p in range(2):
        ref = s.oracle(1, p, x, y0[p], ta, scale=0.5, nthreads=32)
        assert delta_rel_err(ys[p], ref, y0[p]) <= TOL_BF16, p
