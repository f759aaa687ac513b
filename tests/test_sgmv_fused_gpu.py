"""GPU parity of the fused prefill op (plora_sgmv_fused: base projection GEMM
with the paged LoRA as extra K-steps of the same tcgen05 accumulator)
against a torch fp32 base GEMM plus the CPU oracle's LoRA delta."""
import numpy as np
import pytest
import torch

from lora_harness import TOL_BF16, Setup, rel_err, to_f32
from paper_2512_20210_b200 import _native as N, synth
from paper_2512_20210_b200.lora import (BatchPlan, ModelShape, kernel_launch_count, sgmv_fused,
                                        sgmv_fused_layer)

pytestmark = pytest.mark.gpu

RUNS = [(0, 300), (1, 130), (-1, 5), (2, 128), (3, 1), (4, 77), (5, 129), (-1, 2), (6, 64),
        (7, 9), (2, 40)]


def _setup():
    shape = ModelShape(2, (4096, 1024), (4096, 2048), torch.bfloat16)
    ranks = [16, 64, 128, 8, 3, 100, 32, 1]
    return Setup(synth.DecodeConfig("fused", shape, ranks, 1, 2048))


def _delta(s, ta, layer, proj, x, scale):
    """The oracle's LoRA delta (v rounded to bf16, as the tensor-core path)."""
    T = len(ta)
    zero = torch.zeros(T, s.cfg.shape.d_out[proj], dtype=torch.bfloat16)
    bits = s.oracle(layer, proj, x, zero, ta, scale=scale, v_bf16=True)
    return torch.from_numpy(to_f32(bits))


def _run(s, ta, layer, proj, w0, scale, salt):
    shape = s.cfg.shape
    T = len(ta)
    x = synth.activations(T, shape.d_in[proj], shape.dtype, "x", salt=salt)
    plan = BatchPlan(s.store, ta)
    y = torch.full((T, shape.d_out[proj]), 7.0, dtype=torch.bfloat16, device="cuda")  # overwritten
    n0 = kernel_launch_count()
    sgmv_fused(plan, layer, proj, x.cuda(), w0, y, scale)
    torch.cuda.synchronize()
    launches = kernel_launch_count() - n0
    return x, y.cpu(), launches


def test_sgmv_fused_lora_only_matches_oracle(cuda):
    """W0 = 0: y is the LoRA delta alone; rows without an adapter are exactly 0.
    Runs of 1..300 tokens (partial tiles stored per row), ranks 1..128."""
    s = _setup()
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in RUNS])
    for layer, proj in ((0, 0), (1, 1)):
        w0 = torch.zeros(s.cfg.shape.d_out[proj], s.cfg.shape.d_in[proj], dtype=torch.bfloat16,
                         device="cuda")
        x, y, launches = _run(s, ta, layer, proj, w0, 0.5, layer)
        assert launches == 3  # shrink + split reduction + fused GEMM
        ref = _delta(s, ta, layer, proj, x, 0.5)
        assert rel_err(y, ref.numpy()) <= TOL_BF16, (layer, proj)
        assert torch.count_nonzero(y[torch.from_numpy(ta < 0)].float()) == 0


def test_sgmv_fused_base_plus_lora(cuda):
    """Random W0: y = x·W0ᵀ (fp32 torch) + the oracle's delta, within the bf16
    tolerance; the delta is checked separately by the W0 = 0 test."""
    s = _setup()
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in RUNS])
    g = torch.Generator().manual_seed(4321)
    proj = 1
    d_out, d_in = s.cfg.shape.d_out[proj], s.cfg.shape.d_in[proj]
    w0 = (torch.randn(d_out, d_in, generator=g) / d_in ** 0.5).to(torch.bfloat16)
    x, y, _ = _run(s, ta, 1, proj, w0.cuda(), 1.0, 3)
    ref = x.float() @ w0.float().t() + _delta(s, ta, 1, proj, x, 1.0)
    assert rel_err(y, ref.numpy()) <= TOL_BF16


def test_sgmv_fused_cfg3_shape(cuda):
    """BASELINE config 3 call shape at 6 segments × 512 (full tiles: TMA-store
    epilogue), mixed ranks 16/64/128."""
    cfg = synth.cfg3(n_layers=2, n_segments=6)
    s = Setup(cfg)
    ta = synth.segment_assignment(6, 512)
    g = torch.Generator().manual_seed(99)
    w0 = (torch.randn(4096, 4096, generator=g) / 64).to(torch.bfloat16)
    x, y, _ = _run(s, ta, 1, 0, w0.cuda(), 1.0, 11)
    ref = x.float() @ w0.float().t() + _delta(s, ta, 1, 0, x, 1.0)
    assert rel_err(y, ref.numpy()) <= TOL_BF16


def test_sgmv_fused_rejects_bad_shapes(cuda):
    s = _setup()
    ta = np.zeros(10, np.int32)
    plan = BatchPlan(s.store, ta)
    x = torch.zeros(10, 4096, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(10, 4096, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(N.ValidationError):
        sgmv_fused(plan, 0, 0, x, torch.zeros(4096, 4096, device="cuda"), y)  # fp32 weight
    with pytest.raises(N.ValidationError):
        sgmv_fused(plan, 0, 0, x, torch.zeros(2048, 4096, dtype=torch.bfloat16, device="cuda"), y)


@pytest.mark.parametrize("page_bytes", [64, 256, 512, 1024])
def test_sgmv_fused_small_pages(cuda, page_bytes):
    """Bᵀ row segments of a 256-column block straddle pages: the LoRA K-step
    gathers translate every 16-byte piece through the page table."""
    shape = ModelShape(2, (1024, 1024), (1024, 512), torch.bfloat16)
    cfg = synth.DecodeConfig("fused_smallpage", shape, [16, 64, 128, 5], 1, page_bytes)
    s = Setup(cfg)
    runs = [(0, 200), (1, 128), (-1, 3), (2, 150), (3, 20)]
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in runs])
    for proj in (0, 1):
        w0 = torch.zeros(shape.d_out[proj], shape.d_in[proj], dtype=torch.bfloat16, device="cuda")
        x, y, _ = _run(s, ta, 1, proj, w0, 0.5, proj)
        ref = _delta(s, ta, 1, proj, x, 0.5)
        assert rel_err(y, ref.numpy()) <= TOL_BF16, proj


def test_sgmv_fused_layer_matches_per_projection(cuda):
    """plora_sgmv_fused_layer (one shrink for both projections, then one fused
    GEMM each) against torch fp32 base GEMMs plus the oracle's deltas."""
    shape = ModelShape(2, (1024, 1024), (1024, 1024), torch.bfloat16)
    cfg = synth.DecodeConfig("fused_layer", shape, [16, 64, 128, 5], 1, 2048)
    s = Setup(cfg)
    runs = [(0, 200), (1, 128), (-1, 3), (2, 150), (3, 20)]
    ta = np.concatenate([np.full(n, a, np.int32) for a, n in runs])
    T = len(ta)
    g = torch.Generator().manual_seed(77)
    w0 = [(torch.randn(1024, 1024, generator=g) / 32).to(torch.bfloat16) for _ in range(2)]
    x = synth.activations(T, 1024, shape.dtype, "x", salt=9)
    ys = [torch.empty(T, 1024, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    n0 = kernel_launch_count()
    sgmv_fused_layer(BatchPlan(s.store, ta), 1, x.cuda(), [w.cuda() for w in w0], ys, 0.5)
    torch.cuda.synchronize()
    assert kernel_launch_count() - n0 == 4  # joint shrink + reduction + two fused GEMMs
    for p in range(2):
        ref = x.float() @ w0[p].float().t() + _delta(s, ta, 1, p, x, 0.5)
        assert rel_err(ys[p].cpu(), ref.numpy()) <= TOL_BF16, p
