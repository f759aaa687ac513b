"""GPU parity of the tensor-parallel halves (BASELINE cfg5 shapes, 2 layers):
N TP ranks emulated on one device — shrink of every rank, rank-major stack
(what the all-gather produces), expand of every rank into its column shard —
must equal the data-parallel paged BGMV and the CPU oracle on identical
inputs, page tables and adapter assignment."""
import numpy as np
import pytest
import torch

from lora_harness import TOL_BF16, Setup, rel_err
from paper_2512_20210_b200 import ValidationError, synth
from paper_2512_20210_b200.lora import BatchPlan, bgmv
from paper_2512_20210_b200.tp import (TensorParallelLoRA, bgmv_tp_expand, bgmv_tp_shrink,
                                       tp_shard_rows)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup70(cuda):
    cfg = synth.cfg5(n_layers=2, n_adapters=24)
    return Setup(cfg)


@pytest.mark.parametrize("tp_size", [1, 2, 4, 8])
@pytest.mark.parametrize("proj", [0, 1])
def test_tp_emulated_ranks_match_bgmv_and_oracle(setup70, tp_size, proj):
    s = setup70
    cfg = s.cfg
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T, din, dout = len(ta), cfg.shape.d_in[proj], cfg.shape.d_out[proj]
    x = synth.activations(T, din, torch.bfloat16, "x", salt=proj)
    y0 = synth.activations(T, dout, torch.bfloat16, "y", salt=proj)
    plan = BatchPlan(s.store, ta)
    xd = x.cuda()
    rs = tp_shard_rows(plan, tp_size)
    parts = [bgmv_tp_shrink(plan, 1, proj, i, tp_size, xd,
                            torch.empty(T, rs, dtype=torch.float32, device="cuda"))
             for i in range(tp_size)]
    vg = torch.stack(parts).contiguous()
    ncols = dout // tp_size
    y_tp = y0.cuda().clone()
    for i in range(tp_size):
        bgmv_tp_expand(plan, 1, proj, i, tp_size, vg, y_tp[:, i * ncols:(i + 1) * ncols], 0.5)
    y_dp = y0.cuda().clone()
    bgmv(plan, 1, proj, xd, y_dp, 0.5)
    torch.cuda.synchronize()
    ref = s.oracle(1, proj, x, y0, ta, scale=0.5)
    assert rel_err(y_tp, ref) <= TOL_BF16
    # same fp32 v, same single bf16 rounding of y: TP and DP agree to bf16 ulps
    d = (y_tp.float() - y_dp.float()).abs().max().item()
    assert d <= 2e-2 * y_dp.float().abs().max().item()


def test_tp_module_single_rank_and_errors(setup70):
    s = setup70
    ta = synth.token_assignment(s.cfg.n_adapters, s.cfg.tokens_per_adapter)
    plan = BatchPlan(s.store, ta)
    T = len(ta)
    x = synth.activations(T, 8192, torch.bfloat16, "x").cuda()
    y = synth.activations(T, 1024, torch.bfloat16, "y").cuda()
    ref = y.clone()
    bgmv(plan, 0, 1, x, ref)
    TensorParallelLoRA(plan, 0, 1)(0, 1, x, y)
    torch.cuda.synchronize()
    assert (y.float() - ref.float()).abs().max().item() <= 2e-2 * ref.float().abs().max().item()
    with pytest.raises(ValidationError):  # rank 8 adapters are not divisible by 16
        bgmv_tp_shrink(plan, 0, 0, 0, 16, x, torch.empty(T, 8, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValidationError):
        bgmv_tp_shrink(plan, 0, 0, 3, 2, x, torch.empty(T, 64, dtype=torch.float32, device="cuda"))
