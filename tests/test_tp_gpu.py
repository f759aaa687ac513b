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


@pytest.mark.parametrize("tp_size", [1, 2, 4, 8])
def test_fused_allgather_emulated_ranks_bit_identical(setup70, tp_size):
    """The peer-write all-gather (plora_bgmv_tp_shrink_push / _expand_wait):
    N ranks emulated in one process, each with its own pair of gathered
    buffers and arrival flags, every rank's shrink storing into all of them.
    Three calls (buffer parities 0, 1, 0) must equal the unfused halves bit
    for bit, and leave every flag at zero (arrivals consumed)."""
    from paper_2512_20210_b200.tp import bgmv_tp_expand_wait, bgmv_tp_shrink_push
    s = setup70
    cfg = s.cfg
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    plan = BatchPlan(s.store, ta)
    rs = tp_shard_rows(plan, tp_size)
    vg = [torch.zeros(2, tp_size, T, rs, dtype=torch.float32, device="cuda") for _ in range(tp_size)]
    flags = [torch.zeros(tp_size, dtype=torch.int32, device="cuda") for _ in range(tp_size)]
    for call, (layer, proj) in enumerate(((0, 0), (1, 1), (1, 0))):
        din, dout = cfg.shape.d_in[proj], cfg.shape.d_out[proj]
        ncols = dout // tp_size
        x = synth.activations(T, din, torch.bfloat16, "x", salt=call).cuda()
        y0 = synth.activations(T, dout, torch.bfloat16, "y", salt=call).cuda()
        par = call & 1
        y_f, y_u = y0.clone(), y0.clone()
        for r in range(tp_size):
            bgmv_tp_shrink_push(plan, layer, proj, r, tp_size, x, [vg[d][par].data_ptr() for d in range(tp_size)],
                                [flags[d].data_ptr() for d in range(tp_size)])
        for r in range(tp_size):
            bgmv_tp_expand_wait(plan, layer, proj, r, tp_size, vg[r][par], flags[r],
                                y_f[:, r * ncols:(r + 1) * ncols], 0.5)
        parts = [bgmv_tp_shrink(plan, layer, proj, r, tp_size, x,  # (zeros: rows past r/N stay unwritten)
                                torch.zeros(T, rs, dtype=torch.float32, device="cuda")) for r in range(tp_size)]
        vu = torch.stack(parts).contiguous()
        for r in range(tp_size):
            bgmv_tp_expand(plan, layer, proj, r, tp_size, vu, y_u[:, r * ncols:(r + 1) * ncols], 0.5)
        torch.cuda.synchronize()
        for r in range(tp_size):  # every rank's gathered buffer holds every rank's rows
            assert torch.equal(vg[r][par], vu), (call, r)
        assert torch.equal(y_f, y_u), call
        assert all(int(f.abs().sum()) == 0 for f in flags)


def test_fused_allgather_module_tp1_and_graph(setup70):
    s = setup70
    ta = synth.token_assignment(s.cfg.n_adapters, s.cfg.tokens_per_adapter)
    plan = BatchPlan(s.store, ta)
    T = len(ta)
    x = synth.activations(T, 8192, torch.bfloat16, "x").cuda()
    y0 = synth.activations(T, 8192, torch.bfloat16, "y").cuda()
    fused = TensorParallelLoRA(plan, 0, 1, force_split=True, allgather="fused")
    plain = TensorParallelLoRA(plan, 0, 1, force_split=True)
    ya, yb = y0.clone(), y0.clone()
    for layer in (0, 1):
        fused(layer, 0, x, ya)
        plain(layer, 0, x, yb)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
    # a captured step of two calls (even: the buffer parity repeats per replay)
    yg = y0.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fused(0, 0, x, yg)
        fused(1, 0, x, yg)
    yg.copy_(y0)
    g.replay()
    g.replay()
    yc = y0.clone()
    for _ in range(2):
        for layer in (0, 1):
            plain(layer, 0, x, yc)
    torch.cuda.synchronize()
    assert torch.equal(yg, yc)
    assert int(fused._ff.abs().sum()) == 0


@pytest.mark.parametrize("tp_size", [2, 4])
@pytest.mark.parametrize("page_bytes", [2048, 256])
def test_tp_warp_items_edge_cases(cuda, tp_size, page_bytes):
    """The warp-item TP halves away from cfg5: input widths that are not a
    multiple of the 1024-input K slice (1000: a partial last slice), 1-7
    tokens per adapter (jobs of 1-4 tokens, a 6-token adapter over two jobs),
    ranks whose shard is smaller than an item (rs = 2) or spans several row
    blocks (rs = 32), rank 128 (split expand pairs), 256-byte pages (page
    entries by table loads); unfused and fused halves against the oracle and
    each other."""
    from paper_2512_20210_b200.lora import ModelShape
    from paper_2512_20210_b200.tp import bgmv_tp_expand_wait, bgmv_tp_shrink_push
    shape = ModelShape(2, (1000, 1000), (512, 1024), torch.bfloat16)
    ranks = [8, 16, 64, 128, 4 * tp_size, 8]
    s = Setup(synth.DecodeConfig("tp_edge", shape, ranks, 1, page_bytes))
    rng = np.random.default_rng(11)
    ta = np.concatenate([np.full(1 + (3 * a) % 7, a, np.int32) for a in range(len(ranks))])
    rng.shuffle(ta)
    T = len(ta)
    plan = BatchPlan(s.store, ta)
    rs = tp_shard_rows(plan, tp_size)
    for proj in (0, 1):
        din, dout = shape.d_in[proj], shape.d_out[proj]
        ncols = dout // tp_size
        x = synth.activations(T, din, torch.bfloat16, "x", salt=proj + 7)
        y0 = synth.activations(T, dout, torch.bfloat16, "y", salt=proj + 7)
        xd = x.cuda()
        parts = [bgmv_tp_shrink(plan, 1, proj, r, tp_size, xd, torch.zeros(T, rs, dtype=torch.float32, device="cuda"))
                 for r in range(tp_size)]
        vu = torch.stack(parts).contiguous()
        y_u = y0.cuda().clone()
        for r in range(tp_size):
            bgmv_tp_expand(plan, 1, proj, r, tp_size, vu, y_u[:, r * ncols:(r + 1) * ncols], 0.5)
        vg = [torch.zeros(tp_size, T, rs, dtype=torch.float32, device="cuda") for _ in range(tp_size)]
        flags = [torch.zeros(tp_size, dtype=torch.int32, device="cuda") for _ in range(tp_size)]
        y_f = y0.cuda().clone()
        for r in range(tp_size):
            bgmv_tp_shrink_push(plan, 1, proj, r, tp_size, xd, [v.data_ptr() for v in vg],
                                [f.data_ptr() for f in flags])
        for r in range(tp_size):
            bgmv_tp_expand_wait(plan, 1, proj, r, tp_size, vg[r], flags[r], y_f[:, r * ncols:(r + 1) * ncols], 0.5)
        torch.cuda.synchronize()
        ref = s.oracle(1, proj, x, y0, ta, scale=0.5)
        assert rel_err(y_u, ref) <= TOL_BF16, proj
        assert torch.equal(y_f, y_u), proj
        assert all(int(f.abs().sum()) == 0 for f in flags)
