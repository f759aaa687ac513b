"""External sanity check of the C oracle's LoRA arithmetic:
vLLM's pure-torch reference ops (vllm/lora/ops/torch_ops/lora_ops.py,
`bgmv_shrink` / `bgmv_expand`, contiguous weights A [L, r, h_in] and
B [L, h_out, r], y += (x·Aᵀ)·Bᵀ·scale) against oracle/lora_oracle.c reading
the same weights through scattered page tables, at BASELINE config 1 widths.

This is not a reference oracle (the reference ships no LoRA arithmetic,
SPEC.md:70,341) — it pins our restatement's convention and arithmetic to a
widely used third-party implementation.  Runs on CPU."""
import numpy as np
import pytest
import torch

from oracle import lora as OL
from paper_2512_20210_b200 import synth

lora_ops = pytest.importorskip("vllm.lora.ops.torch_ops.lora_ops")


def _unpack(shape, img: torch.Tensor, rank: int, layer: int, proj: int):
    """A (r × d_in) and B = (Bᵀ)ᵀ (d_out × r) of one (layer, proj) block."""
    off = shape.block_offset(rank, layer, proj) // shape.esize
    din, dout = shape.d_in[proj], shape.d_out[proj]
    A = img[off:off + rank * din].view(rank, din)
    Bt = img[off + rank * din:off + rank * (din + dout)].view(rank, dout)
    return A, Bt.t().contiguous()


@pytest.mark.parametrize("layer,proj", [(0, 1), (1, 0)])
def test_oracle_matches_vllm_torch_ops_cfg1(layer, proj):
    cfg = synth.cfg1(n_layers=2)
    shape = cfg.shape
    pool = synth.build_pool(cfg)
    P = cfg.page_bytes
    arena = np.zeros(pool.total_pages() * P, np.uint8)
    rmax = max(cfg.ranks)
    L = cfg.n_adapters
    A_all = torch.zeros(L, rmax, 4096, dtype=torch.float32)   # rank-padded, as vLLM stacks
    B_all = torch.zeros(L, 4096, rmax, dtype=torch.float32)
    for a, r in enumerate(cfg.ranks):
        img = synth.adapter_image(shape, r, a)
        OL.scatter_pages(arena, P, pool.table(a), img.view(torch.int16).numpy().view(np.uint16))
        A, B = _unpack(shape, img, r, layer, proj)
        A_all[a, :r] = A.float()
        B_all[a, :, :r] = B.float()
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    x = synth.activations(T, 4096, torch.bfloat16, "x", salt=9)
    y0 = synth.activations(T, 4096, torch.bfloat16, "y", salt=9)
    scale = 0.5
    # vLLM: fp32 shrink (scaled), fp32 expand added into an fp32 copy of y0
    idx = torch.from_numpy(ta.astype(np.int64))
    v = torch.zeros(T, rmax, dtype=torch.float32)
    lora_ops.bgmv_shrink(x.float(), A_all, v, idx, scale)
    yv = y0.float().clone()
    lora_ops.bgmv_expand(v, B_all, yv, idx, add_inputs=True)
    # oracle: paged reads, double accumulation, fp32 v, bf16 result
    xb = x.view(torch.int16).numpy().view(np.uint16).copy()
    yb = y0.view(torch.int16).numpy().view(np.uint16).copy()
    m = OL.model(2, shape.d_in, shape.d_out, 2)
    OL.paged_lora_apply(m, arena, P, {a: pool.table(a) for a in range(L)},
                        dict(enumerate(cfg.ranks)), layer, proj, xb, yb, ta, scale=scale,
                        nthreads=8)
    got = OL.bf16_bits_to_f32(yb).astype(np.float64)
    want = yv.double().numpy()
    delta = want - y0.double().numpy()
    # the oracle rounds y once to bf16: within half a bf16 ulp of vLLM's fp32
    # result (plus fp32-vs-double accumulation noise)
    ulp = np.abs(want) * 2.0 ** -8 + 1e-6
    assert (np.abs(got - want) <= ulp).all()
    err = np.abs((got - y0.double().numpy()) - delta).max() / np.abs(delta).max()
    assert err <= 1e-2, err
