"""The oracle is pinned before it is trusted: the pure-Python PagePool
restatement against the compiled reference, and the C paged-LoRA oracle
against an independent dense numpy restatement (gather pages -> dense A, B ->
x·Aᵀ·Bᵀ) and against the committed golden fixtures."""
import os
import random

import numpy as np
import pytest

from oracle import lora as OL
from oracle.pagepool import OraclePagePool

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_python_pagepool_restatement_matches_reference(ref):
    rng = random.Random(5)
    ours, theirs = OraclePagePool(4096, 700), ref.RefPagePool(4096, 700)
    live = set()
    for op in range(6000):
        a = rng.randrange(48)
        if op % 333 == 0:
            assert ours.compact() == theirs.compact()
        if a in live:
            ours.release(a)
            theirs.free(a)
            live.discard(a)
        else:
            b = rng.randrange(1, 200_000)
            st = ours.alloc(a, b)
            assert st == theirs.alloc(a, b)
            if st == 0:
                live.add(a)
        for x in live:
            assert ours.table(x) == theirs.table(x)


def _dense_reference(m, arena, page, tables, ranks, layer, proj, x, y, ta, scale, esize):
    """Independent restatement: reassemble each adapter's logical bytes, slice
    the (layer, proj) block, and do the dense math in float64."""
    out = OL.bf16_bits_to_f32(y).astype(np.float64) if esize == 2 else y.astype(np.float64)
    xf = OL.bf16_bits_to_f32(x).astype(np.float64) if esize == 2 else x.astype(np.float64)
    din, dout = m.d_in[proj], m.d_out[proj]
    for a, r in ranks.items():
        nbytes = OL.adapter_bytes(m, r)
        raw = OL.gather_pages(arena, page, tables[a], nbytes)
        vals = raw.view(np.uint16) if esize == 2 else raw.view(np.float32)
        vals = OL.bf16_bits_to_f32(vals).astype(np.float64) if esize == 2 else vals.astype(np.float64)
        off = OL.block_offset(m, r, layer, proj) // esize
        A = vals[off:off + r * din].reshape(r, din)
        Bt = vals[off + r * din:off + r * din + r * dout].reshape(r, dout)
        rows = np.where(ta == a)[0]
        if len(rows):
            v = xf[rows] @ A.T
            out[rows] += scale * (v @ Bt)
    return out


@pytest.mark.parametrize("esize", [2, 4])
def test_c_oracle_matches_dense_restatement(esize):
    z = np.load(os.path.join(GOLDEN, "lora_small.npz"))
    dt = "bf16" if esize == 2 else "f32"
    ranks = {a: int(r) for a, r in enumerate(z[f"{dt}_ranks"])}
    page, total = (int(v) for v in z[f"{dt}_page"])
    m = OL.model(2, (64, 128), (64, 32), esize)
    arena = np.zeros(total * page, np.uint8)
    tables = {a: list(z[f"{dt}_table{a}"]) for a in ranks}
    for a in ranks:
        OL.scatter_pages(arena, page, tables[a], z[f"{dt}_img{a}"])
    ta = z[f"{dt}_tokens"]
    for layer in range(2):
        for proj in range(2):
            x = z[f"{dt}_x_{layer}_{proj}"]
            y0 = z[f"{dt}_y0_{layer}_{proj}"]
            y = y0.copy()
            OL.paged_lora_apply(m, arena, page, tables, ranks, layer, proj, x, y, ta, scale=0.5)
            # the golden fixture pins this exact output
            assert np.array_equal(y, z[f"{dt}_y_{layer}_{proj}_v0"])
            dense = _dense_reference(m, arena, page, tables, ranks, layer, proj, x, y0, ta, 0.5,
                                     esize)
            got = OL.bf16_bits_to_f32(y) if esize == 2 else y
            tol = 1e-2 if esize == 2 else 1e-6
            assert np.abs(got - dense).max() <= tol * max(np.abs(dense).max(), 1.0)


def test_oracle_threading_is_deterministic():
    z = np.load(os.path.join(GOLDEN, "lora_small.npz"))
    ranks = {a: int(r) for a, r in enumerate(z["bf16_ranks"])}
    page, total = (int(v) for v in z["bf16_page"])
    m = OL.model(2, (64, 128), (64, 32), 2)
    arena = np.zeros(total * page, np.uint8)
    tables = {a: list(z[f"bf16_table{a}"]) for a in ranks}
    for a in ranks:
        OL.scatter_pages(arena, page, tables[a], z[f"bf16_img{a}"])
    x, y0 = z["bf16_x_1_0"], z["bf16_y0_1_0"]
    outs = []
    for nt in (1, 3, 8):
        y = y0.copy()
        OL.paged_lora_apply(m, arena, page, tables, ranks, 1, 0, x, y, z["bf16_tokens"],
                            scale=0.5, nthreads=nt)
        outs.append(y)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_bf16_rounding_helpers():
    vals = np.asarray([0.0, 1.0, -2.5, 1.00390625, 1.005859375, 3.4e38, 1e-40], np.float32)
    bits = OL.f32_to_bf16_bits(vals)
    for v, b in zip(vals, bits):
        assert OL.lib().oracle_f32_to_bf16(float(v)) == int(b)
