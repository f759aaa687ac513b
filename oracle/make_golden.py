"""ORACLE ONLY — generates the committed golden fixtures under tests/golden/.

Run here (where /root/reference exists):  python oracle/make_golden.py

  pagepool_appendix_a.json  SURVEY Appendix A vectors from the reference PagePool
  pagepool_churn.json       churn op sequence + reference outcomes + final dump
  policy_golden.json        test_prefetch.cpp scenarios evaluated by the reference
  lora_small.npz            tiny paged-LoRA known-answer vectors: tables from the
                            reference PagePool, outputs from lora_oracle.c
  cfg1_checksums.json       oracle outputs at BASELINE config 1 (sha256 + stats)
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import lora as OL  # noqa: E402
from oracle import ref as R  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
MiB = 1 << 20


def appendix_a():
    p = R.RefPagePool(2048, 16)
    p.alloc(0, 3 * 2048)
    p.alloc(1, 2 * 2048)
    p.alloc(2, 4 * 2048)
    p.free(1)
    p.alloc(3, 5 * 2048 + 1)
    hole = {"a0": p.table(0), "a2": p.table(2), "a3": p.table(3)}
    p.free(0)
    before = {a: p.table(a) for a in p.resident()}
    moved = p.compact()
    relocs = []
    for a in sorted(before):
        after = p.table(a)
        for i, (x, y) in enumerate(zip(before[a], after)):
            if x != y:
                relocs.append([a, i, x, y])
    ext, intf, util = p.report()
    return {"hole_reuse": hole,
            "compaction": {"moved": moved, "a2": p.table(2), "a3": p.table(3),
                           "internal_frag": intf, "utilization": util,
                           "free": p.free_pages(), "dump": p.dump(), "relocations": relocs}}


def churn():
    page, total = 2 * MiB, 256
    p = R.RefPagePool(page, total)
    rng = random.Random(20240611)
    live, ops = set(), []
    for op in range(4000):
        a = rng.randrange(64)
        if op % 512 == 511:
            ops.append(["c", p.compact()])
        if a in live:
            p.free(a)
            live.discard(a)
            ops.append(["f", a])
        else:
            b = rng.randrange(1, 24 * MiB + 1)
            st = p.alloc(a, b)
            if st == 0:
                live.add(a)
            ops.append(["a", a, b, st])
    p.check_invariants()
    return {"page_bytes": page, "total_pages": total, "ops": ops, "final_dump": p.dump()}


class _D:  # plain AdapterDynamics for the ref shim
    def __init__(self, status=0, last=-1.0, decayed=0.0, stamp=0.0, pred=0.0, busy=0, active=False):
        self.status, self.last_access_ms, self.decayed_count = status, last, decayed
        self.decay_stamp_ms, self.prediction, self.busy, self.transfer_active = stamp, pred, busy, active


class _P:
    def __init__(self, **kw):
        self.theta, self.alpha, self.beta, self.gamma = 0.5, 0.3, 0.3, 0.4
        self.tau_ms, self.freq_half_life_ms, self.staging_fraction = 60000.0, 120000.0, 0.1
        for k, v in kw.items():
            setattr(self, k, v)


def policy():
    out = {}
    pol = _P(theta=0.8)
    dyn = [_D() for _ in range(4)]
    units = [2, 2, 2, 2]
    out["strict_threshold"] = R.select_prefetch([0.8, 0.8000001, 0.1, 0.0], dyn, pol, units, 100)
    out["cap2"] = R.select_prefetch([0.9, 0.7, 0.95, -1.0], dyn, pol, units, 2)
    out["cap4"] = R.select_prefetch([0.9, 0.7, 0.95, -1.0], dyn, pol, units, 4)
    dyn2 = [_D() for _ in range(4)]
    dyn2[2].status = 1
    dyn2[0].transfer_active = True
    out["staging_excluded"] = R.select_prefetch([0.9, 0.85, 0.95, 0.99], dyn2, pol, units, 100)
    out["evict_120"] = R.plan_evictions(120, 0, [1, 3, 0, 2], [100, 50, 200, 80])
    out["evict_noop"] = R.plan_evictions(40, 50, [0, 1, 2, 3], [100, 50, 200, 80])
    out["evict_unsat"] = R.plan_evictions(1000, 0, [0, 1], [100, 50, 200, 80])
    # random score vectors (bit-exact doubles)
    rng = random.Random(4242)
    cases = []
    for _ in range(50):
        n = 1 + rng.randrange(12)
        dyn = [_D(status=rng.randrange(3), last=rng.random() * 200000 - 10000,
                  decayed=rng.random() * 10, stamp=rng.random() * 100000, pred=rng.random(),
                  active=rng.random() < 0.2) for _ in range(n)]
        pol = _P(alpha=rng.random(), beta=rng.random(), gamma=rng.random() + 0.01)
        now = 150000.0 + rng.random() * 50000
        probs = [rng.random() for _ in range(n)]
        units = [1 + rng.randrange(8) for _ in range(n)]
        budget = rng.randrange(20)
        cases.append({
            "dyn": [vars(d) for d in dyn], "policy": vars(pol), "now": now, "probs": probs,
            "units": units, "budget": budget,
            "scored": R.scored_residents(dyn, pol, now),
            "picks": R.select_prefetch(probs, dyn, pol, units, budget),
            "scores": [R.eviction_score(d, pol, now, 5.0) for d in dyn],
        })
    out["random"] = cases
    return out


def small_model():
    return dict(n_layers=2, d_in=(64, 128), d_out=(64, 32))


def lora_small():
    """Tiny known-answer vectors: bf16 and fp32, mixed odd ranks, 64-byte pages,
    tokens with no adapter (-1), repeated adapters."""
    arrays = {}
    mdef = small_model()
    ranks = [1, 3, 8, 5, 16, 2]
    for dt, esize in (("bf16", 2), ("f32", 4)):
        m = OL.model(mdef["n_layers"], mdef["d_in"], mdef["d_out"], esize)
        page = 64
        sizes = [OL.adapter_bytes(m, r) for r in ranks]
        total = sum(-(-s // page) for s in sizes) * 2
        pool = R.RefPagePool(page, total)
        for a, s in enumerate(sizes):
            pool.alloc(a, s)
        for a in range(0, len(ranks), 2):
            pool.free(a)
        for a in range(0, len(ranks), 2):
            pool.alloc(a, sizes[a])
        rng = np.random.default_rng(99 + esize)
        arena = np.zeros(total * page, np.uint8)
        tables, images = {}, []
        for a, r in enumerate(ranks):
            img = rng.standard_normal(sizes[a] // esize).astype(np.float32) * 0.3
            img = OL.f32_to_bf16_bits(img) if esize == 2 else img
            images.append(img)
            tables[a] = pool.table(a)
            OL.scatter_pages(arena, page, tables[a], img)
            arrays[f"{dt}_img{a}"] = img
            arrays[f"{dt}_table{a}"] = np.asarray(tables[a], np.uint32)
        T = 23
        ta = rng.integers(-1, len(ranks), size=T).astype(np.int32)
        arrays[f"{dt}_tokens"] = ta
        for layer in range(mdef["n_layers"]):
            for proj in range(2):
                din, dout = mdef["d_in"][proj], mdef["d_out"][proj]
                x = rng.standard_normal((T, din)).astype(np.float32)
                y = rng.standard_normal((T, dout)).astype(np.float32)
                if esize == 2:
                    x, y = OL.f32_to_bf16_bits(x), OL.f32_to_bf16_bits(y)
                arrays[f"{dt}_x_{layer}_{proj}"] = x
                arrays[f"{dt}_y0_{layer}_{proj}"] = y.copy()
                for vb in (0, 1):
                    yy = y.copy()
                    OL.paged_lora_apply(m, arena, page, tables, dict(enumerate(ranks)), layer,
                                        proj, x, yy, ta, scale=0.5, v_bf16=bool(vb))
                    arrays[f"{dt}_y_{layer}_{proj}_v{vb}"] = yy
        arrays[f"{dt}_ranks"] = np.asarray(ranks, np.uint32)
        arrays[f"{dt}_page"] = np.asarray([page, total], np.uint64)
    return arrays


def cfg1_checksums():
    """Oracle outputs at BASELINE config 1 — page tables from the reference
    PagePool under the synth churn prologue; inputs from paper_2512_20210_b200.synth."""
    import torch
    from paper_2512_20210_b200 import synth
    cfg = synth.cfg1()
    m = OL.model(cfg.shape.n_layers, cfg.shape.d_in, cfg.shape.d_out, cfg.shape.esize)
    sizes = [cfg.shape.adapter_bytes(r) for r in cfg.ranks]
    total = int(sum(-(-s // cfg.page_bytes) for s in sizes) * cfg.pool_factor)
    pool = R.RefPagePool(cfg.page_bytes, total)
    for a, s in enumerate(sizes):
        pool.alloc(a, s)
    for a in range(0, cfg.n_adapters, 2):
        pool.free(a)
    for a in range(0, cfg.n_adapters, 2):
        pool.alloc(a, sizes[a])
    arena = np.zeros(total * cfg.page_bytes, np.uint8)
    tables = {}
    for a, r in enumerate(cfg.ranks):
        img = synth.adapter_image(cfg.shape, r, a).view(torch.int16).numpy().view(np.uint16)
        tables[a] = pool.table(a)
        OL.scatter_pages(arena, cfg.page_bytes, tables[a], img)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    out = {"tables_sha256": hashlib.sha256(
        np.concatenate([np.asarray(tables[a], np.uint32) for a in range(cfg.n_adapters)])
        .tobytes()).hexdigest(), "calls": []}
    for layer, proj in ((0, 0), (0, 1), (17, 0), (31, 1)):
        salt = layer * 2 + proj
        x = synth.activations(cfg.n_tokens, 4096, torch.bfloat16, "x", salt=salt)
        y = synth.activations(cfg.n_tokens, 4096, torch.bfloat16, "y", salt=salt)
        xb = x.view(torch.int16).numpy().view(np.uint16).copy()
        yb = y.view(torch.int16).numpy().view(np.uint16).copy()
        y0 = OL.bf16_bits_to_f32(yb).copy()
        OL.paged_lora_apply(m, arena, cfg.page_bytes, tables, dict(enumerate(cfg.ranks)), layer,
                            proj, xb, yb, ta, nthreads=8)
        dy = OL.bf16_bits_to_f32(yb) - y0
        out["calls"].append({"layer": layer, "proj": proj,
                             "y_sha256": hashlib.sha256(yb.tobytes()).hexdigest(),
                             "dy_absmax": float(np.abs(dy).max()),
                             "dy_mean": float(dy.mean())})
    return out


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    with open(os.path.join(GOLDEN, "pagepool_appendix_a.json"), "w") as f:
        json.dump(appendix_a(), f, indent=1)
    with open(os.path.join(GOLDEN, "pagepool_churn.json"), "w") as f:
        json.dump(churn(), f)
    with open(os.path.join(GOLDEN, "policy_golden.json"), "w") as f:
        json.dump(policy(), f)
    np.savez_compressed(os.path.join(GOLDEN, "lora_small.npz"), **lora_small())
    with open(os.path.join(GOLDEN, "cfg1_checksums.json"), "w") as f:
        json.dump(cfg1_checksums(), f, indent=1)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
