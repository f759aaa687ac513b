"""Small paged-LoRA calls for compute-sanitizer (memcheck / racecheck /
synccheck): the warp-item BGMV (the default: per projection, per layer,
multi-layer; 1-4 token jobs; 256 B pages, odd widths), the cluster BGMV and
the hybrid pair (per projection, fused per layer, multi-layer),
the streaming BGMV (4- and 8-token jobs), the SGMV (per projection, per layer,
fused with the base GEMM, 512 B and 1 KiB pages), the TP halves (NCCL-style
and with the fused peer-write all-gather), decode batches with a routed
many-token adapter, and the GPU predict_all.

compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from lora_harness import Setup  # noqa: E402
from paper_2512_20210_b200 import synth  # noqa: E402
from paper_2512_20210_b200.lora import BatchPlan, bgmv, bgmv_layer, sgmv, sgmv_fused, sgmv_layer  # noqa: E402
from paper_2512_20210_b200.tp import bgmv_tp_expand, bgmv_tp_shrink, tp_shard_rows  # noqa: E402


def main():
    cfg = synth.cfg1(n_layers=2)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    x = torch.randn(T, 4096, device="cuda").to(torch.bfloat16)
    ys = [torch.randn(T, 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
    plan = BatchPlan(s.store, ta)
    bgmv(plan, 1, 0, x, ys[0])
    bgmv_layer(plan, 0, x, ys)
    seg = synth.segment_assignment(4, 160)  # runs of 160 tokens: full and partial tiles
    xs = torch.randn(len(seg), 4096, device="cuda").to(torch.bfloat16)
    yss = torch.randn(len(seg), 4096, device="cuda").to(torch.bfloat16)
    sgmv(BatchPlan(s.store, seg), 1, 1, xs, yss)
    seg2 = synth.segment_assignment(3, 300)  # runs of 300: tile pairs sharing the weight chunks
    xs2 = torch.randn(len(seg2), 4096, device="cuda").to(torch.bfloat16)
    ys2 = torch.randn(len(seg2), 4096, device="cuda").to(torch.bfloat16)
    sgmv(BatchPlan(s.store, seg2), 1, 0, xs2, ys2)
    plan2 = BatchPlan(s.store, seg2)
    sgmv_layer(plan2, 1, xs2, [ys2, ys2.clone()])  # both projections from one x chunk
    w0 = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
    sgmv_fused(plan2, 0, 0, xs2, w0, torch.empty_like(ys2))  # base GEMM + LoRA K-steps
    rs = tp_shard_rows(plan, 2)
    vp = torch.empty(2, T, rs, device="cuda")
    for i in range(2):
        bgmv_tp_shrink(plan, 0, 0, i, 2, x, vp[i])
    for i in range(2):
        bgmv_tp_expand(plan, 0, 0, i, 2, vp, ys[0][:, i * 2048:(i + 1) * 2048])
    # multi-layer launch
    from paper_2512_20210_b200.lora import bgmv_layers
    xl = torch.randn(2, T, 4096, device="cuda").to(torch.bfloat16)
    yl = torch.randn(2, 2, T, 4096, device="cuda").to(torch.bfloat16)
    bgmv_layers(plan, 0, xl, [yl[:, 0], yl[:, 1]])
    from paper_2512_20210_b200 import _native as N
    # warp items: jobs of 1..4 tokens (6 tokens per adapter -> 3 + 3), 256 B
    # pages (page entries by table loads) and widths that are not multiples
    # of 256 / 512
    from paper_2512_20210_b200.lora import ModelShape
    for tpa in (1, 3, 6):
        tan = synth.token_assignment(cfg.n_adapters, tpa)
        xn = torch.randn(len(tan), 4096, device="cuda").to(torch.bfloat16)
        yn = [torch.randn(len(tan), 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
        bgmv_layer(BatchPlan(s.store, tan), 1, xn, yn)
    shp = ModelShape(2, (1000, 1000), (520, 1048), torch.bfloat16)
    sw = Setup(synth.DecodeConfig("san_w", shp, [5, 16, 64, 33, 80], 2, 256))
    taw = synth.token_assignment(5, 3)  # (rank 64 / 80: split expand pairs in single-layer calls)
    xw = torch.randn(len(taw), 1000, device="cuda").to(torch.bfloat16)
    bgmv_layer(BatchPlan(sw.store, taw), 1, xw, [torch.randn(len(taw), 520, device="cuda").to(torch.bfloat16),
                                                torch.randn(len(taw), 1048, device="cuda").to(torch.bfloat16)])
    # cluster kernel and the hybrid pair
    for impl in (2, 3):
        N.check(N.lib().plora_debug_set_bgmv_impl(impl))
        pc = BatchPlan(s.store, ta)
        bgmv(pc, 1, 0, x, ys[0])
        bgmv_layer(pc, 0, x, ys)
        bgmv_layers(pc, 0, xl, [yl[:, 0], yl[:, 1]])
    # streaming decode kernel, 4- and 8-token jobs
    N.check(N.lib().plora_debug_set_bgmv_impl(1))
    bgmv_layer(plan, 1, x, ys)
    ta8 = synth.token_assignment(cfg.n_adapters, 6)
    x8 = torch.randn(len(ta8), 4096, device="cuda").to(torch.bfloat16)
    y8 = [torch.randn(len(ta8), 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
    plan8 = BatchPlan(s.store, ta8)
    bgmv_layer(plan8, 0, x8, y8)
    bgmv_layers(plan, 0, xl, [yl[:, 0], yl[:, 1]])
    N.check(N.lib().plora_debug_set_bgmv_impl(0))
    # fused prefill on 512 B / 1 KiB pages (the gather4 thresholds)
    from paper_2512_20210_b200.lora import ModelShape
    for page in (512, 1024):
        shape = ModelShape(2, (1024, 1024), (1024, 512), torch.bfloat16)
        cs = synth.DecodeConfig("san", shape, [16, 64, 128, 5], 1, page)
        ss = Setup(cs)
        sg = synth.segment_assignment(4, 150)
        xx = torch.randn(len(sg), 1024, device="cuda").to(torch.bfloat16)
        pf = BatchPlan(ss.store, sg)
        sgmv_fused(pf, 1, 0, xx, torch.randn(1024, 1024, device="cuda").to(torch.bfloat16),
                   torch.empty(len(sg), 1024, device="cuda", dtype=torch.bfloat16))
        sgmv(pf, 1, 1, xx, torch.randn(len(sg), 512, device="cuda").to(torch.bfloat16))
    # the persistent SGMV expand (a measured alternative, flag bit 20): gather4 pages, 64 B pages (cp.async)
    for page in (2048, 64):
        shape = ModelShape(2, (1024, 1024), (1024, 1024), torch.bfloat16)
        ss = Setup(synth.DecodeConfig("san", shape, [16, 64, 128, 5], 1, page))
        sg = synth.segment_assignment(4, 150)
        xx = torch.randn(len(sg), 1024, device="cuda").to(torch.bfloat16)
        N.check(N.lib().plora_debug_set_sgmv_flags(1 << 20))
        sgmv_layer(BatchPlan(ss.store, sg), 1, xx, [torch.randn(len(sg), 1024, device="cuda").to(torch.bfloat16)
                                                    for _ in range(2)])
        N.check(N.lib().plora_debug_set_sgmv_flags(0))
    # many-token adapters routed to the SGMV path (child plan, second stream)
    import numpy as np
    N.check(N.lib().plora_debug_set_route_tokens(16))
    tr = np.concatenate([np.full(20, 1, np.int32), np.arange(2, cfg.n_adapters, dtype=np.int32)])
    xr = torch.randn(len(tr), 4096, device="cuda").to(torch.bfloat16)
    yr = [torch.randn(len(tr), 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
    pr = BatchPlan(s.store, tr)
    bgmv(pr, 1, 0, xr, yr[0])
    bgmv_layer(pr, 0, xr, yr)
    xrl = torch.randn(2, len(tr), 4096, device="cuda").to(torch.bfloat16)
    yrl = torch.randn(2, 2, len(tr), 4096, device="cuda").to(torch.bfloat16)
    bgmv_layers(pr, 0, xrl, [yrl[:, 0], yrl[:, 1]])
    N.check(N.lib().plora_debug_set_route_tokens(160))
    # TP halves with the fused peer-write all-gather, two emulated ranks
    from paper_2512_20210_b200.tp import bgmv_tp_expand_wait, bgmv_tp_shrink_push
    vgs = [torch.zeros(2, T, rs, device="cuda") for _ in range(2)]
    fl = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    for i in range(2):
        bgmv_tp_shrink_push(plan, 0, 1, i, 2, x, [v.data_ptr() for v in vgs], [f.data_ptr() for f in fl])
    for i in range(2):
        bgmv_tp_expand_wait(plan, 0, 1, i, 2, vgs[i], fl[i], ys[1][:, i * 2048:(i + 1) * 2048])
    # predict_all on the GPU
    from paper_2512_20210_b200.predictor import OnlinePredictor, OnlinePredictorConfig, PredictorConfig
    pred = OnlinePredictor(OnlinePredictorConfig(model=PredictorConfig(num_adapters=50),
                                                 train_every=10 ** 9), 1)
    for a in range(50):
        pred.observe(a, float(a))
    pred.set_device(0)
    pred.predict_arrays(2000.0)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
