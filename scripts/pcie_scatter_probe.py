"""Prefetch path evidence: the page scatter of one adapter image from pinned
host memory into the HBM arena, both ways the engine can move it —
PLORA_COPY_SM (page_scatter_h2d_kernel reading mapped pinned memory over
PCIe; run under ncu for its PCIe / DRAM bytes) and PLORA_COPY_CE
(cudaMemcpyAsync per contiguous physical run) — timed with CUDA events.
Llama-7B q/v adapters of rank 64 (64 MiB) at 2 KiB and 2 MiB pages, tables
scattered by the churn prologue."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore  # noqa: E402

out = {}
for page in (2048, 2 << 20):
    cfg = synth.DecodeConfig("pcie", synth.cfg2().shape, [64] * 8, 1, page)
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, 8)
    img = synth.adapter_image(cfg.shape, 64, 0).view(torch.uint8).contiguous().pin_memory()
    nbytes = img.numel()
    for a in range(8):
        store.register(a, 64)
    res = {}
    for name, mode in (("sm", N.PLORA_COPY_SM), ("ce", N.PLORA_COPY_CE)):
        for a in range(2):
            store.write_pages(a, img, mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for a in range(8):
            store.write_pages(a, img, mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 8
        res[name] = {"ms_per_adapter": ms, "gbs": nbytes / (ms / 1e3) / 1e9}
    out[f"page_{page}"] = {"adapter_bytes": nbytes, **res}
    del store, pool
print(json.dumps(out, indent=1))
