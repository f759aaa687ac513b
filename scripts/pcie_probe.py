"""Pinned host <-> device copy bandwidth on the box, for the e2e pipeline's
chunking: H2D alone, D2H alone and both at once, at several copy sizes and
stream counts (CUDA events around the whole batch)."""
import json

import torch

TOTAL = 192 << 20  # bytes per direction per trial (one cfg2 step's H2D)


def run(sizes, h2d=True, d2h=False, streams=1):
    out = {}
    for sz in sizes:
        n = TOTAL // sz
        hs = [torch.empty(sz, dtype=torch.uint8).pin_memory() for _ in range(n)]
        ds = [torch.empty(sz, dtype=torch.uint8, device="cuda") for _ in range(n)]
        ho = [torch.empty(sz, dtype=torch.uint8).pin_memory() for _ in range(n)]
        st = [torch.cuda.Stream() for _ in range(2 * streams)]
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in st:
                s.wait_stream(torch.cuda.current_stream())
            for i in range(n):
                if h2d:
                    with torch.cuda.stream(st[i % streams]):
                        ds[i].copy_(hs[i], non_blocking=True)
                if d2h:
                    with torch.cuda.stream(st[streams + i % streams]):
                        ho[i].copy_(ds[(i + n // 2) % n], non_blocking=True)
            for s in st:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[f"{sz >> 20}MiB"] = round(TOTAL / ms / 1e6, 1)
        del hs, ds, ho
    return out


sizes = [2 << 20, 8 << 20, 32 << 20]
res = {"h2d_only_gbs": run(sizes), "d2h_only_gbs": run(sizes, h2d=False, d2h=True),
       "both_gbs_per_direction": run(sizes, d2h=True), "h2d_2streams": run(sizes, streams=2),
       "both_2streams": run(sizes, d2h=True, streams=2)}
print(json.dumps(res))
