"""Benchmark: paged multi-LoRA decode at Llama-7B shapes (BASELINE.json configs[1]).

One step = one decode step of the hot path: the paged BGMV applied to all
32 layers × {q, v} = 64 (layer, proj) calls for a batch of 256 tokens over 128
resident adapters with ranks [8,16,32,64][a % 4] (2 tokens per adapter, in
shuffled order), weights read out of the 2 KiB-page HBM arena through the
device page table.  Synthetic, seeded data (paper_2512_20210_b200.synth).

  value   tokens/s with inputs resident in HBM (CUDA events, K steps)
  e2e     the same metric through the public API from pinned HOST buffers:
          per step H2D of x (all layers) and y, the plan upload, 64 calls, D2H y,
          pipelined per layer over copy / compute streams in one CUDA graph
  roofline  the BGMV kernel: algorithmic bytes per launch / mean launch time
  cpu_baseline  the CPU oracle port (oracle/lora_oracle.c) on a bounded sample

Multi-GPU (torchrun): request/adapter sharding — every rank serves its own
batch from its own pool (no data-path collective), weak scaling; time = max
over ranks.  ``--impl reference`` times the CPU reference path instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "paged multi-LoRA tokens/sec at Llama-7B shapes; BGMV HBM GB/s vs peak"
UNIT = "tokens/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def load_tensor_peak(sustained: bool = False):
    """Dense bf16 TFLOP/s: the burst figure for a kernel timed alone, the
    sustained one (4 s back to back, power-capped clocks) for a long step."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if sustained and "bf16_tflops_sustained" in d:
            return "measured sustained", d["bf16_tflops_sustained"]
        return "measured", d.get("bf16_tflops", 1590.0)
    return "fallback", 1590.0


def call_bytes(shape, ranks, proj, n_tokens):
    """Algorithmic bytes of one (layer, proj) call: each adapter's A and Bᵀ
    block once + x read + y read-modify-write."""
    w = sum(r * (shape.d_in[proj] + shape.d_out[proj]) for r in ranks) * shape.esize
    return w + n_tokens * shape.d_in[proj] * shape.esize + 2 * n_tokens * shape.d_out[proj] * shape.esize


class ClockSampler:
    """NVML sampling of SM clocks / throttle reasons during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._dev = device_index
        self._period = period_s
        self._thread = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self._dev)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
            }

            def run():
                while not self._stop.is_set():
                    self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    for b, n in names.items():
                        if bits & b:
                            self.reasons.add(n)
                    time.sleep(self._period)

            self._thread = threading.Thread(target=run, daemon=True)
            self._thread.start()
        except Exception as e:  # NVML missing: record why
            self.reasons.add(f"nvml-unavailable: {e.__class__.__name__}")
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


# --------------------------------------------------------------------- CPU arms
def cfg2_config(page_bytes: int, world: int) -> dict:
    """The workload both arms print (identical dict: the driver compares them)."""
    return {"workload": ("cfg2 decode BGMV: 256 tokens / 128 adapters per GPU, "
                         "r=[8,16,32,64][a%4], Llama-7B q/v (32 layers x 2 projections "
                         "per step)"),
            "page_bytes": page_bytes, "tokens_per_step_per_gpu": 256,
            "parallelism": f"request-sharded x{world} (no collective)",
            "l2": "inputs > L2: 3.84 GB of adapter pages + 192 MiB activations per step"}


def run_reference(args):
    """--impl reference: the reference-side CPU path of the decode step on this
    box's host cores — oracle/cpu_arm.py: every page table from the
    reference's own PagePool (oracle/_ref/libref.so), the paged LoRA apply by
    the C restatement with all host threads, all 64 (layer, proj) calls of
    every step (no extrapolation).  The product package is never imported."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_arm
    nthreads = os.cpu_count() or 1
    t0 = time.perf_counter()
    cpu = cpu_arm.CpuDecodeStep(n_layers=32, page_bytes=args.page_bytes, nthreads=nthreads)
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        cpu.step()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        cpu.step()
        times.append(time.perf_counter() - t)
    step_s = statistics.mean(times)
    value = cpu.n_tokens / step_s
    sample = (f"the full cfg2 decode step: 64 (layer, proj) calls over the 32-layer catalog "
              f"(3.84 GB of 2 KiB pages laid out by the reference PagePool), every step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": cfg2_config(args.page_bytes, max(1, args.gpus)),  # the GPU arm's config at the same N
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_arm.cpu_model_name()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup_s,
        "note": "the reference ships no LoRA arithmetic (SPEC.md:70,341): the CPU arm is the "
                "oracle port (oracle/lora_oracle.c) reading weights through page tables made by "
                "the reference's own PagePool (oracle/_ref/libref.so); libplora.so is not loaded",
    }
    print(json.dumps(line))


# --------------------------------------------------------------------- GPU arm
def dist_setup():
    """(world, rank, local device index) from the torchrun environment; one
    process per GPU over NCCL.  PLORA_BENCH_BACKEND=gloo with more ranks than
    GPUs (ranks sharing a device, LOCAL_RANK modulo the device count) only
    exercises the multi-rank code path on a one-GPU box (tests/; its numbers
    mean nothing)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("PLORA_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_20210_b200 import synth
    from paper_2512_20210_b200.lora import (AdapterStore, BatchPlan, bgmv, bgmv_layer,
                                            kernel_launch_count, sgmv, sgmv_layer)

    world, rank, local = dist_setup()

    prefill = args.workload == "cfg3"
    cfg = synth.cfg3(page_bytes=args.page_bytes) if prefill else synth.cfg2(page_bytes=args.page_bytes)
    op = sgmv if prefill else bgmv
    shape = cfg.shape
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, shape, cfg.n_adapters, device=local)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        img = synth.adapter_image(shape, r, a + 1000 * rank, device=f"cuda:{local}")
        store.write_pages(a, img.view(torch.uint8))  # D2D page scatter
        store.publish(a)
        del img
    if prefill:
        ta = synth.segment_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    else:
        ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter,
                                    seed=synth.SEED_ASSIGN + rank)
    T = len(ta)
    L, NP = shape.n_layers, shape.n_proj
    plan = BatchPlan(store, ta)
    dev = torch.device("cuda", local)
    x = torch.randn(L, T, 4096, device=dev).to(torch.bfloat16)
    y = torch.randn(L * NP, T, 4096, device=dev).to(torch.bfloat16)
    stream = torch.cuda.current_stream()

    # both projections of a layer (they read the same x) in one call unless
    # --per-proj: decode one launch, prefill one shrink + reduction + expand
    fused = not args.per_proj
    LPS = NP if not fused else 1  # calls per layer
    layer_op = sgmv_layer if prefill else bgmv_layer

    mlp = max(1, args.layers_per_launch) if not prefill else 1
    if mlp > 1:
        from paper_2512_20210_b200.lora import bgmv_layers
        yv = y.view(L, NP, T, 4096)
        LPS = 1.0 / mlp  # launches per layer

    def step(ev=None):
        if mlp > 1:
            for i, l0 in enumerate(range(0, L, mlp)):
                if ev is not None:
                    ev[2 * i].record()
                n = min(mlp, L - l0)
                bgmv_layers(plan, l0, x[l0:l0 + n], [yv[l0:l0 + n, p] for p in range(NP)])
                if ev is not None:
                    ev[2 * i + 1].record()
            return
        for l in range(L):
            if fused:
                if ev is not None:
                    ev[2 * l].record()
                layer_op(plan, l, x[l], [y[l * NP + p] for p in range(NP)])
                if ev is not None:
                    ev[2 * l + 1].record()
                continue
            for p in range(NP):
                if ev is not None:
                    ev[2 * (l * NP + p)].record()
                op(plan, l, p, x[l], y[l * NP + p])
                if ev is not None:
                    ev[2 * (l * NP + p) + 1].record()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # The decode step runs as one CUDA graph (as serving engines run decode):
    # `graph` holds the 64 calls back to back (consecutive launches overlap
    # through programmatic dependent launch) and is what `value` times;
    # `tgraph` is the same step with an event pair around every call, used
    # only for the per-launch kernel duration of the roofline (the events
    # serialise the launches, so it is not used for throughput).
    graph = tgraph = None
    gevs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2 * L * NP)]
    n_graph0 = kernel_launch_count()
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        per_replay = kernel_launch_count() - n_graph0
        tgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(tgraph):
            step(gevs)
        for _ in range(2):
            graph.replay()
            tgraph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * L * NP)] for _ in range(K)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = kernel_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for k in range(K):
            if graph is not None:
                graph.replay()
            else:
                step(evs[k])
        end.record(stream)
        torch.cuda.synchronize()
    if graph is not None:
        launches = per_replay * K  # kernels inside each replayed graph
        kern_ms = []
        for _ in range(3):  # per-launch durations (separate, serialised replays)
            tgraph.replay()
            torch.cuda.synchronize()
            kern_ms += [gevs[2 * i].elapsed_time(gevs[2 * i + 1]) for i in range(int(L * LPS))]
    else:
        launches = kernel_launch_count() - n0
        kern_ms = [evs[k][2 * i].elapsed_time(evs[k][2 * i + 1])
                   for k in range(K) for i in range(int(L * LPS))]
    step_ms = start.elapsed_time(end) / K
    mean_kern_ms = statistics.mean(kern_ms)
    # the same step with one plora_bgmv_layer launch per layer (the form a
    # model's forward uses when each layer's input depends on the previous one)
    per_layer_ms = None
    if mlp > 1 and graph is not None:
        def step_layer():
            for l in range(L):
                bgmv_layer(plan, l, x[l], [y[l * NP + p] for p in range(NP)])
        for _ in range(3):
            step_layer()
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            step_layer()
        g1.replay()
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(K):
            g1.replay()
        p1.record(stream)
        torch.cuda.synchronize()
        per_layer_ms = p0.elapsed_time(p1) / K
    if world > 1:
        t = torch.tensor([step_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = t.item()
    value = world * T / (step_ms / 1e3)

    # ---- e2e through the public API from pinned host buffers.  The step is
    # pipelined per layer over three streams — H2D of layer l's x and y rows,
    # the layer's calls once they landed, D2H of its y rows once computed —
    # and captured as one CUDA graph (the copies overlap the kernels and each
    # other: PCIe is full duplex).
    e2e = None
    if not args.no_e2e and not prefill:
        xh = x.cpu().pin_memory()
        yh = y.cpu().pin_memory()
        yout = torch.empty_like(yh).pin_memory()
        hs, ds = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ein = [torch.cuda.Event() for _ in range(L)]
        eout = [torch.cuda.Event() for _ in range(L)]

        def layer(l):
            if fused:
                bgmv_layer(plan, l, x[l], [y[l * NP + p] for p in range(NP)])
            else:
                for p in range(NP):
                    op(plan, l, p, x[l], y[l * NP + p])

        G = max(1, args.e2e_group)  # layers per copy (bigger PCIe transfers, longer pipeline fill)

        def e2e_step():
            cur = torch.cuda.current_stream()
            hs.wait_stream(cur)
            ds.wait_stream(cur)
            with torch.cuda.stream(hs):
                for l0 in range(0, L, G):
                    l1 = min(L, l0 + G)
                    x[l0:l1].copy_(xh[l0:l1], non_blocking=True)
                    y[l0 * NP:l1 * NP].copy_(yh[l0 * NP:l1 * NP], non_blocking=True)
                    ein[l0].record(hs)
            for l in range(L):
                if l % G == 0:
                    cur.wait_event(ein[l])
                layer(l)
                if (l + 1) % G == 0 or l + 1 == L:
                    eout[l - l % G].record(cur)
            with torch.cuda.stream(ds):
                for l0 in range(0, L, G):
                    l1 = min(L, l0 + G)
                    ds.wait_event(eout[l0])
                    yout[l0 * NP:l1 * NP].copy_(y[l0 * NP:l1 * NP], non_blocking=True)
            cur.wait_stream(hs)
            cur.wait_stream(ds)

        egraph = None
        if not args.no_graph:
            e2e_step()
            torch.cuda.synchronize()
            egraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(egraph):
                e2e_step()
        Ke = max(3, min(K, 10))
        for it in range(Ke + 2):
            if it == 2:
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            plan.update(ta)  # same batch shape: the captured graphs stay valid
            if egraph is not None:
                egraph.replay()
            else:
                e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / Ke
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = t.item()
        plan_bytes = 32 * cfg.n_adapters + 4 * T + 8 * 2 * 3000
        e2e = {"value": world * T / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": xh.numel() * 2 + yh.numel() * 2 + plan_bytes,
               "d2h_bytes_per_step": yout.numel() * 2, "ms_per_step": e2e_ms,
               "pipeline": f"per {G} layer(s): H2D | calls | D2H on three streams, one CUDA graph"}

    # ---- roofline of the op (per (layer, proj) call, mean over the timed region)
    per_call = statistics.mean(call_bytes(shape, cfg.ranks, p, T) for p in range(NP))
    if fused:  # one launch applies every projection of the layer (x read once)
        per_call = sum(call_bytes(shape, cfg.ranks, p, T) for p in range(NP)) - \
            (NP - 1) * T * shape.d_in[0] * shape.esize
    if prefill:  # every adapter serves one 512-token segment; weights read once per tile
        toks = cfg.tokens_per_adapter
        per_proj_flops = [sum(2 * toks * r * (shape.d_in[p] + shape.d_out[p]) for r in cfg.ranks)
                          for p in range(NP)]
        flops = sum(per_proj_flops) if fused else statistics.mean(per_proj_flops)
    peak, peak_kind = load_peaks()
    # average launch duration over the timed region: the step is the L·NP
    # launches back to back (overlapping through PDL), nothing else
    avg_launch_ms = step_ms / (L * LPS)
    if mlp > 1:  # one launch serves mlp layers: its bytes are mlp layers' worth
        per_call *= mlp
    achieved = per_call / (avg_launch_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "sgmv_traffic.json" if prefill else "bgmv_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not prefill:
        from oracle import cpu_arm
        nthreads = os.cpu_count() or 1
        per_call_s, n = cpu_arm.CpuDecodeStep(n_layers=2, nthreads=nthreads).sample_calls(
            args.cpu_sample_s)
        cpu = {"value": T / (per_call_s * L * NP), "unit": UNIT, "cores": nthreads, "kind": "port",
               "cpu_model": cpu_arm.cpu_model_name(),
               "sample": f"{n} cfg2 (layer,proj) calls of the CPU oracle over reference-PagePool "
                         f"tables (2-layer catalog: identical per-call work), scaled to the "
                         f"64-call step ({per_call_s * 1e3:.1f} ms/call)"}

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": max(args.warmup, 3), "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": ({"workload": ("cfg3 prefill SGMV (tcgen05): 32 segments x 512 tokens per GPU, "
                                 "r=[16,64,128][s%3], Llama-7B q/v (32 layers x 2 projections "
                                 "per step)"),
                    "page_bytes": args.page_bytes, "tokens_per_step_per_gpu": T,
                    "parallelism": f"request-sharded x{world} (no collective)",
                    "l2": "inputs > L2: 2.1 GiB of adapter pages + 12 GiB activations per step"}
                   if prefill else cfg2_config(args.page_bytes, world)),
        "impl_detail": {"cuda_graph": graph is not None, "launches_per_layer": LPS,
                        "launch": (f"plora_bgmv_layers: {mlp} layers per call (inputs resident)")
                                  if mlp > 1 else "plora_bgmv_layer: one call per layer"},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": per_call,
                     "avg_launch_us": avg_launch_ms * 1e3,
                     "serialized_launch_us": mean_kern_ms * 1e3,
                     "achieved_serialized": per_call / (mean_kern_ms / 1e3) / 1e9,
                     "launch_time": "step time / launches per step (CUDA events on the launching "
                                    "stream around the timed graph replays); serialized = the same "
                                    "launches bracketed one by one by events (no PDL overlap)"},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if mlp > 1 and not prefill:  # the decode launch's split (plora_bgmv_layers)
        import ctypes as C
        from paper_2512_20210_b200 import _native as N
        info = (C.c_double * 4)()
        N.check(N.lib().plora_debug_plan_hybrid(plan.handle, info))
        if info[0] == 0:
            line["roofline"]["kernels"] = (
                "one plora_bgmv_layers call = bgmv_warp_shrink_kernel (S items: <= 8 rank rows of one "
                "job, v = x·Aᵀ in fp32) then bgmv_warp_expand_kernel (E items: <= 512 output columns "
                "over every rank row, y += scale·v·Bᵀ), chained by programmatic dependent launch, both "
                "over all 32 layers (grid.y); achieved = the step's algorithmic bytes / the call's time")
        if info[0] > 0:
            line["roofline"]["kernels"] = (
                f"the launch pair of plora_bgmv_layers: bgmv_cluster_kernel ({int(info[2])} 4-CTA "
                f"clusters, {1 - info[1]:.3f} of the weight rows) and, concurrently on the "
                f"{int(info[0])} SMs the clusters leave idle, bgmv_stream_kernel ({int(info[3])} CTAs, "
                f"{info[1]:.3f}); achieved = the step's algorithmic bytes / the pair's time")
    if per_layer_ms is not None:
        lb = per_call / mlp  # one layer's bytes
        line["per_layer_launch"] = {
            "value": world * T / (per_layer_ms / 1e3), "ms_per_step": per_layer_ms,
            "avg_launch_us": per_layer_ms * 1e3 / L,
            "roofline_frac": lb / (per_layer_ms / L / 1e3) / 1e9 / peak,
            "note": "32 plora_bgmv_layer launches per step (one per layer), same plan and inputs"}
    if prefill:
        _, tpeak = load_tensor_peak()
        tach = flops / (avg_launch_ms / 1e3) / 1e12
        line["roofline"]["tensor"] = {"achieved": tach, "peak": tpeak, "unit": "TFLOP/s",
                                      "frac": tach / tpeak, "flops_per_launch": flops}
    print(json.dumps(line))


# --------------------------------------------------------------------- cfg4
def h2d_roof_gbs(dev, nbytes=256 << 20):
    """Pinned host -> HBM copy bandwidth (the prefetch roof), measured here."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 4 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9


def run_cfg4(args):
    """BASELINE configs[3]: synthetic Azure-Functions-like trace over 1000
    distinct adapters held in a pinned host adapter store, LSTM-driven page
    prefetch overlapped with the paged BGMV; request-sharded over ranks
    (adapter k -> rank k mod N).  The same trace is served three times from a
    cold pool — prediction source lstm (the online predictor), oracle (the
    future arrivals, engine.cpp:555-562) and off (demand loads only) — and
    each run reports hit rate, demand-stall time, prefetch traffic and the
    per-interval prediction accuracy (engine.cpp:598-633)."""
    import torch
    import torch.distributed as dist

    from paper_2512_20210_b200 import synth
    from paper_2512_20210_b200.engine import EngineConfig
    from paper_2512_20210_b200.hoststore import HostAdapterStore
    from paper_2512_20210_b200.lora import ModelShape, bgmv_layer, kernel_launch_count
    from paper_2512_20210_b200.predictor import OnlinePredictorConfig, PredictorConfig
    from paper_2512_20210_b200.prefetch import PrefetchPolicy
    from paper_2512_20210_b200.serving import DecodeServer, ServerConfig, shard_keys
    from paper_2512_20210_b200.workload import SyntheticProfile, generate_synthetic

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    shape = ModelShape.llama7b_qv()
    n_total = args.cfg4_adapters
    keys = shard_keys(n_total, rank, world)
    ranks = [(8, 16, 32, 64)[k % 4] for k in keys]
    # the host adapter store: every local adapter's own bytes, pinned and
    # page-aligned (distinct images: each transfer moves that adapter's data)
    t0 = time.perf_counter()
    hstore = HostAdapterStore.create([shape.adapter_bytes(r) for r in ranks], ranks,
                                     align=args.cfg4_page_bytes)
    for i, (k, r) in enumerate(zip(keys, ranks)):
        img = synth.adapter_image(shape, r, k, device=dev)
        hstore.view(i).copy_(img.view(torch.uint8), non_blocking=True)
        del img
    torch.cuda.synchronize()
    store_s = time.perf_counter() - t0
    # trace: rate scales with N so every rank sees the same per-GPU load
    prof = SyntheticProfile(num_adapters=n_total, base_rate=args.cfg4_rate * world,
                            hot_set_size=args.cfg4_hot, hot_rotation_s=args.cfg4_rotation_s,
                            hot_share=0.9)
    W, K, T = max(args.warmup, 3), args.steps, 256
    # steady state: the LSTM buckets counts per 1 s over a 30-interval window
    # (predictor.hpp:46), so the serving loop first runs cfg4_warm_s seconds
    # of trace time (untimed) before the W warm-up and K timed steps
    pre = int(args.cfg4_warm_s * args.cfg4_rate / T)
    W += pre
    need = (W + K + 2) * T * world
    duration = need / prof.base_rate * 1.3 + 10
    tr = generate_synthetic(prof, duration, seed=42)
    mine = np.nonzero(tr.adapter % world == rank)[0]
    local_of = {k: i for i, k in enumerate(keys)}
    arr_keys = np.asarray([local_of[int(k)] for k in tr.adapter[mine]], np.uint32)
    arr_t = tr.arrival_ms[mine]
    if len(arr_keys) < (W + K) * T:
        raise RuntimeError("trace too short for the requested steps")
    future = [np.sort(arr_t[arr_keys == i]) for i in range(len(keys))]
    stream = torch.cuda.current_stream()
    roof = h2d_roof_gbs(dev)
    modes = [m for m in args.cfg4_modes.split(",") if m]
    results = {}
    for mode in modes:
        pol = PrefetchPolicy(staging_fraction=args.cfg4_staging)
        # the reference trains every 100 observations at 50 requests/s
        # (defaults.ini:20, 68): the same training cadence per second of trace
        train_every = args.cfg4_train_every or max(100, int(round(100 * args.cfg4_rate / 50.0)))
        pcfg = OnlinePredictorConfig(model=PredictorConfig(num_adapters=len(keys)),
                                     interval_ms=1000.0, train_every=train_every, batch_size=64)
        scfg = ServerConfig(
            shape=shape, ranks=ranks, pool_bytes=int(args.cfg4_pool_gib * (1 << 30)),
            page_bytes=args.cfg4_page_bytes, batch_tokens=T, round_ms=100.0,
            engine=EngineConfig(policy=pol, chunk_bytes=8 << 20, prefetch_inflight_bytes=64 << 20,
                                prefetch=mode != "off"),
            predictor=pcfg, seed=42, device=local, prediction=mode)
        srv = DecodeServer(scfg, hstore.view, future=future)
        if srv.predictor is not None:
            if not args.cfg4_host_predictor:
                srv.predictor.set_device(local)  # predict_all on the GPU (FP64)
            srv.engine.attach_predictor(srv.predictor, asynchronous=True)
        # score intervals once the LSTM window (30 x 1 s) has seen 10 s of trace
        srv.engine.set_accuracy_interval(1000.0, warmup_ms=float(arr_t[0]) + 10000.0)

        def run_steps(k0, n, evs=None):
            for st_ in range(k0, k0 + n):
                a = arr_keys[st_ * T:(st_ + 1) * T]
                srv.step(a, float(arr_t[(st_ + 1) * T - 1]), events=evs[st_ - k0] if evs else None)

        tw = time.perf_counter()
        run_steps(0, W)
        if srv.predictor is not None:
            srv.engine.flush_predictor()
        torch.cuda.synchronize()
        warm_s = time.perf_counter() - tw
        st0 = srv.engine.stats()
        d0 = len(srv.engine.decisions())
        if world > 1:
            dist.barrier()
        evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(K)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = kernel_launch_count()
        tok0 = srv.stats["tokens"]
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            e0.record(stream)
            run_steps(W, K, evs)
            e1.record(stream)
            torch.cuda.synchronize()
        launches = kernel_launch_count() - n0
        tokens = srv.stats["tokens"] - tok0
        ms = e0.elapsed_time(e1)
        stall_ms = sum(a.elapsed_time(b) for a, b, _ in evs) / K
        bgmv_ms = sum(b.elapsed_time(c) for _, b, c in evs) / K
        st1 = srv.engine.stats()
        rows = srv.engine.decisions(d0)
        # BGMV alone: the last batch replayed with the engine idle
        srv.engine.sync()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(10):
            srv.apply(srv.last_batch)
        a1.record(stream)
        torch.cuda.synchronize()
        alone_ms = a0.elapsed_time(a1) / 10
        d = {k: st1[k] - st0[k] for k in ("arrivals", "hits", "demand_loads", "prefetch_issued",
                                            "promotions", "evictions", "admission_failures",
                                            "upgrades", "bytes_h2d", "transfer_ms",
                                            "prediction_rounds", "compactions")}
        tot = torch.tensor([ms, float(tokens)], device=dev, dtype=torch.float64)
        if world > 1:
            mx = tot.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = tot.clone()
            dist.all_reduce(sm, op=dist.ReduceOp.SUM)
            ms, tokens = mx[0].item(), sm[1].item()
        acts = {}
        for r_ in rows:
            acts[r_[1]] = acts.get(r_[1], 0) + 1
        results[mode] = {
            "value": tokens / (ms / 1e3), "ms_per_step": ms / K, "launches": launches,
            "hit_rate": d["hits"] / max(d["arrivals"], 1),
            "demand_stall_ms_per_step": stall_ms,
            "bgmv_ms_per_step_with_prefetch": bgmv_ms, "bgmv_ms_per_step_alone": alone_ms,
            "overlap": alone_ms / max(bgmv_ms, 1e-9),
            "bytes_h2d_per_step": d["bytes_h2d"] / K,
            "h2d_gbs_over_timed_region": d["bytes_h2d"] / (ms / 1e3) / 1e9,
            "link_busy_frac": d["bytes_h2d"] / (ms / 1e3) / 1e9 / roof,
            "interval_accuracy": st1["acc_sum"] / max(st1["acc_intervals"], 1),
            "accuracy_intervals": st1["acc_intervals"],
            "accuracy_tp_fp_fn": [st1["acc_tp"], st1["acc_fp"], st1["acc_fn"]],
            "predictor_busy_ms": st1["predictor_ms"], "trace_served_s": warm_s + ms / 1e3,
            "predictor": {"train_every": train_every, "predict_all": "host" if args.cfg4_host_predictor
                          else "gpu"},
            "decisions_in_timed_region": acts, "counters": d, "clocks": clk.summary()}
        del srv
        torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    head = results.get("lstm") or results[modes[0]]
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": (f"cfg4: generate_synthetic trace, {n_total} distinct adapters in a "
                                f"pinned host adapter store (r=[8,16,32,64][k%4], Llama-7B q/v), per "
                                f"GPU {len(keys)} adapters, 256-token decode steps, async LSTM "
                                f"predictor (predict_all on the GPU), page prefetch overlapped "
                                f"with BGMV"),
                   "pool_gib_per_gpu": args.cfg4_pool_gib, "page_bytes": args.cfg4_page_bytes,
                   "trace": {"base_rate_per_gpu": args.cfg4_rate, "hot_set_size": args.cfg4_hot,
                             "hot_rotation_s": args.cfg4_rotation_s, "hot_share": 0.9},
                   "host_store": {"bytes_per_gpu": hstore.total_bytes(), "build_s": store_s,
                                  "distinct_images": len(keys)},
                   "parallelism": f"request-sharded x{world} (adapter k -> rank k mod N)",
                   "l2": "inputs > L2 (adapter pages)"},
        "gpu_launches": head["launches"],
        "prefetch": {"h2d_roof_gbs": roof, "trace_warm_s": args.cfg4_warm_s,
                     "untimed_serving_steps": pre, "by_prediction_source": results},
        "clocks": head["clocks"],
    }
    print(json.dumps(line))


# --------------------------------------------------------------------- cfg5
def run_cfg5(args):
    """BASELINE configs[4]: Llama-2-70B q/v (q 8192 -> 8192, v 8192 -> 1024)
    tensor-parallel LoRA: every rank serves the same 256 decode tokens; rank i
    shrinks its r/N rows, the shard outputs are all-gathered (NCCL over
    NVLink) and rank i expands into its d_out/N output columns.  80 layers x
    2 projections per step, captured in one CUDA graph (collectives included).
    Strong scaling: the total work is fixed as N grows."""
    import torch
    import torch.distributed as dist

    from paper_2512_20210_b200 import synth
    from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, kernel_launch_count
    from paper_2512_20210_b200.tp import TensorParallelLoRA

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    cfg = synth.cfg5(n_layers=args.cfg5_layers, page_bytes=args.page_bytes)
    shape = cfg.shape
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, shape, cfg.n_adapters, device=local)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        img = synth.adapter_image(shape, r, a, device=dev)  # identical on every rank
        store.write_pages(a, img.view(torch.uint8))
        store.publish(a)
        del img
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    L, NP = shape.n_layers, shape.n_proj
    plan = BatchPlan(store, ta)
    tp = TensorParallelLoRA(plan, rank, world, allgather=args.cfg5_allgather)
    x = torch.randn(L, T, shape.d_in[0], device=dev).to(torch.bfloat16)
    ys = [torch.randn(L, T, shape.d_out[p] // world, device=dev).to(torch.bfloat16)
          for p in range(NP)]

    def step():
        for l in range(L):
            for p in range(NP):
                tp(l, p, x[l], ys[p][l])

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    n_g0 = kernel_launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    per_replay = kernel_launch_count() - n_g0
    graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    K = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(K):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    # per-rank algorithmic bytes of one (layer, proj) call: its A rows, its Bᵀ
    # columns, x, its y shard RMW
    split = None
    fused_ms = None
    rank0 = {}
    if world == 1:  # the per-rank halves themselves (shrink, copy, expand) at TP = 1
        tps = TensorParallelLoRA(plan, 0, 1, force_split=True)

        def step_split():
            for l in range(L):
                for p in range(NP):
                    tps(l, p, x[l], ys[p][l])

        for _ in range(3):
            step_split()
        torch.cuda.synchronize()
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            step_split()
        g2.replay()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(K):
            g2.replay()
        s1.record(stream)
        torch.cuda.synchronize()
        split = s0.elapsed_time(s1) / K
        # the same halves with the all-gather fused into the shrink (peer-write
        # + arrival flags; at TP = 1 the peer is this GPU)
        tpf = TensorParallelLoRA(plan, 0, 1, force_split=True, allgather="fused")

        def step_fused():
            for l in range(L):
                for p in range(NP):
                    tpf(l, p, x[l], ys[p][l])

        for _ in range(3):
            step_fused()
        torch.cuda.synchronize()
        g4 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g4):
            step_fused()
        g4.replay()
        torch.cuda.synchronize()
        s0.record(stream)
        for _ in range(K):
            g4.replay()
        s1.record(stream)
        torch.cuda.synchronize()
        fused_ms = s0.elapsed_time(s1) / K
        # one rank's halves at TP = 2, 4, 8 (the collective excluded: rank 0
        # expands from a gathered buffer filled once by every rank's shrink)
        from paper_2512_20210_b200.tp import bgmv_tp_expand, bgmv_tp_shrink, tp_shard_rows
        rank0 = {}
        for n in (2, 4, 8):
            rs = tp_shard_rows(plan, n)
            vg = torch.zeros(NP, n, T, rs, dtype=torch.float32, device=dev)
            ysh = [torch.randn(L, T, shape.d_out[p] // n, device=dev).to(torch.bfloat16) for p in range(NP)]
            for p in range(NP):
                for i in range(n):
                    bgmv_tp_shrink(plan, 0, p, i, n, x[0], vg[p, i])

            def step_rank0(n=n, vg=vg, ysh=ysh):
                for l in range(L):
                    for p in range(NP):
                        bgmv_tp_shrink(plan, l, p, 0, n, x[l], vg[p, 0])
                        bgmv_tp_expand(plan, l, p, 0, n, vg[p], ysh[p][l])

            for _ in range(3):
                step_rank0()
            torch.cuda.synchronize()
            g3 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g3):
                step_rank0()
            g3.replay()
            torch.cuda.synchronize()
            s0.record(stream)
            for _ in range(K):
                g3.replay()
            s1.record(stream)
            torch.cuda.synchronize()
            t_ms = s0.elapsed_time(s1) / K
            b_call = statistics.mean(
                sum((r // n) * shape.d_in[p] + r * (shape.d_out[p] // n) for r in cfg.ranks) * 2
                + T * shape.d_in[p] * 2 + 2 * T * (shape.d_out[p] // n) * 2 for p in range(NP))
            rank0[f"tp{n}"] = {"us_per_call": t_ms * 1e3 / (L * NP),
                               "alg_bytes_per_call": b_call,
                               "hbm_frac": b_call / (t_ms / (L * NP) / 1e3) / 1e9 / load_peaks()[0]}
            del vg, ysh, g3
    per_call = statistics.mean(
        sum((r // world) * shape.d_in[p] + r * (shape.d_out[p] // world) for r in cfg.ranks) * 2
        + T * shape.d_in[p] * 2 + 2 * T * (shape.d_out[p] // world) * 2 for p in range(NP))
    peak, peak_kind = load_peaks()
    avg_call_ms = ms / (L * NP)
    gather_bytes = world * T * (max(cfg.ranks) // world) * 4
    line = {
        "metric": METRIC, "value": T / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": (f"cfg5 tensor-parallel LoRA, Llama-2-70B q/v (q 8192->8192, "
                                f"v 8192->1024), {L} layers x 2 per step, 256 tokens / "
                                f"{cfg.n_adapters} adapters, r=[8,16,64][a%3], TP={world}"),
                   "page_bytes": args.page_bytes,
                   "parallelism": f"tp{world} (S-LoRA all-gather: {args.cfg5_allgather})",
                   "cuda_graph": True, "all_gather_bytes_per_call": gather_bytes,
                   "l2": "inputs > L2: adapter pages of 160 (layer, proj) blocks per step"},
        "gpu_launches": per_replay * K,
        "roofline": {"bound": "hbm", "achieved": per_call / (avg_call_ms / 1e3) / 1e9,
                     "peak": peak, "unit": "GB/s",
                     "frac": per_call / (avg_call_ms / 1e3) / 1e9 / peak, "traffic": None,
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": per_call,
                     "avg_launch_us": avg_call_ms * 1e3,
                     "note": "per (layer, proj) call = shrink + all-gather + expand on one rank"},
        "tp_halves_at_tp1": None if split is None else {
            "ms_per_step": split, "us_per_call": split * 1e3 / (L * NP),
            "hbm_frac": per_call / (split / (L * NP) / 1e3) / 1e9 / peak,
            "note": "tp_shrink + tp_expand forced at TP=1 (the per-rank kernels of the N>1 path; "
                    "value above uses the fused data-parallel op at TP=1)"},
        "tp_fused_allgather_at_tp1": None if split is None else {
            "ms_per_step": fused_ms, "us_per_call": fused_ms * 1e3 / (L * NP),
            "hbm_frac": per_call / (fused_ms / (L * NP) / 1e3) / 1e9 / peak,
            "note": "plora_bgmv_tp_shrink_push + plora_bgmv_tp_expand_wait (peer-write all-gather, "
                    "arrival flags) forced at TP=1"},
        "tp_rank0_halves": None if split is None else {
            **rank0,
            "note": "rank 0's shrink + expand per (layer, proj) call at TP = N on one GPU, the "
                    "all-gather excluded (its v_gathered filled once by every rank's shrink)"},
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def run_cfg3f(args):
    """BASELINE configs[2] with the base projections fused in (SURVEY §8(f)
    row 3): per layer one plora_sgmv_fused_layer call computes, for q and v,
    y = x·W0ᵀ + scale·(x·Aᵀ)·Bᵀ for 32 segments × 512 tokens, r = 16/64/128,
    Llama-7B q/v (4096 -> 4096), 32 layers × 2 per step, one CUDA graph.
    Tensor-bound: the roofline is the measured dense bf16 peak."""
    import torch

    from paper_2512_20210_b200 import synth
    from paper_2512_20210_b200.lora import (AdapterStore, BatchPlan, kernel_launch_count,
                                            sgmv_fused_layer)

    dev = torch.device("cuda", 0)
    cfg = synth.cfg3(page_bytes=args.page_bytes)
    shape = cfg.shape
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(shape, r, a, device=dev).view(torch.uint8))
        store.publish(a)
    ta = synth.segment_assignment(32, 512)
    T = len(ta)
    L, NP = shape.n_layers, shape.n_proj
    plan = BatchPlan(store, ta)
    g = torch.Generator(device=dev).manual_seed(1234)
    x = torch.randn(L, T, shape.d_in[0], device=dev, generator=g).to(torch.bfloat16)
    w0 = [[(torch.randn(shape.d_out[p], shape.d_in[p], device=dev, generator=g) /
            shape.d_in[p] ** 0.5).to(torch.bfloat16) for p in range(NP)] for _ in range(L)]
    ys = [torch.empty(L, T, shape.d_out[p], device=dev, dtype=torch.bfloat16) for p in range(NP)]

    def step():  # per layer: one shrink for q and v (x read once), then a fused GEMM each
        for l in range(L):
            sgmv_fused_layer(plan, l, x[l], w0[l], [ys[p][l] for p in range(NP)], 1.0)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    n_g0 = kernel_launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    per_replay = kernel_launch_count() - n_g0
    graph.replay()
    torch.cuda.synchronize()
    K = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(K):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    calls = L * NP
    flops = statistics.mean(2.0 * T * shape.d_in[p] * shape.d_out[p] +
                            sum(2.0 * 512 * r * (shape.d_in[p] + shape.d_out[p]) for r in cfg.ranks)
                            for p in range(NP))
    kind, tpeak = load_tensor_peak(sustained=True)  # a 30 ms step of back-to-back GEMMs
    call_ms = ms / calls
    achieved = flops / (call_ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": T / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": K,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": ("cfg3 prefill with the base projection fused: y = x·W0ᵀ + "
                                "(x·Aᵀ)·Bᵀ, 32 segments x 512 tokens, r=[16,64,128][s%3], "
                                f"Llama-7B q/v 4096->4096, {L} layers x 2 calls per step "
                                "(per layer: one shrink + split reduction for both projections, "
                                "then one fused tcgen05 GEMM each)"),
                   "page_bytes": args.page_bytes, "cuda_graph": True,
                   "l2": "inputs > L2: 4 GiB of x, 2 GiB of base weights per step"},
        "gpu_launches": per_replay * K,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s",
                     "frac": achieved / tpeak, "traffic": None, "peak_kind": kind,
                     "flops_per_launch": flops, "avg_launch_us": call_ms * 1e3,
                     "launch_time": "step time / (layer, proj) calls per step (a layer = 4 launches)"},
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--page-bytes", type=int, default=2048)
    ap.add_argument("--cpu-sample-s", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the 64 calls eagerly")
    ap.add_argument("--e2e-group", type=int, default=2,
                    help="layers per host<->device copy in the e2e pipeline (profiles/r02o_e2e_group.txt)")
    ap.add_argument("--layers-per-launch", type=int, default=32,
                    help="decode: layers served by one plora_bgmv_layers launch (1 = one "
                         "plora_bgmv_layer launch per layer)")
    ap.add_argument("--per-proj", action="store_true",
                    help="decode: one launch per (layer, proj) instead of one per layer")
    ap.add_argument("--cfg5-layers", type=int, default=80)
    ap.add_argument("--cfg5-allgather", default="nccl", choices=["nccl", "fused"],
                    help="TP all-gather: NCCL between the halves, or fused into the shrink (peer-write)")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3", "cfg3f", "cfg4", "cfg5"],
                    help="cfg2 = decode BGMV (headline), cfg3 = prefill SGMV, "
                         "cfg3f = prefill with the base projection GEMM fused in, "
                         "cfg4 = trace-driven decode with LSTM prefetch, "
                         "cfg5 = tensor-parallel 70B (run under torchrun for N > 1)")
    ap.add_argument("--cfg4-adapters", type=int, default=1000)
    ap.add_argument("--cfg4-modes", default="lstm,oracle,off",
                    help="prediction sources served in turn (lstm, oracle, off)")
    ap.add_argument("--cfg4-train-every", type=int, default=0,
                    help="observations per LSTM train step (0: the reference's cadence per "
                         "second of trace, 100 at 50 req/s)")
    ap.add_argument("--cfg4-host-predictor", action="store_true",
                    help="run predict_all on the host threads instead of the GPU")
    ap.add_argument("--cfg4-pool-gib", type=float, default=16.0)
    ap.add_argument("--cfg4-page-bytes", type=int, default=2 << 20)
    ap.add_argument("--cfg4-staging", type=float, default=0.25)
    ap.add_argument("--cfg4-rate", type=float, default=4000.0, help="requests/s per GPU")
    ap.add_argument("--cfg4-hot", type=int, default=100)
    ap.add_argument("--cfg4-rotation-s", type=float, default=7.0)
    ap.add_argument("--cfg4-warm-s", type=float, default=40.0,
                    help="seconds of trace served (untimed) before the timed steps")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "cfg4":
        run_cfg4(args)
    elif args.workload == "cfg5":
        run_cfg5(args)
    elif args.workload == "cfg3f":
        run_cfg3f(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
