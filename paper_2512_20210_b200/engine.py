"""Real-time loading / prefetch engine (libplora ``plora_engine_*``).

The reference runs residency control inside its discrete-event
``Simulation`` (src/engine.cpp:197-333, 406-497, 515-571): demand loads at
arrival and admission, eviction by lowest score among idle residents,
predictor-driven prefetch into a staging budget, promotion at batch
boundaries, idle compaction.  Here the same decisions drive real page
scatters of pinned host images into the HBM arena on side streams, and the
device page table is published on the compute stream.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .lora import AdapterStore, current_stream_handle
from .prefetch import AdapterDynamics, PrefetchPolicy, Residency


class Admit(enum.IntEnum):
    loading = N.PLORA_ADMIT_LOADING
    ready = N.PLORA_ADMIT_READY
    failed = N.PLORA_ADMIT_FAILED


@dataclass
class EngineConfig:
    policy: PrefetchPolicy = None
    copy_mode: int = N.PLORA_COPY_AUTO
    prefetch: bool = True
    compaction: bool = True
    chunk_bytes: int = 1 << 20
    prefetch_inflight_bytes: int = 4 << 20

    def to_c(self) -> N.plora_engine_config:
        c = N.plora_engine_config()
        N.lib().plora_engine_config_default(C.byref(c))
        c.policy = (self.policy or PrefetchPolicy()).to_c()
        c.copy_mode = self.copy_mode
        c.prefetch = int(self.prefetch)
        c.compaction = int(self.compaction)
        c.chunk_bytes = self.chunk_bytes
        c.prefetch_inflight_bytes = self.prefetch_inflight_bytes
        return c


class PrefetchEngine:
    """Owner of residency for one AdapterStore (one GPU)."""

    def __init__(self, store: AdapterStore, cfg: Optional[EngineConfig] = None):
        self.store = store  # keep alive
        self.cfg = cfg or EngineConfig()
        h = C.c_void_p()
        N.check(N.lib().plora_engine_create(store.handle, C.byref(self.cfg.to_c()), C.byref(h)))
        self._h = h
        self._sources = {}  # keep host images alive
        self._predictor = None

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            N.lib().plora_engine_destroy(h)

    @property
    def handle(self):
        return self._h

    @staticmethod
    def _s(stream) -> int:
        return current_stream_handle() if stream is None else stream

    def set_source(self, adapter: int, host: torch.Tensor) -> None:
        """Register the adapter's packed image (host tensor, pinned for async/SM copies)."""
        host = host.contiguous()
        if host.is_cuda:
            raise ValueError("set_source expects a host tensor")
        self._sources[adapter] = host
        N.check(N.lib().plora_engine_set_source(self._h, adapter, host.data_ptr(),
                                                host.numel() * host.element_size()))

    def attach_predictor(self, predictor, asynchronous: bool = False) -> None:
        """asynchronous=True: the predictor runs on the engine's worker thread
        (rounds use the previous round's predictions)."""
        self._predictor = predictor
        N.check(N.lib().plora_engine_attach_predictor(
            self._h, predictor._h if predictor else None, int(asynchronous)))

    def flush_predictor(self) -> None:
        N.check(N.lib().plora_engine_flush_predictor(self._h))

    def on_arrival(self, adapter: int, now_ms: float, stream=None) -> bool:
        return bool(N.check(N.lib().plora_engine_on_arrival(self._h, adapter, now_ms,
                                                            self._s(stream))))

    def round(self, now_ms: float, stream=None) -> None:
        N.check(N.lib().plora_engine_round(self._h, now_ms, self._s(stream)))

    def set_predictions(self, probs) -> None:
        p = np.ascontiguousarray(probs, dtype=np.float64)
        N.check(N.lib().plora_engine_set_predictions(
            self._h, p.ctypes.data_as(C.POINTER(C.c_double)), len(p)))

    def acquire(self, adapter: int, now_ms: float, stream=None) -> Admit:
        return Admit(N.check(N.lib().plora_engine_acquire(self._h, adapter, now_ms,
                                                          self._s(stream))))

    def wait_ready(self, adapter: int, stream=None) -> None:
        N.check(N.lib().plora_engine_wait_ready(self._h, adapter, self._s(stream)))

    def release(self, adapter: int) -> None:
        N.check(N.lib().plora_engine_release(self._h, adapter))

    # batched forms (one C call per step instead of one per request)
    @staticmethod
    def _u32(keys):
        a = np.ascontiguousarray(keys, dtype=np.uint32)
        return a, a.ctypes.data_as(C.POINTER(C.c_uint32))

    def on_arrivals(self, adapters, now_ms: float, stream=None) -> int:
        a, p = self._u32(adapters)
        return N.check(int(N.lib().plora_engine_on_arrivals(self._h, p, len(a), now_ms,
                                                            self._s(stream))))

    def admit(self, adapters, now_ms: float, wait: bool = True, stream=None) -> np.ndarray:
        a, p = self._u32(adapters)
        st = np.zeros(max(len(a), 1), dtype=np.int32)
        N.check(N.lib().plora_engine_admit(self._h, p, len(a), now_ms, self._s(stream),
                                           int(wait), st.ctypes.data_as(C.POINTER(C.c_int32))))
        return st[:len(a)]

    def release_many(self, adapters) -> None:
        a, p = self._u32(adapters)
        N.check(N.lib().plora_engine_release_many(self._h, p, len(a)))

    def boundary(self, now_ms: float, stream=None) -> int:
        return N.check(N.lib().plora_engine_boundary(self._h, now_ms, self._s(stream)))

    def sync(self) -> None:
        N.check(N.lib().plora_engine_sync(self._h))

    def status(self, adapter: int) -> AdapterDynamics:
        c = N.plora_dynamics()
        N.check(N.lib().plora_engine_status(self._h, adapter, C.byref(c)))
        return AdapterDynamics(Residency(c.status), c.last_access_ms, c.decayed_count,
                               c.decay_stamp_ms, c.prediction, c.busy, bool(c.transfer_active))

    def residency(self, adapter: int) -> Residency:
        return Residency(self.status(adapter).status)

    def stats(self) -> dict:
        s = N.plora_engine_stats()
        N.lib().plora_engine_get_stats(self._h, C.byref(s))
        return {n: getattr(s, n) for n, _ in N.plora_engine_stats._fields_ if n != "reserved"}

    DECISION_ACTIONS = ("evict", "prefetch", "demand_load", "promote", "admission_failure",
                        "compact")

    def decisions(self, start: int = 0) -> list:
        """Decision-log rows (time_ms, action, adapter, score, detail) from
        `start` on — the reference's decisions.csv (src/report.cpp:106-113)."""
        n = int(N.lib().plora_engine_decisions(self._h, start, None, 0))
        if n <= start:
            return []
        buf = (N.plora_decision * (n - start))()
        N.lib().plora_engine_decisions(self._h, start, buf, n - start)
        return [(r.t_ms, self.DECISION_ACTIONS[r.action], None if r.adapter == 0xFFFFFFFF else r.adapter,
                 r.score, r.detail) for r in buf]

    def set_decision_log(self, enabled: bool) -> None:
        N.check(N.lib().plora_engine_set_decision_log(self._h, int(enabled)))

    def set_accuracy_interval(self, interval_ms: float, warmup_ms: float = 0.0) -> None:
        """Per-interval prediction accuracy bookkeeping (engine.cpp:598-633)."""
        N.check(N.lib().plora_engine_set_accuracy_interval(self._h, interval_ms, warmup_ms))

    def streams(self):
        d, p = C.c_void_p(), C.c_void_p()
        N.check(N.lib().plora_engine_streams(self._h, C.byref(d), C.byref(p)))
        return d.value, p.value
