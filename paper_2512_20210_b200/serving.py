"""Decode serving loop over the paged LoRA op and the prefetch engine — the
real-time host control loop of SURVEY §8(f) rank 1.

Per step (one decode token for each of up to ``batch_tokens`` requests):

  1. arrivals      ``engine.on_arrival`` per request (access statistics,
                   predictor observation, reactive demand load;
                   src/engine.cpp:515-545);
  2. prediction    every ``round_ms`` of trace time ``engine.round``
                   (predict_all -> probabilities, :547-561);
  3. admission     ``engine.acquire`` per distinct adapter; loading ones are
                   made ready by a device-side wait on their transfer
                   (``wait_ready``), failed ones are deferred to the next
                   step (:416-457);
  4. apply         plan update + the paged BGMV of every layer (one
                   plora_bgmv_layer launch per layer for both projections) on
                   the compute stream;
  5. boundary      release + ``engine.boundary`` (completions, promotions,
                   prefetch issue on the side streams, idle compaction;
                   :406-414).

Request sharding across GPUs: adapter key k belongs to rank
k mod world; each rank runs its own server over its own pool — no
collective on the data path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from .engine import Admit, EngineConfig, PrefetchEngine
from .lora import AdapterStore, BatchPlan, ModelShape, bgmv, bgmv_layer
from .memory import PagePool
from .predictor import OnlinePredictor, OnlinePredictorConfig


def owner_of(adapter: int, world: int) -> int:
    """Rank that serves an adapter key (request sharding, no collective)."""
    return adapter % world


def shard_keys(n_adapters: int, rank: int, world: int) -> List[int]:
    return [a for a in range(n_adapters) if owner_of(a, world) == rank]


@dataclass
class ServerConfig:
    shape: ModelShape
    ranks: Sequence[int]                 # per local adapter key
    pool_bytes: int
    page_bytes: int = 2 << 20
    batch_tokens: int = 256
    round_ms: float = 100.0              # cost_model round_ms (defaults.ini:92)
    engine: EngineConfig = field(default_factory=EngineConfig)
    predictor: Optional[OnlinePredictorConfig] = None
    seed: int = 42
    device: int = 0
    # prediction source for the prefetch hook: "lstm" (the attached online
    # predictor), "oracle" (the future arrivals, engine.cpp:555-562) or "off"
    prediction: str = "lstm"
    oracle_horizon_ms: float = 2000.0   # policy.oracle_horizon_ms (defaults.ini:57)


class DecodeServer:
    def __init__(self, cfg: ServerConfig, host_image: Callable[[int], torch.Tensor],
                 future: Optional[Sequence[np.ndarray]] = None):
        """future: per local adapter key, the sorted arrival times of the trace
        (the oracle prediction source)."""
        self.cfg = cfg
        n = len(cfg.ranks)
        self.pool = PagePool(cfg.page_bytes, cfg.pool_bytes // cfg.page_bytes)
        self.store = AdapterStore(self.pool, cfg.shape, n, device=cfg.device)
        for a, r in enumerate(cfg.ranks):
            self.store.register(a, r)
        self.engine = PrefetchEngine(self.store, cfg.engine)
        for a in range(n):
            self.engine.set_source(a, host_image(a))
        self.predictor = None
        self.future = future
        if cfg.prediction == "lstm" and cfg.predictor is not None:
            self.predictor = OnlinePredictor(cfg.predictor, cfg.seed)
            self.engine.attach_predictor(self.predictor)
        if cfg.predictor is not None:
            self.engine.set_accuracy_interval(cfg.predictor.interval_ms)
        if cfg.prediction == "oracle" and future is None:
            raise ValueError("the oracle prediction source needs the future arrivals")
        dev = torch.device("cuda", cfg.device)
        T = cfg.batch_tokens
        self.x = [torch.randn(T, d, device=dev).to(torch.bfloat16) for d in cfg.shape.d_in]
        self.y = [torch.randn(T, d, device=dev).to(torch.bfloat16) for d in cfg.shape.d_out]
        self.plan: Optional[BatchPlan] = None
        self.next_round_ms = 0.0
        self.deferred: List[int] = []
        self.stats = {"tokens": 0, "deferred": 0, "waited": 0, "steps": 0}
        self.fused = cfg.shape.n_proj > 1 and len(set(cfg.shape.d_in)) == 1 and \
            len(set(cfg.shape.d_out)) == 1
        self.last_batch = 0

    def step(self, arrivals: Sequence[int], now_ms: float, events=None) -> int:
        """Serve one decode token for each request in `arrivals` (adapter keys,
        plus any deferred from the previous step).  Returns tokens served."""
        eng = self.engine
        arrivals = np.asarray(arrivals, dtype=np.uint32)
        if events is not None:
            events[0].record()  # the step starts: demand stalls count from here
        eng.on_arrivals(arrivals, now_ms)
        if now_ms >= self.next_round_ms and self.cfg.prediction != "off":
            if self.predictor is not None:
                eng.round(now_ms)
            elif self.cfg.prediction == "oracle":
                eng.set_predictions(self._oracle(now_ms))
            self.next_round_ms = now_ms + self.cfg.round_ms
        want = np.concatenate([np.asarray(self.deferred, dtype=np.uint32), arrivals])
        take, later = want[:self.cfg.batch_tokens], list(want[self.cfg.batch_tokens:])
        uniq = np.unique(take)
        # admission of the distinct adapters; loading ones become ready through
        # a device-side wait of the compute stream on their copies
        st = eng.admit(uniq, now_ms, wait=True)
        self.stats["waited"] += int((st == Admit.loading).sum())
        ok = uniq[st != Admit.failed]
        keep = np.isin(take, ok)
        batch = [int(a) for a in take[keep]]
        later = [int(a) for a in take[~keep]] + [int(a) for a in later]
        self.deferred = later
        self.stats["deferred"] += len(later)
        if batch:
            if self.plan is None:
                self.plan = BatchPlan(self.store, batch)
            else:
                self.plan.update(batch)
            T = len(batch)
            self.last_batch = T
            if events is not None:
                events[1].record()  # demand copies waited for: the kernels start
            self.apply(T)
            if events is not None:
                events[2].record()
        elif events is not None:
            events[1].record()
            events[2].record()
        eng.release_many(ok)
        eng.boundary(now_ms)
        self.stats["tokens"] += len(batch)
        self.stats["steps"] += 1
        return len(batch)

    def apply(self, T: int) -> None:
        """The paged LoRA of every layer for the plan's T tokens."""
        for l in range(self.cfg.shape.n_layers):
            if self.fused:
                bgmv_layer(self.plan, l, self.x[0][:T], [y[:T] for y in self.y])
            else:
                for p in range(self.cfg.shape.n_proj):
                    bgmv(self.plan, l, p, self.x[p][:T], self.y[p][:T])

    def _oracle(self, now_ms: float) -> np.ndarray:
        """The reference's oracle predictions (engine.cpp:555-562): 0.99 for
        adapters with an arrival in (now, now + horizon], else 0.01."""
        p = np.full(len(self.future), 0.01)
        h = now_ms + self.cfg.oracle_horizon_ms
        for a, times in enumerate(self.future):
            i = np.searchsorted(times, now_ms, side="right")
            if i < len(times) and times[i] <= h:
                p[a] = 0.99
        return p

