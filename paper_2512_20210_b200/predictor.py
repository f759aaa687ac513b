"""Demand predictor for predictor-driven prefetch — lorasim's PredictorModel /
OnlinePredictor (include/lorasim/lstm.hpp:11-85, include/lorasim/predictor.hpp:12-111)
over libplora's C++ re-host (csrc/predictor.cpp, no Eigen).

Same names, argument meaning and exceptions as the reference; ``parameters``
is a live numpy view of θ like ``PredictorModel::parameters()``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .errors import ValidationError


@dataclass
class PredictorConfig:  # lstm.hpp:19-33
    window: int = 30
    hidden: int = 64
    layers: int = 2
    embedding_dim: int = 8
    num_adapters: int = 0
    learning_rate: float = 1e-3
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8

    def _c(self) -> N.plora_lstm_config:
        return N.plora_lstm_config(self.window, self.hidden, self.layers, self.embedding_dim,
                                   self.num_adapters, self.learning_rate, self.adam_beta1,
                                   self.adam_beta2, self.adam_eps)

    @classmethod
    def _from_c(cls, c) -> "PredictorConfig":
        return cls(*(getattr(c, n) for n, _ in N.plora_lstm_config._fields_))


@dataclass
class TrainingExample:  # lstm.hpp:13-17
    adapter: int = 0
    window: List[float] = field(default_factory=list)
    label: float = 0.0


@dataclass
class FeatureWindow:  # predictor.hpp:14-18
    adapter: int = 0
    counts: List[float] = field(default_factory=list)
    interval_s: float = 1.0


@dataclass
class Prediction:  # predictor.hpp:20-24
    adapter: int = 0
    probability: float = 0.5
    issued_at_ms: float = 0.0


def cross_entropy(probabilities: Sequence[float], labels: Sequence[float]) -> float:
    """Summed clamped binary cross-entropy (lstm.cpp:37-44)."""
    if len(probabilities) != len(labels):
        raise ValidationError("predictions and labels differ in length")
    p = np.ascontiguousarray(probabilities, dtype=np.float64)
    y = np.ascontiguousarray(labels, dtype=np.float64)
    out = C.c_double()
    N.check(N.lib().plora_cross_entropy(_dp(p), _dp(y), len(p), C.byref(out)))
    return out.value


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pack(model_cfg: PredictorConfig, batch: Sequence[TrainingExample]):
    n = len(batch)
    adapters = np.zeros(max(n, 1), dtype=np.uint32)
    labels = np.zeros(max(n, 1), dtype=np.float64)
    windows = np.zeros((max(n, 1), model_cfg.window), dtype=np.float64)
    for i, ex in enumerate(batch):
        if len(ex.window) != model_cfg.window:
            raise ValidationError(f"window length {len(ex.window)} does not match configured "
                                  f"window {model_cfg.window}")
        if not 0 <= ex.adapter < model_cfg.num_adapters:
            raise ValidationError("adapter index out of range")
        adapters[i] = ex.adapter
        windows[i] = ex.window
        labels[i] = ex.label
    return n, adapters, windows, labels


class PredictorModel:
    """Stacked LSTM over per-adapter count windows (lstm.hpp:39-85)."""

    def __init__(self, cfg: PredictorConfig, seed: int, _handle=None, _owner=None):
        self._owner = _owner
        if _handle is None:
            h = C.c_void_p()
            N.check(N.lib().plora_lstm_create(C.byref(cfg._c()), seed, C.byref(h)))
            _handle = h
        self._h = _handle
        self._cfg = cfg

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and self._owner is None:
            N.lib().plora_lstm_destroy(h)

    def config(self) -> PredictorConfig:
        return self._cfg

    def parameter_count(self) -> int:
        return int(N.lib().plora_lstm_param_count(self._h))

    def parameters(self) -> np.ndarray:
        """Live view of θ (writes change the model)."""
        n = self.parameter_count()
        ptr = N.lib().plora_lstm_parameters(self._h)
        return np.ctypeslib.as_array(ptr, shape=(n,))

    def _call(self, fn, batch, out):
        n, a, w, y = _pack(self._cfg, batch)
        if n == 0:
            raise ValidationError("empty batch")
        N.check(fn(self._h, a.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(w), _dp(y), n, out))

    def forward(self, batch: Sequence[TrainingExample]) -> np.ndarray:
        n, a, w, _ = _pack(self._cfg, batch)
        if n == 0:
            raise ValidationError("empty batch")
        p = np.empty(n, dtype=np.float64)
        N.check(N.lib().plora_lstm_forward(self._h, a.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           _dp(w), n, _dp(p)))
        return p

    def forward_arrays(self, adapters: np.ndarray, windows: np.ndarray) -> np.ndarray:
        """Batched forward on packed arrays (no per-example Python objects)."""
        a = np.ascontiguousarray(adapters, dtype=np.uint32)
        w = np.ascontiguousarray(windows, dtype=np.float64)
        p = np.empty(len(a), dtype=np.float64)
        N.check(N.lib().plora_lstm_forward(self._h, a.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           _dp(w), len(a), _dp(p)))
        return p

    def predict(self, adapter: int, window: Sequence[float]) -> float:
        return float(self.forward([TrainingExample(adapter, list(window))])[0])

    def loss_on(self, batch: Sequence[TrainingExample]) -> float:
        out = C.c_double()
        self._call(N.lib().plora_lstm_loss, batch, C.byref(out))
        return out.value

    def gradient(self, batch: Sequence[TrainingExample]) -> np.ndarray:
        g = np.empty(self.parameter_count(), dtype=np.float64)
        self._call(N.lib().plora_lstm_gradient, batch, _dp(g))
        return g

    def train_step(self, batch: Sequence[TrainingExample]) -> float:
        out = C.c_double()
        self._call(N.lib().plora_lstm_train_step, batch, C.byref(out))
        return out.value

    def save(self, path: str) -> None:
        N.check(N.lib().plora_lstm_save(self._h, str(path).encode()))

    @staticmethod
    def load(path: str) -> "PredictorModel":
        h = C.c_void_p()
        N.check(N.lib().plora_lstm_load(str(path).encode(), C.byref(h)))
        c = N.plora_lstm_config()
        N.lib().plora_lstm_get_config(h, C.byref(c))
        return PredictorModel(PredictorConfig._from_c(c), 0, _handle=h)


@dataclass
class OnlinePredictorConfig:  # predictor.hpp:45-51
    model: PredictorConfig = field(default_factory=PredictorConfig)
    interval_ms: float = 1000.0
    train_every: int = 100
    batch_size: int = 64
    replay_capacity: int = 10000

    def _c(self) -> N.plora_predictor_config:
        return N.plora_predictor_config(self.model._c(), self.interval_ms, self.train_every,
                                        self.batch_size, self.replay_capacity)


class ReplayBufferView:
    """Read-only view of the predictor's replay buffer (predictor.hpp:26-43)."""

    def __init__(self, pred: "OnlinePredictor"):
        self._p = pred

    def size(self) -> int:
        return self._p._stats().buffered

    def __len__(self) -> int:
        return self.size()

    def capacity(self) -> int:
        return self._p._cfg.replay_capacity

    def at(self, i: int) -> TrainingExample:
        w = np.empty(self._p._cfg.model.window, dtype=np.float64)
        a, y = C.c_uint32(), C.c_double()
        N.check(N.lib().plora_predictor_buffer_at(self._p._h, i, C.byref(a), _dp(w), C.byref(y)))
        return TrainingExample(a.value, w.tolist(), y.value)


class OnlinePredictor:
    """Per-adapter count series + replay-trained LSTM (predictor.hpp:54-111)."""

    def __init__(self, cfg: OnlinePredictorConfig, seed: int):
        h = C.c_void_p()
        N.check(N.lib().plora_predictor_create(C.byref(cfg._c()), seed, C.byref(h)))
        self._h = h
        self._cfg = cfg
        self._model = PredictorModel(cfg.model, 0, _handle=N.lib().plora_predictor_model(h),
                                     _owner=self)
        n = max(cfg.model.num_adapters, 1)
        self._ids = np.empty(n, dtype=np.uint32)
        self._probs = np.empty(n, dtype=np.float64)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            N.lib().plora_predictor_destroy(h)

    def _stats(self):
        s = N.plora_predictor_stats_t()
        N.lib().plora_predictor_stats(self._h, C.byref(s))
        return s

    def observe(self, adapter: int, t_ms: float) -> None:
        if adapter < 0:
            raise ValidationError("adapter index out of range in observe()")
        N.check(N.lib().plora_predictor_observe(self._h, adapter, t_ms))

    def roll_to(self, t_ms: float) -> None:
        N.check(N.lib().plora_predictor_roll_to(self._h, t_ms))

    def set_device(self, device: int) -> None:
        """predict_all's LSTM forward on CUDA `device` (FP64), or the host (-1)."""
        N.check(N.lib().plora_predictor_set_device(self._h, int(device)))

    def predict_arrays(self, now_ms: float):
        """(adapters uint32[k], probabilities f64[k]) for every known adapter."""
        n = N.lib().plora_predictor_predict_all(
            self._h, now_ms, self._ids.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(self._probs),
            len(self._ids))
        N.check(int(n) if n < 0 else 0)
        return self._ids[:n].copy(), self._probs[:n].copy()

    def predict_all(self, now_ms: float) -> List[Prediction]:
        ids, probs = self.predict_arrays(now_ms)
        return [Prediction(int(a), float(p), now_ms) for a, p in zip(ids, probs)]

    def train_step(self) -> Optional[float]:
        loss = C.c_double()
        rc = N.check(N.lib().plora_predictor_train_step(self._h, C.byref(loss)))
        return loss.value if rc == 1 else None

    def window_for(self, adapter: int) -> FeatureWindow:
        if adapter < 0:
            raise ValidationError("adapter index out of range in window_for()")
        w = np.empty(self._cfg.model.window, dtype=np.float64)
        N.check(N.lib().plora_predictor_window(self._h, adapter, _dp(w)))
        return FeatureWindow(adapter, w.tolist(), self._cfg.interval_ms / 1000.0)

    def known(self, adapter: int) -> bool:
        return bool(N.check(N.lib().plora_predictor_known(self._h, adapter)))

    def known_count(self) -> int:
        return int(self._stats().known)

    def observed(self) -> int:
        return int(self._stats().observed)

    def train_steps(self) -> int:
        return int(self._stats().train_steps)

    def last_loss(self) -> float:
        return float(self._stats().last_loss)

    def current_interval(self) -> int:
        return int(self._stats().current_interval)

    def model(self) -> PredictorModel:
        return self._model

    def buffer(self) -> ReplayBufferView:
        return ReplayBufferView(self)
