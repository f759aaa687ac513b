"""Prefetch / eviction policy — mirrors include/lorasim/prefetch.hpp:11-72
(the host half of the predictor-driven prefetch hook) over the C ABI.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

from . import _native as N


class Residency(enum.IntEnum):
    """prefetch.hpp:23."""
    not_resident = 0
    staging = 1
    resident = 2


@dataclass
class PrefetchPolicy:
    """prefetch.hpp:11-21 (defaults identical)."""
    theta: float = 0.5
    alpha: float = 0.3
    beta: float = 0.3
    gamma: float = 0.4
    tau_ms: float = 60_000.0
    freq_half_life_ms: float = 120_000.0
    staging_fraction: float = 0.1

    def to_c(self) -> N.plora_policy:
        return N.plora_policy(self.theta, self.alpha, self.beta, self.gamma, self.tau_ms,
                              self.freq_half_life_ms, self.staging_fraction)

    def validate(self) -> None:
        c = self.to_c()
        N.check(N.lib().plora_policy_validate(C.byref(c)))


@dataclass
class AdapterDynamics:
    """prefetch.hpp:26-37."""
    status: Residency = Residency.not_resident
    last_access_ms: float = -1.0
    decayed_count: float = 0.0
    decay_stamp_ms: float = 0.0
    prediction: float = 0.0
    busy: int = 0
    transfer_active: bool = False

    def to_c(self) -> N.plora_dynamics:
        return N.plora_dynamics(int(self.status), self.busy, self.last_access_ms,
                                self.decayed_count, self.decay_stamp_ms, self.prediction,
                                1 if self.transfer_active else 0, 0)

    def _pull(self, c: N.plora_dynamics) -> None:
        self.last_access_ms = c.last_access_ms
        self.decayed_count = c.decayed_count
        self.decay_stamp_ms = c.decay_stamp_ms

    def record_access(self, now_ms: float, half_life_ms: float) -> None:
        c = self.to_c()
        N.lib().plora_record_access(C.byref(c), now_ms, half_life_ms)
        self._pull(c)

    def decayed_at(self, now_ms: float, half_life_ms: float) -> float:
        c = self.to_c()
        return N.lib().plora_decayed_at(C.byref(c), now_ms, half_life_ms)


def _dyn_array(dyn: list[AdapterDynamics]):
    arr = (N.plora_dynamics * max(len(dyn), 1))()
    for i, d in enumerate(dyn):
        arr[i] = d.to_c()
    return arr


def recency_score(last_access_ms: float, now_ms: float, tau_ms: float) -> float:
    return N.lib().plora_recency_score(last_access_ms, now_ms, tau_ms)


def eviction_score(dyn: AdapterDynamics, policy: PrefetchPolicy, now_ms: float,
                   max_freq: float) -> float:
    c, p = dyn.to_c(), policy.to_c()
    return N.lib().plora_eviction_score(C.byref(c), C.byref(p), now_ms, max_freq)


def scored_residents(dyn: list[AdapterDynamics], policy: PrefetchPolicy,
                     now_ms: float) -> list[tuple[float, int]]:
    n = len(dyn)
    scores = (C.c_double * max(n, 1))()
    keys = (C.c_uint32 * max(n, 1))()
    p = policy.to_c()
    k = N.lib().plora_scored_residents(_dyn_array(dyn), n, C.byref(p), now_ms, scores, keys)
    return [(scores[i], keys[i]) for i in range(k)]


def select_prefetch(probabilities: list[float], dyn: list[AdapterDynamics],
                    policy: PrefetchPolicy, units_for: list[int],
                    staging_budget_units: int) -> list[int]:
    n = len(dyn)
    out = (C.c_uint32 * max(n, 1))()
    p = policy.to_c()
    k = N.lib().plora_select_prefetch(N.f64_array(probabilities), len(probabilities),
                                      _dyn_array(dyn), n, C.byref(p), N.u64_array(units_for),
                                      len(units_for), staging_budget_units, out)
    return list(out[:k])


@dataclass
class EvictionPlan:
    victims: list[int]
    satisfied: bool


def plan_evictions(bytes_needed: int, free_bytes: int, eligible: list[int],
                   bytes_for: list[int]) -> EvictionPlan:
    victims = (C.c_uint32 * max(len(eligible), 1))()
    nv = C.c_uint64()
    sat = N.lib().plora_plan_evictions(bytes_needed, free_bytes, N.u32_array(eligible),
                                       len(eligible), N.u64_array(bytes_for), len(bytes_for),
                                       victims, C.byref(nv))
    return EvictionPlan(list(victims[: nv.value]), bool(sat))
