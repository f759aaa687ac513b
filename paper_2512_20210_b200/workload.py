"""Synthetic Azure-Functions-like workload (the host-side input of BASELINE
config 4) — generate_synthetic of src/workload.cpp:59-144, restated in the C++
library with the same libstdc++ engines so traces are bit-identical.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass
class SyntheticProfile:
    """include/lorasim/workload.hpp:19-50 (defaults identical)."""
    num_adapters: int = 20
    base_rate: float = 50.0
    diurnal_amplitude: float = 0.0
    period_s: float = 3600.0
    hot_set_size: int = 5
    hot_rotation_s: float = 7.0
    hot_share: float = 0.9
    rotation_jitter: float = 0.0
    burstiness_cv: float = 1.0
    input_median: float = 256.0
    input_sigma: float = 0.6
    output_median: float = 128.0
    output_sigma: float = 0.6
    max_tokens: int = 8192

    def to_c(self) -> N.plora_synthetic_profile:
        return N.plora_synthetic_profile(
            self.num_adapters, self.base_rate, self.diurnal_amplitude, self.period_s,
            self.hot_set_size, self.hot_rotation_s, self.hot_share, self.rotation_jitter,
            self.burstiness_cv, self.input_median, self.input_sigma, self.output_median,
            self.output_sigma, self.max_tokens)


@dataclass
class Trace:
    arrival_ms: np.ndarray     # float64, sorted
    adapter: np.ndarray        # uint32 catalog index
    input_tokens: np.ndarray   # uint32
    output_tokens: np.ndarray  # uint32

    def __len__(self) -> int:
        return len(self.arrival_ms)


def generate_synthetic(profile: SyntheticProfile, duration_s: float, seed: int) -> Trace:
    lib = N.lib()
    prof = profile.to_c()
    n = N.check(int(lib.plora_generate_synthetic(C.byref(prof), duration_s, seed, None, None,
                                                 None, None, 0)))
    arr = np.zeros(n, np.float64)
    ad = np.zeros(n, np.uint32)
    inp = np.zeros(n, np.uint32)
    out = np.zeros(n, np.uint32)
    P = C.POINTER
    lib.plora_generate_synthetic(
        C.byref(prof), duration_s, seed, arr.ctypes.data_as(P(C.c_double)),
        ad.ctypes.data_as(P(C.c_uint32)), inp.ctypes.data_as(P(C.c_uint32)),
        out.ctypes.data_as(P(C.c_uint32)), n)
    return Trace(arr, ad, inp, out)
