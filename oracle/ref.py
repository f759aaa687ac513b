"""ORACLE ONLY — ctypes over oracle/_ref/libref.so, the reference's own
PagePool / prefetch policy / adapter model / generate_synthetic compiled from
/root/reference/proj/src (see oracle/Makefile, oracle/ref_shim.cpp)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference "
                              "exists")
        L = C.CDLL(REF_SO)
        u32, u64, i32, i64, dbl, vp = (C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double,
                                       C.c_void_p)
        P = C.POINTER
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_lstm_forward_probability": (dbl, [u32, u32, u32, u32, u32, P(dbl), u32,
                                                   P(dbl)]),
            "ref_pool_create": (C.c_int, [u64, u32, P(vp)]),
            "ref_pool_destroy": (None, [vp]),
            "ref_pool_pages_needed": (u32, [vp, u64]),
            "ref_pool_alloc": (C.c_int, [vp, u32, u64]),
            "ref_pool_free": (C.c_int, [vp, u32]),
            "ref_pool_translate": (C.c_int, [vp, u32, u32, P(u32)]),
            "ref_pool_table": (C.c_int, [vp, u32, P(u32), u64, P(u64), P(u64)]),
            "ref_pool_has": (C.c_int, [vp, u32]),
            "ref_pool_compact": (u64, [vp]),
            "ref_pool_report": (None, [vp, P(dbl)]),
            "ref_pool_free_pages": (u32, [vp]),
            "ref_pool_total_pages": (u32, [vp]),
            "ref_pool_used_bytes": (u64, [vp]),
            "ref_pool_allocated_bytes": (u64, [vp]),
            "ref_pool_total_bytes": (u64, [vp]),
            "ref_pool_check_invariants": (C.c_int, [vp]),
            "ref_pool_resident": (u64, [vp, P(u32), u64]),
            "ref_pool_dump": (u64, [vp, C.c_char_p, u64]),
            "ref_policy_validate": (C.c_int, [vp]),
            "ref_recency_score": (dbl, [dbl, dbl, dbl]),
            "ref_decayed_at": (dbl, [vp, dbl, dbl]),
            "ref_record_access": (None, [vp, dbl, dbl]),
            "ref_eviction_score": (dbl, [vp, vp, dbl, dbl]),
            "ref_scored_residents": (u64, [vp, u64, vp, dbl, P(dbl), P(u32)]),
            "ref_select_prefetch": (u64, [P(dbl), u64, vp, u64, vp, P(u64), u64, u64, P(u32)]),
            "ref_plan_evictions": (C.c_int, [u64, u64, P(u32), u64, P(u64), u64, P(u32),
                                             P(u64)]),
            "ref_param_count": (C.c_int, [u32, u32, u32, u32, u32, P(u64)]),
            "ref_size_table_bytes": (C.c_int, [u32, u64, C.c_int, P(u32), P(u64), u64, u32,
                                               P(u64)]),
            "ref_generate_catalog": (C.c_int, [u32, P(u32), P(dbl), u64, u64, u32, u32, u32,
                                               u32, P(u32), P(u64)]),
            "ref_load_catalog_json": (i64, [C.c_char_p, P(u32), P(u64), u64]),
            "ref_generate_synthetic": (i64, [u32, dbl, dbl, dbl, u32, dbl, dbl, dbl, dbl, dbl,
                                             u64, P(dbl), P(u32), P(u32), P(u32), u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # -1 ValidationError, -2 logic_error, -3 ConfigError


def _check(rc: int) -> int:
    if rc < 0:
        raise RefError(rc, lib().ref_last_error().decode())
    return rc


class RefPagePool:
    """The reference lorasim::PagePool itself (src/memory.cpp)."""

    def __init__(self, page_bytes: int, total_pages: int):
        h = C.c_void_p()
        _check(lib().ref_pool_create(page_bytes, total_pages, C.byref(h)))
        self._h = h
        self._lib = lib()

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.ref_pool_destroy(self._h)
            self._h = None

    def pages_needed(self, n: int) -> int:
        return self._lib.ref_pool_pages_needed(self._h, n)

    def alloc(self, a: int, n: int) -> int:
        return _check(self._lib.ref_pool_alloc(self._h, a, n))

    def free(self, a: int) -> None:
        _check(self._lib.ref_pool_free(self._h, a))

    def translate(self, a: int, logical: int) -> int:
        out = C.c_uint32()
        _check(self._lib.ref_pool_translate(self._h, a, logical, C.byref(out)))
        return out.value

    def table(self, a: int) -> list[int]:
        n, wb = C.c_uint64(), C.c_uint64()
        _check(self._lib.ref_pool_table(self._h, a, None, 0, C.byref(n), C.byref(wb)))
        buf = (C.c_uint32 * max(n.value, 1))()
        _check(self._lib.ref_pool_table(self._h, a, buf, n.value, C.byref(n), C.byref(wb)))
        return list(buf[: n.value])

    def has(self, a: int) -> bool:
        return bool(self._lib.ref_pool_has(self._h, a))

    def compact(self) -> int:
        return self._lib.ref_pool_compact(self._h)

    def report(self) -> tuple[float, float, float]:
        out = (C.c_double * 3)()
        self._lib.ref_pool_report(self._h, out)
        return out[0], out[1], out[2]

    def free_pages(self) -> int:
        return self._lib.ref_pool_free_pages(self._h)

    def total_pages(self) -> int:
        return self._lib.ref_pool_total_pages(self._h)

    def used_bytes(self) -> int:
        return self._lib.ref_pool_used_bytes(self._h)

    def allocated_bytes(self) -> int:
        return self._lib.ref_pool_allocated_bytes(self._h)

    def total_bytes(self) -> int:
        return self._lib.ref_pool_total_bytes(self._h)

    def check_invariants(self) -> None:
        _check(self._lib.ref_pool_check_invariants(self._h))

    def resident(self) -> list[int]:
        n = self._lib.ref_pool_resident(self._h, None, 0)
        buf = (C.c_uint32 * max(n, 1))()
        self._lib.ref_pool_resident(self._h, buf, n)
        return list(buf[:n])

    def dump(self) -> str:
        n = self._lib.ref_pool_dump(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self._lib.ref_pool_dump(self._h, buf, n + 1)
        return buf.value.decode()


# ---- prefetch policy: plain-struct mirrors (layout == ref_shim.cpp DynC/PolicyC)
class DynC(C.Structure):
    _fields_ = [("status", C.c_int32), ("busy", C.c_uint32), ("last_access_ms", C.c_double),
                ("decayed_count", C.c_double), ("decay_stamp_ms", C.c_double),
                ("prediction", C.c_double), ("transfer_active", C.c_int32), ("pad", C.c_int32)]


class PolicyC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("theta", "alpha", "beta", "gamma", "tau_ms",
                                          "freq_half_life_ms", "staging_fraction")]


def dyn_c(d) -> DynC:
    return DynC(int(d.status), d.busy, d.last_access_ms, d.decayed_count, d.decay_stamp_ms,
                d.prediction, 1 if d.transfer_active else 0, 0)


def policy_c(p) -> PolicyC:
    return PolicyC(p.theta, p.alpha, p.beta, p.gamma, p.tau_ms, p.freq_half_life_ms,
                   p.staging_fraction)


def eviction_score(d, p, now, max_freq) -> float:
    dc, pc = dyn_c(d), policy_c(p)
    return lib().ref_eviction_score(C.byref(dc), C.byref(pc), now, max_freq)


def scored_residents(dyn, p, now):
    arr = (DynC * max(len(dyn), 1))(*[dyn_c(d) for d in dyn])
    scores = (C.c_double * max(len(dyn), 1))()
    keys = (C.c_uint32 * max(len(dyn), 1))()
    pc = policy_c(p)
    n = lib().ref_scored_residents(arr, len(dyn), C.byref(pc), now, scores, keys)
    return [(scores[i], keys[i]) for i in range(n)]


def select_prefetch(probs, dyn, p, units, budget):
    arr = (DynC * max(len(dyn), 1))(*[dyn_c(d) for d in dyn])
    pr = (C.c_double * max(len(probs), 1))(*probs)
    un = (C.c_uint64 * max(len(units), 1))(*units)
    out = (C.c_uint32 * max(len(dyn), 1))()
    pc = policy_c(p)
    n = lib().ref_select_prefetch(pr, len(probs), arr, len(dyn), C.byref(pc), un, len(units),
                                  budget, out)
    return list(out[:n])


def plan_evictions(need, free_bytes, eligible, bytes_for):
    el = (C.c_uint32 * max(len(eligible), 1))(*eligible)
    bf = (C.c_uint64 * max(len(bytes_for), 1))(*bytes_for)
    vic = (C.c_uint32 * max(len(eligible), 1))()
    nv = C.c_uint64()
    sat = lib().ref_plan_evictions(need, free_bytes, el, len(eligible), bf, len(bytes_for), vic,
                                   C.byref(nv))
    return list(vic[: nv.value]), bool(sat)


def policy_validate(p) -> int:
    pc = policy_c(p)
    return lib().ref_policy_validate(C.byref(pc))


def record_access(d, now, half_life):
    dc = dyn_c(d)
    lib().ref_record_access(C.byref(dc), now, half_life)
    return dc.last_access_ms, dc.decayed_count, dc.decay_stamp_ms


def decayed_at(d, now, half_life) -> float:
    dc = dyn_c(d)
    return lib().ref_decayed_at(C.byref(dc), now, half_life)


def recency_score(last, now, tau) -> float:
    return lib().ref_recency_score(last, now, tau)


# ---- adapter model / workload
def param_count(d, k, r, adapted, bpp):
    out = C.c_uint64()
    _check(lib().ref_param_count(d, k, r, adapted, bpp, C.byref(out)))
    return out.value


def size_table_bytes(rank, anchor_rank=8, anchor_bytes=13 << 20, linear=True, explicit=()):
    ranks = (C.c_uint32 * max(len(explicit), 1))(*[r for r, _ in explicit])
    byts = (C.c_uint64 * max(len(explicit), 1))(*[b for _, b in explicit])
    out = C.c_uint64()
    _check(lib().ref_size_table_bytes(anchor_rank, anchor_bytes, 1 if linear else 0, ranks, byts,
                                      len(explicit), rank, C.byref(out)))
    return out.value


def generate_catalog(count, mix, seed, d=4096, k=4096, adapted=64, bpp=2):
    mr = (C.c_uint32 * len(mix))(*[r for r, _ in mix])
    mw = (C.c_double * len(mix))(*[w for _, w in mix])
    ranks = (C.c_uint32 * count)()
    byts = (C.c_uint64 * count)()
    _check(lib().ref_generate_catalog(count, mr, mw, len(mix), seed, d, k, adapted, bpp, ranks,
                                      byts))
    return list(ranks), list(byts)


def load_catalog_json(path, cap=4096):
    """The reference's own load_catalog_json (base dims 4096/4096/64/bf16,
    default size table): (ranks, bytes), or raises RefError with the code
    (-1 ValidationError, -3 ConfigError, -5 ParseError)."""
    ranks = (C.c_uint32 * cap)()
    byts = (C.c_uint64 * cap)()
    n = lib().ref_load_catalog_json(path.encode(), ranks, byts, cap)
    if n < 0:
        raise RefError(int(n), lib().ref_last_error().decode())
    return list(ranks[:n]), list(byts[:n])


def generate_synthetic(profile, duration_s, seed):
    p = profile
    args = (p.num_adapters, p.base_rate, p.diurnal_amplitude, p.period_s, p.hot_set_size,
            p.hot_rotation_s, p.hot_share, p.rotation_jitter, p.burstiness_cv, duration_s, seed)
    n = lib().ref_generate_synthetic(*args, None, None, None, None, 0)
    if n < 0:
        raise RefError(-1, lib().ref_last_error().decode())
    arr = (C.c_double * max(n, 1))()
    ad = (C.c_uint32 * max(n, 1))()
    i = (C.c_uint32 * max(n, 1))()
    o = (C.c_uint32 * max(n, 1))()
    lib().ref_generate_synthetic(*args, arr, ad, i, o, n)
    return list(arr[:n]), list(ad[:n]), list(i[:n]), list(o[:n])


def lstm_forward_probability(cfg, theta, adapter, window) -> float:
    """tests/support/lstm_reference.hpp forward_probability (the reference's scalar oracle)."""
    import numpy as np
    th = np.ascontiguousarray(theta, dtype=np.float64)
    w = np.ascontiguousarray(window, dtype=np.float64)
    P = C.POINTER(C.c_double)
    return lib().ref_lstm_forward_probability(cfg.window, cfg.hidden, cfg.layers,
                                              cfg.embedding_dim, cfg.num_adapters,
                                              th.ctypes.data_as(P), adapter, w.ctypes.data_as(P))
