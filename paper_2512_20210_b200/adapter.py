"""Adapter model / registry — mirrors include/lorasim/adapter.hpp:15-76 and
the ``LoraDims`` / ``param_count`` / ``adapter_size_bytes`` bindings
(bindings/module.cpp:53-73) over the C ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import json

from . import _native as N
from .errors import ConfigError, ParseError, ValidationError

MiB = 1 << 20


@dataclass(frozen=True)
class LoraDims:
    """adapter.hpp:15-23; validated on construction like the binding does."""
    d: int = 4096
    k: int = 4096
    r: int = 8
    adapted_matrices: int = 64
    bytes_per_param: int = 2

    def __post_init__(self):
        self.validate()

    def validate(self) -> None:
        N.check(N.lib().plora_lora_dims_validate(self.d, self.k, self.r, self.adapted_matrices,
                                                 self.bytes_per_param))


def param_count(d: int = 4096, k: int = 4096, r: int = 8, adapted_matrices: int = 64,
                bytes_per_param: int = 2) -> int:
    """adapted · r · (d + k) (src/adapter.cpp:22-26)."""
    out = C.c_uint64()
    N.check(N.lib().plora_param_count(d, k, r, adapted_matrices, bytes_per_param,
                                      C.byref(out)))
    return out.value


class AdapterSizeTable:
    """Rank -> resident bytes (adapter.hpp:32-47): explicit entries win,
    else linear in rank from the anchor (default rank 8 at 13 MiB)."""

    def __init__(self, anchor_rank: int = 8, anchor_bytes: int = 13 * MiB,
                 linear_fallback: bool = True):
        h = C.c_void_p()
        N.check(N.lib().plora_size_table_create(anchor_rank, anchor_bytes,
                                                1 if linear_fallback else 0, C.byref(h)))
        self._h = h
        self._lib = N.lib()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.plora_size_table_destroy(h)
            self._h = None

    def set(self, rank: int, nbytes: int) -> None:
        N.check(self._lib.plora_size_table_set(self._h, rank, nbytes))

    def bytes_for(self, rank: int) -> int:
        out = C.c_uint64()
        N.check(self._lib.plora_size_table_bytes_for(self._h, rank, C.byref(out)))
        return out.value


def adapter_size_bytes(rank: int) -> int:
    """bindings/module.cpp:71-73 — the default size table."""
    return AdapterSizeTable().bytes_for(rank)


@dataclass(frozen=True)
class AdapterSpec:
    """One serveable adapter (adapter.hpp:49-61)."""
    id: str
    dims: LoraDims
    weight_bytes: int
    nominal_size_override: int | None = None

    @staticmethod
    def derived(id: str, dims: LoraDims) -> "AdapterSpec":
        return AdapterSpec(id, dims, param_count(dims.d, dims.k, dims.r, dims.adapted_matrices,
                                                 dims.bytes_per_param) * dims.bytes_per_param)

    @staticmethod
    def sized(id: str, dims: LoraDims, nbytes: int) -> "AdapterSpec":
        if nbytes <= 0:
            raise ValidationError("adapter weight_bytes must be > 0")
        return AdapterSpec(id, dims, nbytes, nbytes)


def catalog_id(index: int, count: int) -> str:
    """Zero-padded ids "a000".. as generate_catalog names them (adapter.cpp:121-138)."""
    width = max(1, len(str(max(count - 1, 0))))
    return "a" + str(index).zfill(width)


def generate_catalog(count: int, mix: list[tuple[int, float]], seed: int,
                     sizes: AdapterSizeTable | None = None,
                     base: LoraDims | None = None) -> list[AdapterSpec]:
    """generate_catalog (src/adapter.cpp:110-144), bit-identical rank draws."""
    base = base if base is not None else LoraDims()
    ranks = (C.c_uint32 * max(count, 1))()
    nbytes = (C.c_uint64 * max(count, 1))()
    N.check(N.lib().plora_generate_catalog(
        count, N.u32_array([r for r, _ in mix]), N.f64_array([w for _, w in mix]), len(mix),
        seed, sizes._h if sizes is not None else None, base.d, base.k, base.adapted_matrices,
        base.bytes_per_param, ranks, nbytes))
    out = []
    for i in range(count):
        dims = LoraDims(base.d, base.k, ranks[i], base.adapted_matrices, base.bytes_per_param)
        out.append(AdapterSpec(catalog_id(i, count), dims, nbytes[i], nbytes[i]))
    return out


def load_catalog_json(path: str, sizes: AdapterSizeTable | None = None,
                      base: LoraDims | None = None) -> list[AdapterSpec]:
    """load_catalog_json (src/adapter.cpp:81-108) through the C ABI
    (plora_load_catalog_json): a JSON array of ``{"id": str, "rank": int[,
    "size_bytes": int]}``; sizes default to the size table's bytes for the
    rank.  Errors as the reference raises them: ConfigError (cannot open),
    ParseError (malformed / not an array / entry without id or rank),
    ValidationError (empty catalog, invalid dims)."""
    base = base if base is not None else LoraDims()
    sz = sizes if sizes is not None else AdapterSizeTable()
    L = N.lib()
    args = (path.encode(), sz._h, base.d, base.k, base.adapted_matrices, base.bytes_per_param)
    n = L.plora_load_catalog_json(*args, None, None, None, 0, 0)
    N.check(n)
    ranks = (C.c_uint32 * n)()
    nbytes = (C.c_uint64 * n)()
    stride = 256
    ids = C.create_string_buffer(n * stride)
    N.check(L.plora_load_catalog_json(*args, ranks, nbytes, ids, stride, n))
    out = []
    for i in range(n):
        ident = C.string_at(C.addressof(ids) + i * stride).decode("utf-8", "replace")
        dims = LoraDims(base.d, base.k, ranks[i], base.adapted_matrices, base.bytes_per_param)
        out.append(AdapterSpec.sized(ident, dims, nbytes[i]))
    return out
