"""Host adapter store (libplora ``plora_hoststore_*``): the pinned host copy
of every adapter of a catalog, page-aligned with an offset index, optionally
saved to / mapped from a "PLHS" file.  Engines page adapters in from it
(``PrefetchEngine.set_source_ptr``), so every transfer moves that adapter's
own bytes (sizes from the reference's LoraDims,
src/adapter.cpp:12-26)."""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np
import torch

from . import _native as N


class HostAdapterStore:
    def __init__(self, _h):
        self._h = _h

    @classmethod
    def create(cls, sizes: Sequence[int], ranks: Sequence[int] = (), align: int = 2 << 20):
        b = np.ascontiguousarray(sizes, dtype=np.uint64)
        r = np.ascontiguousarray(ranks if len(ranks) else np.zeros(len(b)), dtype=np.uint32)
        h = C.c_void_p()
        N.check(N.lib().plora_hoststore_create(b.ctypes.data_as(C.POINTER(C.c_uint64)),
                                               r.ctypes.data_as(C.POINTER(C.c_uint32)), len(b),
                                               align, C.byref(h)))
        return cls(h)

    @classmethod
    def open(cls, path: str):
        h = C.c_void_p()
        N.check(N.lib().plora_hoststore_open(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        N.check(N.lib().plora_hoststore_save(self._h, path.encode()))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            N.lib().plora_hoststore_destroy(h)

    def __len__(self) -> int:
        return int(N.lib().plora_hoststore_count(self._h))

    @property
    def handle(self):
        return self._h

    def entry(self, key: int):
        """(host pointer, bytes, rank) of adapter `key`."""
        p, b, r = C.c_void_p(), C.c_uint64(), C.c_uint32()
        N.check(N.lib().plora_hoststore_entry(self._h, key, C.byref(p), C.byref(b), C.byref(r)))
        return p.value, b.value, r.value

    def view(self, key: int) -> torch.Tensor:
        """A uint8 CPU tensor over adapter `key`'s pinned bytes (no copy; the
        store must outlive it)."""
        ptr, nbytes, _ = self.entry(key)
        buf = (C.c_uint8 * nbytes).from_address(ptr)
        return torch.frombuffer(buf, dtype=torch.uint8, count=nbytes)

    def total_bytes(self) -> int:
        v = C.c_uint64()
        N.check(N.lib().plora_hoststore_bytes(self._h, C.byref(v)))
        return v.value
