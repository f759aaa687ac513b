"""Python face of the page pool — mirrors ``lorasim._core.PagePool``
(bindings/module.cpp:86-97) over the C ABI (include/plora.h), and adds what
the reference's binding omits (``table``, ``has``, byte accessors, the
compaction relocation list).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

from . import _native as N


class AllocStatus(enum.IntEnum):
    """include/lorasim/memory.hpp:18-22."""
    ok = 0
    out_of_memory = 1
    fragmentation_failure = 2


@dataclass(frozen=True)
class FragmentationReport:
    """include/lorasim/memory.hpp:24-28."""
    external_frag: float
    internal_frag: float
    utilization: float


@dataclass(frozen=True)
class Relocation:
    adapter: int
    logical: int
    src: int
    dst: int


class PagePool:
    """Fixed-size page inventory with per-adapter page tables.

    Placement is bit-identical to lorasim::PagePool (src/memory.cpp:7-146):
    lowest-free-first allocation, atomic OOM, compaction in adapter-key then
    logical order.
    """

    def __init__(self, page_bytes: int, total_pages: int):
        lib = N.lib()
        h = C.c_void_p()
        N.check(lib.plora_pool_create(int(page_bytes), int(total_pages), C.byref(h)))
        self._h = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.plora_pool_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def pages_needed(self, nbytes: int) -> int:
        return self._lib.plora_pool_pages_needed(self._h, int(nbytes))

    def alloc(self, adapter: int, weight_bytes: int) -> AllocStatus:
        return AllocStatus(N.check(self._lib.plora_pool_alloc(self._h, int(adapter),
                                                              int(weight_bytes))))

    def free(self, adapter: int) -> None:
        N.check(self._lib.plora_pool_free(self._h, int(adapter)))

    def translate(self, adapter: int, logical: int) -> int:
        out = C.c_uint32()
        N.check(self._lib.plora_pool_translate(self._h, int(adapter), int(logical),
                                               C.byref(out)))
        return out.value

    def table(self, adapter: int) -> list[int]:
        """Logical -> physical entries (PagePool::table, src/memory.cpp:64-69)."""
        ptr = C.POINTER(C.c_uint32)()
        n = C.c_uint32()
        wb = C.c_uint64()
        N.check(self._lib.plora_pool_table(self._h, int(adapter), C.byref(ptr), C.byref(n),
                                           C.byref(wb)))
        return ptr[: n.value] if n.value else []

    def weight_bytes(self, adapter: int) -> int:
        wb = C.c_uint64()
        N.check(self._lib.plora_pool_table(self._h, int(adapter), None, None, C.byref(wb)))
        return wb.value

    def has(self, adapter: int) -> bool:
        return bool(self._lib.plora_pool_has(self._h, int(adapter)))

    def compact(self) -> int:
        moved = C.c_uint64()
        N.check(self._lib.plora_pool_compact(self._h, C.byref(moved)))
        return moved.value

    def last_relocations(self) -> list[Relocation]:
        ptr = C.POINTER(N.plora_reloc)()
        n = C.c_uint64()
        self._lib.plora_pool_last_relocations(self._h, C.byref(ptr), C.byref(n))
        return [Relocation(ptr[i].adapter, ptr[i].logical, ptr[i].src, ptr[i].dst)
                for i in range(n.value)]

    def report(self) -> FragmentationReport:
        r = N.plora_frag_report()
        self._lib.plora_pool_report(self._h, C.byref(r))
        return FragmentationReport(r.external_frag, r.internal_frag, r.utilization)

    def free_pages(self) -> int:
        return self._lib.plora_pool_free_pages(self._h)

    def total_pages(self) -> int:
        return self._lib.plora_pool_total_pages(self._h)

    def page_bytes(self) -> int:
        return self._lib.plora_pool_page_bytes(self._h)

    def used_bytes(self) -> int:
        return self._lib.plora_pool_used_bytes(self._h)

    def allocated_bytes(self) -> int:
        return self._lib.plora_pool_allocated_bytes(self._h)

    def total_bytes(self) -> int:
        return self._lib.plora_pool_total_bytes(self._h)

    def resident(self) -> list[int]:
        n = self._lib.plora_pool_resident(self._h, None, 0)
        buf = (C.c_uint32 * max(n, 1))()
        self._lib.plora_pool_resident(self._h, buf, n)
        return list(buf[:n])

    def check_invariants(self) -> None:
        N.check(self._lib.plora_pool_check_invariants(self._h))

    def dump(self) -> str:
        """PagePool::dump().dump() — byte-identical JSON text."""
        n = C.c_uint64()
        N.check(self._lib.plora_pool_dump(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        N.check(self._lib.plora_pool_dump(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()
