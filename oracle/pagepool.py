"""ORACLE ONLY — pure-Python restatement of lorasim::PagePool
(/root/reference/proj/src/memory.cpp:7-146).  A min-heap plays the role of
the ordered std::set free list (``free_.begin()`` == ``heap[0]``).  Pinned
against the compiled reference (oracle.ref) in tests/test_oracle.py."""
from __future__ import annotations

import heapq


class OraclePagePool:
    def __init__(self, page_bytes: int, total_pages: int):  # memory.cpp:7-12
        if page_bytes == 0:
            raise ValueError("page size must be positive")
        self.page_bytes = page_bytes
        self.total_pages = total_pages
        self.free = list(range(total_pages))  # already a valid heap
        self.owner = [-1] * total_pages
        self.tables: dict[int, tuple[int, list[int]]] = {}
        self.used_bytes = 0

    def pages_needed(self, nbytes: int) -> int:  # memory.cpp:14-16
        return ((nbytes + self.page_bytes - 1) % (1 << 64)) // self.page_bytes % (1 << 32)

    def alloc(self, adapter: int, nbytes: int) -> int:  # memory.cpp:18-38
        if nbytes == 0:
            raise ValueError("cannot allocate zero bytes")
        if adapter in self.tables:
            raise RuntimeError(f"adapter {adapter} already allocated")
        need = self.pages_needed(nbytes)
        if len(self.free) < need:
            return 1  # out_of_memory
        entries = [heapq.heappop(self.free) for _ in range(need)]
        for p in entries:
            self.owner[p] = adapter
        self.used_bytes += nbytes
        self.tables[adapter] = (nbytes, entries)
        return 0

    def release(self, adapter: int) -> None:  # memory.cpp:40-53
        if adapter not in self.tables:
            raise RuntimeError(f"free of adapter {adapter} which holds no pages")
        nbytes, entries = self.tables.pop(adapter)
        for p in entries:
            self.owner[p] = -1
            heapq.heappush(self.free, p)
        self.used_bytes -= nbytes

    def table(self, adapter: int) -> list[int]:
        return list(self.tables[adapter][1])

    def compact(self) -> int:  # memory.cpp:71-89
        live = self.total_pages - len(self.free)
        moved = 0
        for adapter in sorted(self.tables):
            entries = self.tables[adapter][1]
            for i, phys in enumerate(entries):
                if phys < live:
                    continue
                target = heapq.heappop(self.free)
                heapq.heappush(self.free, phys)
                self.owner[target] = self.owner[phys]
                self.owner[phys] = -1
                entries[i] = target
                moved += 1
        return moved
