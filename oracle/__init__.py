"""ORACLE / TEST INFRASTRUCTURE ONLY.

Checkers for the product (``paper_2512_20210_b200``), used by tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs — never by the product path.

  oracle.ref       ctypes over oracle/_ref/libref.so: the UNMODIFIED reference
                   sources (/root/reference/proj/src/{memory,prefetch,adapter,
                   workload}.cpp) compiled where they lie (oracle/Makefile).
  oracle.lora      ctypes over oracle/liboracle.so: the C restatement of the
                   paged LoRA apply (PAPER.md:64-69 through PagePool tables).
  oracle.pagepool  pure-Python restatement of PagePool (src/memory.cpp:7-146),
                   pinned against oracle.ref in tests.
"""
