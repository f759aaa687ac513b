"""PagePool drop-in parity: the reference's own unit tests
(/root/reference/proj/tests/test_memory.cpp) re-expressed against the product,
plus bit-exact placement against the compiled reference PagePool on churn."""
import json
import os
import random

import pytest

from paper_2512_20210_b200 import (AllocStatus, LogicError, PagePool, ValidationError)

MiB = 1 << 20
kPage = 2 * MiB
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_13mib_takes_7_pages():  # test_memory.cpp:17-24
    pool = PagePool(kPage, 16)
    assert pool.pages_needed(13 * MiB) == 7
    assert pool.alloc(1, 13 * MiB) == AllocStatus.ok
    assert len(pool.table(1)) == 7
    assert pool.free_pages() == 9
    pool.check_invariants()


def test_exact_fit_wastes_nothing():  # :26-31
    pool = PagePool(kPage, 4)
    assert pool.alloc(1, kPage) == AllocStatus.ok
    assert len(pool.table(1)) == 1
    assert pool.report().internal_frag == 0.0


def test_failed_alloc_leaves_pool_unchanged():  # :33-39
    pool = PagePool(kPage, 6)
    assert pool.alloc(1, 13 * MiB) == AllocStatus.out_of_memory
    assert pool.free_pages() == 6
    assert not pool.has(1)
    pool.check_invariants()


def test_free_restores_and_double_free_is_logic_error():  # :41-48
    pool = PagePool(kPage, 16)
    assert pool.alloc(3, 5 * MiB) == AllocStatus.ok
    pool.free(3)
    assert pool.free_pages() == 16
    assert pool.used_bytes() == 0
    with pytest.raises(LogicError, match="free of adapter 3 which holds no pages"):
        pool.free(3)


def test_fresh_pool_identity_translation():  # :50-55
    pool = PagePool(kPage, 8)
    assert pool.alloc(0, 3 * kPage) == AllocStatus.ok
    for i in range(3):
        assert pool.translate(0, i) == i
    with pytest.raises(ValidationError, match=r"logical page 3 out of range \(adapter has 3 pages\)"):
        pool.translate(0, 3)


def test_compaction_fixed_point_and_prefix():  # :57-74
    pool = PagePool(kPage, 8)
    for a in range(3):
        assert pool.alloc(a, 2 * kPage) == AllocStatus.ok
    assert pool.compact() == 0
    pool.free(1)
    assert pool.compact() == 2
    for i in range(2):
        assert pool.translate(0, i) < 4
        assert pool.translate(2, i) < 4
    pool.check_invariants()
    assert pool.compact() == 0


def test_empty_report_all_zero():  # :98-107
    r = PagePool(kPage, 8).report()
    assert r.external_frag == 0.0 and r.utilization == 0.0


def test_dump_parseable():  # :109-118
    pool = PagePool(kPage, 4)
    assert pool.alloc(9, 3 * MiB) == AllocStatus.ok
    j = json.loads(pool.dump())
    assert j["total_pages"] == 4
    assert "9" in j["tables"]


def test_error_contract():
    with pytest.raises(ValidationError, match="page size must be positive"):
        PagePool(0, 4)
    pool = PagePool(2048, 4)
    with pytest.raises(ValidationError, match="cannot allocate zero bytes"):
        pool.alloc(0, 0)
    pool.alloc(0, 10)
    with pytest.raises(LogicError, match="adapter 0 already allocated"):
        pool.alloc(0, 10)
    with pytest.raises(ValidationError, match="no page table for adapter 5"):
        pool.translate(5, 0)
    # ValidationError/ConfigError are ValueErrors, as bindings/module.cpp:48-50 registers them
    assert issubclass(ValidationError, ValueError)


def test_appendix_a_golden_vectors():
    """SURVEY Appendix A, captured from the reference memory.o."""
    with open(os.path.join(GOLDEN, "pagepool_appendix_a.json")) as f:
        g = json.load(f)
    pool = PagePool(2048, 16)
    pool.alloc(0, 3 * 2048)
    pool.alloc(1, 2 * 2048)
    pool.alloc(2, 4 * 2048)
    pool.free(1)
    pool.alloc(3, 5 * 2048 + 1)
    assert pool.table(0) == g["hole_reuse"]["a0"]
    assert pool.table(2) == g["hole_reuse"]["a2"]
    assert pool.table(3) == g["hole_reuse"]["a3"]
    pool.free(0)
    assert pool.compact() == g["compaction"]["moved"]
    assert pool.table(2) == g["compaction"]["a2"]
    assert pool.table(3) == g["compaction"]["a3"]
    r = pool.report()
    assert r.internal_frag == g["compaction"]["internal_frag"]
    assert r.utilization == g["compaction"]["utilization"]
    assert pool.free_pages() == g["compaction"]["free"]
    assert pool.dump() == g["compaction"]["dump"]
    relocs = [(x.adapter, x.logical, x.src, x.dst) for x in pool.last_relocations()]
    assert relocs == [tuple(r) for r in g["compaction"]["relocations"]]


def test_churn_golden_fixture():
    """10^5-op churn (test_memory.cpp:120-154 seeding) — final tables pinned by
    the reference (tests/golden/pagepool_churn.json, oracle/make_golden.py)."""
    with open(os.path.join(GOLDEN, "pagepool_churn.json")) as f:
        g = json.load(f)
    pool = PagePool(g["page_bytes"], g["total_pages"])
    for op in g["ops"]:
        if op[0] == "a":
            assert int(pool.alloc(op[1], op[2])) == op[3]
        elif op[0] == "f":
            pool.free(op[1])
        else:
            assert pool.compact() == op[1]
    assert pool.dump() == g["final_dump"]


def _churn_ops(seed, n_ops, n_ids, max_bytes, compact_every):
    rng = random.Random(seed)
    live = set()
    for op in range(n_ops):
        a = rng.randrange(n_ids)
        if op % compact_every == compact_every - 1:
            yield ("c",)
        if a in live:
            live.discard(a)
            yield ("f", a)
        else:
            b = rng.randrange(1, max_bytes + 1)
            yield ("a", a, b)
            live.add(a)


@pytest.mark.parametrize("page_bytes,total,max_bytes,seed", [
    (2 * MiB, 256, 24 * MiB, 20240611),   # test_memory.cpp:120-154 scale
    (2048, 4096, 300_000, 7),
    (4096, 1000, 2_000_000, 99),          # non-multiple-of-64 page count
])
def test_bit_exact_vs_reference_churn(ref, page_bytes, total, max_bytes, seed):
    ours = PagePool(page_bytes, total)
    theirs = ref.RefPagePool(page_bytes, total)
    live = set()
    for i, op in enumerate(_churn_ops(seed, 20000, 64, max_bytes, 997)):
        if op[0] == "a":
            st_o = int(ours.alloc(op[1], op[2]))
            st_t = theirs.alloc(op[1], op[2])
            assert st_o == st_t
            if st_o == 0:
                live.add(op[1])
                assert ours.table(op[1]) == theirs.table(op[1])
        elif op[0] == "f":
            if op[1] in live:
                ours.free(op[1])
                theirs.free(op[1])
                live.discard(op[1])
        else:
            assert ours.compact() == theirs.compact()
            for a in live:
                assert ours.table(a) == theirs.table(a)
        assert ours.free_pages() == theirs.free_pages()
        if i % 2000 == 0:
            ours.check_invariants()
            assert ours.dump() == theirs.dump()
    ours.check_invariants()
    assert ours.dump() == theirs.dump()
    assert ours.report() == type(ours.report())(*theirs.report())


def test_error_codes_match_reference(ref):
    ours, theirs = PagePool(2048, 4), ref.RefPagePool(2048, 4)
    for fn in (lambda p: p.alloc(0, 0), lambda p: p.translate(1, 0)):
        with pytest.raises(ValidationError) as e1:
            fn(ours)
        with pytest.raises(ref.RefError) as e2:
            fn(theirs)
        assert str(e1.value) == str(e2.value) and e2.value.code == -1
    with pytest.raises(LogicError) as e1:
        ours.free(2)
    with pytest.raises(ref.RefError) as e2:
        theirs.free(2)
    assert str(e1.value) == str(e2.value) and e2.value.code == -2


def test_paged_sufficiency_and_no_fragmentation_failure():
    """any request <= free_pages·P succeeds; paged alloc never
    reports fragmentation_failure (test_memory.cpp:156-193 claim)."""
    rng = random.Random(7)
    pool = PagePool(kPage, 128)
    live = {}
    for _ in range(20000):
        a = rng.randrange(32)
        if a in live:
            pool.free(a)
            del live[a]
            continue
        b = (13 + rng.randrange(8) * 13) * MiB
        free_before = pool.free_pages()
        st = pool.alloc(a, b)
        assert st != AllocStatus.fragmentation_failure
        assert (st == AllocStatus.ok) == (pool.pages_needed(b) <= free_before)
        if st == AllocStatus.ok:
            live[a] = b
    pool.check_invariants()


def test_large_pool_is_fast():
    """The bitmap pool handles 2^20 pages (the 2 GiB arena at 2 KiB pages) and
    rank-64 adapters (32768 pages) in milliseconds (reference: 308 ms ctor,
    5.8 ms per rank-64 free — BASELINE.md §2)."""
    import time
    t0 = time.perf_counter()
    pool = PagePool(2048, 1 << 20)
    for a in range(16):
        assert pool.alloc(a, 64 * MiB) == AllocStatus.ok
    for a in range(0, 16, 2):
        pool.free(a)
    for a in range(16, 24):
        assert pool.alloc(a, 64 * MiB) == AllocStatus.ok
    dt = time.perf_counter() - t0
    pool.check_invariants()
    assert dt < 2.0
