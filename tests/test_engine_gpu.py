"""Loading / prefetch engine on the GPU: the reference simulator's
behavioural pins (tests/test_engine.cpp) restated on real transfers, plus
content checks of every page the engine moved and BGMV parity after
eviction, reload and compaction.

Reference behaviours mirrored:
  * oracle prediction -> prefetch_issued == 1, promotions == 1, resident
    (warm) when the request arrives (test_engine.cpp:160-173);
  * a request for an adapter whose prefetch is in flight waits only for the
    rest of it: the transfer is upgraded, not restarted (:175-189,
    engine.cpp:449-455);
  * busy or in-flight adapters are never evicted (engine.cpp:297-298,
    :317-323); admission fails when nothing can be evicted (:427-431);
  * a prefetch evicts only victims scoring below gamma * p (:321);
  * idle compaction relocates pages and the data stays addressable
    (:486-497).
"""
import numpy as np
import pytest
import torch

from oracle import lora as OL
from paper_2512_20210_b200 import _native as N
from paper_2512_20210_b200.engine import Admit, EngineConfig, PrefetchEngine
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, ModelShape, bgmv
from paper_2512_20210_b200.memory import PagePool
from paper_2512_20210_b200.prefetch import PrefetchPolicy, Residency
from paper_2512_20210_b200 import synth

pytestmark = pytest.mark.gpu

SHAPE = ModelShape(2, (512, 512), (512, 256))


class Rig:
    def __init__(self, ranks, pool_pages, page_bytes=2048, copy_mode=N.PLORA_COPY_AUTO,
                 policy=None, compaction=True, prefetch=True, chunk_bytes=64 << 10,
                 inflight=256 << 10):
        self.ranks = list(ranks)
        self.page_bytes = page_bytes
        self.pool = PagePool(page_bytes, pool_pages)
        self.store = AdapterStore(self.pool, SHAPE, max_adapters=len(ranks))
        self.images = {}
        for a, r in enumerate(ranks):
            self.store.register(a, r)
            self.images[a] = synth.adapter_image(SHAPE, r, a).view(torch.uint8).pin_memory()
        self.eng = PrefetchEngine(self.store, EngineConfig(
            policy=policy or PrefetchPolicy(staging_fraction=0.5), copy_mode=copy_mode, prefetch=prefetch,
            compaction=compaction, chunk_bytes=chunk_bytes, prefetch_inflight_bytes=inflight))
        for a in range(len(ranks)):
            self.eng.set_source(a, self.images[a])

    def check_content(self, a):
        n = self.images[a].numel()
        got = self.store.read_pages(a, n)
        assert torch.equal(got.cpu(), self.images[a]), f"adapter {a} pages differ"

    def settle(self, now):
        self.eng.sync()
        torch.cuda.synchronize()
        self.eng.boundary(now)
        torch.cuda.synchronize()


def pages_for(rank):
    return -(-SHAPE.adapter_bytes(rank) // 2048)


@pytest.mark.parametrize("mode", [N.PLORA_COPY_CE, N.PLORA_COPY_SM])
def test_demand_load_on_arrival(mode):
    rig = Rig([8, 16], pool_pages=4 * pages_for(16), copy_mode=mode)
    assert rig.eng.on_arrival(1, 0.0) is False  # cold: demand load starts at arrival
    assert rig.eng.residency(1) == Residency.staging
    assert rig.eng.acquire(1, 0.0) == Admit.loading
    rig.settle(1.0)
    assert rig.eng.residency(1) == Residency.resident
    assert rig.store.is_published(1)
    rig.check_content(1)
    st = rig.eng.stats()
    assert st["demand_loads"] == 1 and st["prefetch_issued"] == 0
    assert st["bytes_h2d"] == SHAPE.adapter_bytes(16)
    assert st["copy_mode"] == mode
    rig.eng.release(1)
    assert rig.eng.on_arrival(1, 2.0) is True  # warm now


def test_wait_ready_is_device_side():
    rig = Rig([32], pool_pages=2 * pages_for(32))
    assert rig.eng.acquire(0, 0.0) == Admit.loading
    rig.eng.wait_ready(0)  # no host sync: compute stream waits on the copy
    assert rig.eng.residency(0) == Residency.resident
    torch.cuda.synchronize()
    rig.check_content(0)


def test_oracle_prefetch_is_promoted_at_boundary():  # test_engine.cpp:160-173
    rig = Rig([8, 16, 8], pool_pages=8 * pages_for(16))
    rig.eng.set_predictions([0.01, 0.99, 0.01])
    rig.eng.boundary(0.0)
    st = rig.eng.stats()
    assert st["prefetch_issued"] == 1
    assert rig.eng.residency(1) == Residency.staging
    rig.settle(5.0)  # transfer done -> staged -> promoted at this boundary
    st = rig.eng.stats()
    assert st["promotions"] == 1 and st["demand_loads"] == 0
    assert rig.eng.residency(1) == Residency.resident
    assert rig.eng.on_arrival(1, 6.0) is True  # warm at arrival
    assert rig.eng.acquire(1, 6.0) == Admit.ready
    rig.check_content(1)


def test_in_flight_prefetch_is_upgraded_not_restarted():  # test_engine.cpp:175-189
    # tiny chunks and in-flight cap so the prefetch is still being issued
    rig = Rig([64], pool_pages=2 * pages_for(64), chunk_bytes=2048, inflight=4096)
    rig.eng.set_predictions([0.99])
    rig.eng.boundary(0.0)
    assert rig.eng.residency(0) == Residency.staging
    assert rig.eng.acquire(0, 0.1) in (Admit.loading, Admit.ready)
    rig.settle(1.0)
    st = rig.eng.stats()
    assert st["prefetch_issued"] == 1 and st["demand_loads"] == 0
    assert st["transfers_completed"] == 1
    assert st["upgrades"] + st["promotions"] >= 1
    assert rig.eng.residency(0) == Residency.resident
    rig.check_content(0)


def test_eviction_skips_busy_and_admission_fails_when_all_busy():
    # room for exactly two rank-16 adapters
    rig = Rig([16, 16, 16], pool_pages=2 * pages_for(16), compaction=False)
    for a, t in ((0, 0.0), (1, 1.0)):
        rig.eng.on_arrival(a, t)
        assert rig.eng.acquire(a, t) == Admit.loading
    rig.settle(2.0)
    # both busy: the third cannot be admitted
    rig.eng.on_arrival(2, 3.0)
    assert rig.eng.acquire(2, 3.0) == Admit.failed
    assert rig.eng.stats()["admission_failures"] == 1
    assert rig.eng.residency(0) == Residency.resident and rig.eng.residency(1) == Residency.resident
    # release the older one: it becomes the victim (lowest recency/frequency score)
    rig.eng.release(0)
    assert rig.eng.acquire(2, 4.0) == Admit.loading
    rig.settle(5.0)
    assert rig.eng.residency(0) == Residency.not_resident
    assert rig.eng.residency(2) == Residency.resident
    assert not rig.store.is_published(0)
    assert rig.eng.stats()["evictions"] == 1
    rig.check_content(1)
    rig.check_content(2)


def test_prefetch_evicts_only_below_gamma_p():
    pol = PrefetchPolicy(gamma=0.4, staging_fraction=1.0)
    rig = Rig([16, 16], pool_pages=pages_for(16), policy=pol, compaction=False)
    rig.eng.on_arrival(0, 0.0)
    rig.eng.acquire(0, 0.0)
    rig.settle(1.0)
    rig.eng.release(0)
    # adapter 0 was just used: its score is ~alpha + beta = 0.6 >= gamma * 0.9
    rig.eng.set_predictions([0.0, 0.9])
    rig.eng.boundary(2.0)
    st = rig.eng.stats()
    assert st["prefetch_issued"] == 0 and st["evictions"] == 0
    assert rig.eng.residency(0) == Residency.resident


def test_bgmv_after_eviction_reload_and_compaction():
    ranks = [8, 16, 32, 16, 8, 64]
    cap = pages_for(64) + pages_for(32) + pages_for(16)
    rig = Rig(ranks, pool_pages=cap, compaction=True)
    now = 0.0
    order = [5, 1, 2, 0, 3, 4, 5, 2, 1]
    for a in order:
        now += 10.0
        rig.eng.on_arrival(a, now)
        if rig.eng.acquire(a, now) == Admit.failed:
            pytest.fail(f"admission failed for {a}")
        rig.eng.wait_ready(a)
        rig.eng.release(a)
        rig.eng.boundary(now)
    rig.settle(now + 1)  # idle: compaction may relocate pages
    torch.cuda.synchronize()
    rig.pool.check_invariants()
    resident = [a for a in range(len(ranks)) if rig.eng.residency(a) == Residency.resident]
    assert resident and rig.eng.stats()["evictions"] > 0
    for a in resident:
        rig.check_content(a)
    # a decode batch over the resident adapters matches the oracle
    ta = [resident[i % len(resident)] for i in range(3 * len(resident))]
    T = len(ta)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(T, 512, generator=g).to(torch.bfloat16).cuda()
    y = torch.randn(T, 256, generator=g).to(torch.bfloat16).cuda()
    y0 = y.clone()
    plan = BatchPlan(rig.store, ta)
    bgmv(plan, 1, 1, x, y, scale=0.5)
    torch.cuda.synchronize()
    m = OL.model(SHAPE.n_layers, SHAPE.d_in, SHAPE.d_out, SHAPE.esize)
    arena = np.zeros(rig.pool.total_pages() * 2048, np.uint8)
    tables = {}
    for a in resident:
        tables[a] = rig.pool.table(a)
        OL.scatter_pages(arena, 2048, tables[a], rig.images[a].numpy())
    from lora_harness import rel_err, to_np_bits, TOL_BF16
    yb = to_np_bits(y0)
    OL.paged_lora_apply(m, arena, 2048, tables, {a: ranks[a] for a in resident}, 1, 1,
                        to_np_bits(x), yb, ta, scale=0.5)
    assert rel_err(y, yb) < TOL_BF16


@pytest.mark.parametrize("asynchronous", [False, True])
def test_predictor_driven_rounds(asynchronous):
    from paper_2512_20210_b200.predictor import (OnlinePredictor, OnlinePredictorConfig,
                                                 PredictorConfig)
    ranks = [8] * 6
    rig = Rig(ranks, pool_pages=6 * pages_for(8))
    pred = OnlinePredictor(OnlinePredictorConfig(
        model=PredictorConfig(window=5, hidden=8, embedding_dim=2, num_adapters=6),
        interval_ms=100.0, train_every=20, batch_size=16), 7)
    rig.eng.attach_predictor(pred, asynchronous=asynchronous)
    now = 0.0
    for i in range(200):
        now += 7.0
        a = i % 3  # adapters 0..2 hot
        rig.eng.on_arrival(a, now)
        assert rig.eng.acquire(a, now) != Admit.failed
        rig.eng.wait_ready(a)
        rig.eng.release(a)
        if i % 10 == 0:
            rig.eng.round(now)
        rig.eng.boundary(now)
    rig.eng.flush_predictor()
    rig.settle(now + 1)
    st = rig.eng.stats()
    assert st["prediction_rounds"] == 20
    assert pred.observed() == 200 and pred.train_steps() == 10
    for a in range(3):
        assert rig.eng.residency(a) == Residency.resident
        rig.check_content(a)


def test_engine_errors():
    rig = Rig([8], pool_pages=pages_for(8))
    with pytest.raises(N.ValidationError if hasattr(N, "ValidationError") else Exception):
        rig.eng.acquire(5, 0.0)
    with pytest.raises(Exception):
        rig.eng.release(0)  # release without acquire -> logic error
    with pytest.raises(Exception):
        rig.eng.set_source(0, torch.zeros(10, dtype=torch.uint8))  # wrong size


def test_decision_log_and_interval_accuracy():
    """Every decision is logged with its time (engine.cpp:304-495 -> decisions.csv),
    and each closed interval is scored tp / (tp + fp + fn) over the known
    adapters, the predicted set snapshotted when the interval's first
    prediction arrives (engine.cpp:547-561, 598-633)."""
    rig = Rig([4, 4, 4], pool_pages=400)
    eng = rig.eng
    eng.set_accuracy_interval(100.0)
    for a in range(3):
        eng.on_arrival(a, 10.0)
    rig.settle(20.0)
    eng.on_arrival(0, 120.0)  # interval 1: adapters 0, 1 arrive
    eng.set_predictions([0.01, 0.99, 0.01])  # predicted {1}
    eng.on_arrival(1, 150.0)
    eng.boundary(210.0)  # closes interval 1
    st = eng.stats()
    assert st["acc_intervals"] == 1
    assert (st["acc_tp"], st["acc_fp"], st["acc_fn"]) == (1, 0, 1)
    assert abs(st["acc_sum"] - 0.5) < 1e-12
    rows = eng.decisions()
    loads = [r for r in rows if r[1] == "demand_load"]
    assert [r[2] for r in loads[:3]] == [0, 1, 2] and all(r[0] == 10.0 for r in loads[:3])
    assert loads[0][4] == SHAPE.adapter_bytes(4)
    eng.set_decision_log(False)
    assert eng.decisions() == []
