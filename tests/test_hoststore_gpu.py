"""Host adapter store (plora_hoststore_*): page-aligned pinned images with an
offset index, saved to and mapped back from a PLHS file, feeding the engine's
transfers (each adapter's own bytes land in its pages)."""
import os

import pytest
import torch

from paper_2512_20210_b200 import synth
from paper_2512_20210_b200._native import ValidationError
from paper_2512_20210_b200.engine import EngineConfig, PrefetchEngine
from paper_2512_20210_b200.hoststore import HostAdapterStore
from paper_2512_20210_b200.lora import AdapterStore, ModelShape
from paper_2512_20210_b200.memory import PagePool

pytestmark = pytest.mark.gpu
SHAPE = ModelShape(2, (512, 512), (512, 256))


def test_store_layout_file_roundtrip_and_engine_loads(cuda, tmp_path):
    ranks = [3, 8, 16, 5]
    sizes = [SHAPE.adapter_bytes(r) for r in ranks]
    hs = HostAdapterStore.create(sizes, ranks, align=4096)
    assert len(hs) == 4
    imgs = [synth.adapter_image(SHAPE, r, 40 + a).view(torch.uint8) for a, r in enumerate(ranks)]
    prev_end = 0
    for a, img in enumerate(imgs):
        ptr, nbytes, rank = hs.entry(a)
        assert nbytes == sizes[a] and rank == ranks[a] and ptr % 4096 == 0 and ptr >= prev_end
        prev_end = ptr + nbytes
        hs.view(a).copy_(img)
    path = os.path.join(tmp_path, "catalog.plhs")
    hs.save(path)
    mapped = HostAdapterStore.open(path)
    for a, img in enumerate(imgs):
        assert torch.equal(mapped.view(a), img)
    with pytest.raises(ValidationError):
        mapped.entry(4)
    # the engine pages every adapter in from the mapped (pinned) file
    pool = PagePool(2048, 4000)
    store = AdapterStore(pool, SHAPE, max_adapters=4)
    for a, r in enumerate(ranks):
        store.register(a, r)
    eng = PrefetchEngine(store, EngineConfig(prefetch=False))
    for a in range(4):
        eng.set_source(a, mapped.view(a))
    for a in range(4):
        eng.on_arrival(a, 1.0 + a)
    eng.sync()
    eng.boundary(10.0)
    torch.cuda.synchronize()
    for a, img in enumerate(imgs):
        assert torch.equal(store.read_pages(a, img.numel()).cpu(), img)
    del eng, store


def test_store_rejects_bad_arguments(cuda, tmp_path):
    with pytest.raises(ValidationError):
        HostAdapterStore.create([10, 0], align=4096)
    with pytest.raises(ValidationError):
        HostAdapterStore.create([10], align=3000)
    bad = os.path.join(tmp_path, "bad.plhs")
    with open(bad, "wb") as f:
        f.write(b"NOPE" + bytes(100))
    from paper_2512_20210_b200._native import ParseError
    with pytest.raises(ParseError):
        HostAdapterStore.open(bad)
