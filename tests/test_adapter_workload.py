"""Adapter model (tests/test_adapter.cpp re-expressed) and the synthetic
workload generator — both bit-exact against the compiled reference."""
import pytest

from paper_2512_20210_b200 import (AdapterSizeTable, AdapterSpec, ConfigError, LoraDims,
                                   SyntheticProfile, ValidationError, adapter_size_bytes,
                                   generate_catalog, generate_synthetic, param_count)

MiB = 1 << 20


def test_param_count_hand_arithmetic():  # test_adapter.cpp:15-21
    assert param_count(4096, 4096, 8, 64, 2) == 4194304
    assert param_count(2, 2, 1, 1, 2) == 4


def test_param_count_rejects_invalid():  # :23-32
    for args in ((4096, 4096, 0, 64, 2), (16, 16, 16, 1, 2), (64, 64, 4, 1, 3)):
        with pytest.raises(ValidationError):
            param_count(*args)


def test_param_count_linear_in_rank():  # :34-40
    for r in (1, 2, 4, 8, 16):
        assert param_count(4096, 4096, 2 * r, 64, 2) == 2 * param_count(4096, 4096, r, 64, 2)


def test_size_table():  # :42-62
    t = AdapterSizeTable()
    assert (t.bytes_for(8), t.bytes_for(64), t.bytes_for(16)) == (13 * MiB, 104 * MiB, 26 * MiB)
    t = AdapterSizeTable(8, 13 * MiB, False)
    t.set(8, 14 * MiB)
    assert t.bytes_for(8) == 14 * MiB
    with pytest.raises(ConfigError):
        t.bytes_for(32)
    prev = 0
    for r in (1, 4, 8, 16, 32, 64, 128):
        assert adapter_size_bytes(r) >= prev
        prev = adapter_size_bytes(r)


def test_derived_and_sized_specs():  # :64-74
    dims = LoraDims(4096, 4096, 8, 64, 2)
    assert AdapterSpec.derived("x", dims).weight_bytes == 4194304 * 2
    s = AdapterSpec.sized("y", dims, 13 * MiB)
    assert s.weight_bytes == 13 * MiB and s.nominal_size_override is not None


def test_catalog_deterministic_and_matches_reference(ref):  # :97-106
    mix = [(8, 0.5), (64, 0.5)]
    a = generate_catalog(50, mix, 7)
    b = generate_catalog(50, mix, 7)
    assert [x.dims.r for x in a] == [x.dims.r for x in b]
    assert a[0].id == "a00" and a[49].id == "a49"
    r_ranks, r_bytes = ref.generate_catalog(50, mix, 7)
    assert [x.dims.r for x in a] == r_ranks
    assert [x.weight_bytes for x in a] == r_bytes
    mix = [(8, 1.0), (16, 2.0), (32, 1.0), (64, 0.5)]
    c = generate_catalog(1000, mix, 20240611)
    assert [x.dims.r for x in c] == ref.generate_catalog(1000, mix, 20240611)[0]


def test_size_table_matches_reference(ref):
    for r in (1, 3, 8, 16, 33, 64, 128):
        assert AdapterSizeTable().bytes_for(r) == ref.size_table_bytes(r)
        assert param_count(4096, 4096, r, 64, 2) == ref.param_count(4096, 4096, r, 64, 2)


@pytest.mark.parametrize("prof,dur,seed", [
    (SyntheticProfile(), 30.0, 1),
    (SyntheticProfile(num_adapters=1000, base_rate=200.0, hot_set_size=50, hot_rotation_s=5.0,
                      diurnal_amplitude=0.5, period_s=60.0, rotation_jitter=0.3,
                      burstiness_cv=2.0), 20.0, 20240611),
    (SyntheticProfile(num_adapters=7, hot_set_size=7, hot_share=0.5, burstiness_cv=0.5),
     10.0, 3),
])
def test_generate_synthetic_bit_exact(ref, prof, dur, seed):
    tr = generate_synthetic(prof, dur, seed)
    arr, ad, i, o = ref.generate_synthetic(prof, dur, seed)
    assert len(tr) == len(arr) > 0
    assert list(tr.arrival_ms) == arr
    assert list(tr.adapter) == ad
    assert list(tr.input_tokens) == i
    assert list(tr.output_tokens) == o


def test_generate_synthetic_validation():
    with pytest.raises(ValidationError):
        generate_synthetic(SyntheticProfile(hot_set_size=0), 1.0, 1)
    with pytest.raises(ValidationError):
        generate_synthetic(SyntheticProfile(), -1.0, 1)


CATALOGS = {
    "golden": '[{"id": "alpha", "rank": 8}, {"id": "beta", "rank": 64, "size_bytes": 999}]',
    "mixed": "[" + ", ".join(
        f'{{"id": "a{i:03d}", "rank": {(8, 16, 32, 64, 128)[i % 5]}'
        + (f', "size_bytes": {1 + 4096 * i}' if i % 3 == 0 else "") + "}" for i in range(40)) + "]",
    "not_array": '{"id": "alpha", "rank": 8}',
    "missing_rank": '[{"id": "alpha"}]',
    "empty": "[]",
    "malformed": '[{"id": "alpha", "rank": 8',
    "zero_rank": '[{"id": "alpha", "rank": 0}]',
}


@pytest.mark.parametrize("name", sorted(CATALOGS))
def test_load_catalog_json_matches_reference(ref, tmp_path, name):
    """load_catalog_json (src/adapter.cpp:81-108) against the compiled
    reference: the same specs, or the same error class."""
    from paper_2512_20210_b200 import ConfigError, ParseError, ValidationError
    from paper_2512_20210_b200.adapter import load_catalog_json
    path = tmp_path / f"{name}.json"
    path.write_text(CATALOGS[name])
    codes = {ValidationError: -1, ConfigError: -3, ParseError: -5}
    try:
        want = ref.load_catalog_json(str(path))
    except ref.RefError as e:
        with pytest.raises(tuple(k for k, v in codes.items() if v == e.code)):
            load_catalog_json(str(path))
        return
    got = load_catalog_json(str(path))
    assert [s.dims.r for s in got] == want[0]
    assert [s.weight_bytes for s in got] == want[1]
    if name == "golden":  # tests/test_adapter.cpp:76-95
        assert [s.id for s in got] == ["alpha", "beta"]
        assert got[0].weight_bytes == 13 * (1 << 20)


def test_load_catalog_json_missing_file_is_config_error(ref, tmp_path):
    from paper_2512_20210_b200 import ConfigError
    from paper_2512_20210_b200.adapter import load_catalog_json
    with pytest.raises(ConfigError):
        load_catalog_json(str(tmp_path / "does_not_exist.json"))
    with pytest.raises(ref.RefError):
        ref.load_catalog_json(str(tmp_path / "does_not_exist.json"))
