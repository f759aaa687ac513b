"""predict_all on the GPU (plora_predictor_set_device): FP64 LSTM forward over
every known adapter, checked against the host path (same summation order;
only exp / tanh rounding differs) and timed against the 5 ms budget at 1000
adapters (2.3 ms per 100 ms round)."""
import statistics
import time

import numpy as np
import pytest

from paper_2512_20210_b200.predictor import OnlinePredictor, OnlinePredictorConfig, PredictorConfig

pytestmark = pytest.mark.gpu


def _predictor(n=1000, layers=2):
    cfg = OnlinePredictorConfig(model=PredictorConfig(num_adapters=n, layers=layers),
                                train_every=10 ** 9)
    pred = OnlinePredictor(cfg, 7)
    rng = np.random.default_rng(3)
    t = 0.0
    for _ in range(20000):  # a skewed arrival history over ~40 intervals
        t += float(rng.exponential(2.0))
        pred.observe(int(min(n - 1, rng.zipf(1.3) - 1)), t)
    return pred, t


@pytest.mark.parametrize("layers", [1, 2])
def test_gpu_predict_all_matches_host(cuda, layers):
    pred, t = _predictor(n=1000, layers=layers)
    ids_h, p_h = (a.copy() for a in pred.predict_arrays(t + 1.0))
    pred.set_device(0)
    ids_g, p_g = (a.copy() for a in pred.predict_arrays(t + 1.0))
    assert np.array_equal(ids_h, ids_g)
    assert np.max(np.abs(p_h - p_g)) < 1e-12
    pred.set_device(-1)
    _, p_h2 = pred.predict_arrays(t + 1.0)
    assert np.array_equal(p_h2, p_h)


def test_gpu_predict_all_speed_1000_adapters(cuda):
    cfg = OnlinePredictorConfig(model=PredictorConfig(num_adapters=1000), train_every=10 ** 9)
    pred = OnlinePredictor(cfg, 1)
    for a in range(1000):
        pred.observe(a, float(a))
    pred.set_device(0)
    times = []
    for i in range(8):  # a new interval each call: no cached round
        t0 = time.perf_counter()
        ids, p = pred.predict_arrays(1500.0 + 1000.0 * i)
        times.append(time.perf_counter() - t0)
        assert len(ids) == 1000 and np.all((p > 0) & (p < 1))
    assert statistics.median(times[2:]) < 5e-3, times
