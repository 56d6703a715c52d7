"""Device evaluation metrics (csrc/metrics.cu; metrics.hpp:11-51) against the numpy restatement of
metrics.cpp, plus the reference's error behaviour."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import fbmp_numpy as F  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,H,W,crop", [(4, 64, 80, 0), (4, 64, 80, 10), (8, 257, 130, 3), (1, 30, 30, 14)])
def test_metrics_match_oracle(gpu, N, H, W, crop):
    rng = np.random.default_rng(N * H + W + crop)
    ref = rng.uniform(0.0, 255.0, (N, H, W))
    est = ref * rng.uniform(0.8, 1.2) + rng.normal(0.0, 6.0, ref.shape)
    est[:, 5, 7] = 0.0  # a zero spectral vector: no angle (metrics.cpp:132)
    ref[:, 5, 7] = 0.0
    m = gpu.metrics(est, ref, factor=4, crop=crop)
    e, r = F.crop_border(est, crop), F.crop_border(ref, crop)
    per, avg = F.psnr_avg(e, r)
    assert np.allclose(m["psnr_per_band"], per, rtol=1e-12, atol=0)
    assert m["psnr_avg"] == pytest.approx(avg, rel=1e-12)
    assert m["psnr_reg_avg"] == pytest.approx(F.psnr_reg_avg(e, r), rel=1e-11)
    assert m["ergas"] == pytest.approx(F.ergas(e, r, 4), rel=1e-11)
    assert m["sam_deg"] == pytest.approx(F.sam_deg(e, r), rel=1e-10)
    assert m["rase"] == pytest.approx(F.rase(e, r), rel=1e-11)


def test_metrics_ideal_values(gpu):  # test_metrics.cpp: identical / offset / scaled cubes
    ref = np.random.default_rng(3).uniform(0.0, 255.0, (3, 12, 12))
    m = gpu.metrics(ref, ref)
    assert np.isinf(m["psnr_avg"]) and np.isinf(m["psnr_reg_avg"])
    assert m["ergas"] == 0.0 and m["rase"] == 0.0 and abs(m["sam_deg"]) < 1e-6
    assert abs(gpu.psnr_avg(ref + 255.0, ref)[1]) < 1e-12
    assert gpu.psnr_reg_avg(ref * 0.5 + 3.0, ref) > 200.0
    assert abs(gpu.sam_deg(3.0 * ref, ref)) < 1e-6


def test_metrics_errors(gpu):
    ref = np.random.default_rng(4).uniform(0.0, 255.0, (2, 20, 20))
    with pytest.raises(gpu.ParamError):
        gpu.metrics(ref, ref, crop=-1)
    with pytest.raises(gpu.DimensionError):
        gpu.metrics(ref, ref, crop=10)
    with pytest.raises(gpu.DimensionError):
        gpu.metrics(ref, ref[:, :, :19])
    with pytest.raises(gpu.NumericalError):
        gpu.ergas(ref, np.zeros_like(ref), 4)
    with pytest.raises(gpu.NumericalError):
        gpu.rase(ref, np.zeros_like(ref))
    assert gpu.sam_deg(ref, np.zeros_like(ref)) == 0.0  # every vector is zero: no angle, 0
