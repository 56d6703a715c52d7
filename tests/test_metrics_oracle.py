"""The numpy restatement of the reference's evaluation metrics (oracle/fbmp_numpy.py, checker of
the device metrics) against the known answers of tests/test_metrics.cpp (CPU)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import fbmp_numpy as F  # noqa: E402


def scene(bands, h, w, seed):  # test_metrics.cpp: scaled_scene (uniform on [0, 255])
    return np.random.default_rng(seed).uniform(0.0, 255.0, (bands, h, w))


def test_crop_border():  # test_metrics.cpp: "crop_border basics"
    img = scene(2, 30, 30, 1)
    assert F.crop_border(img, 0).shape == (2, 30, 30)
    inner = F.crop_border(img, 10)
    assert inner.shape == (2, 10, 10) and inner[0, 0, 0] == img[0, 10, 10]
    with pytest.raises(ValueError):
        F.crop_border(img, 15)


def test_border_only_perturbation():  # "metrics see only the interior after border cropping"
    ref = scene(1, 30, 30, 2)
    est = ref.copy()
    est[0, 0, 0] += 50.0
    assert np.isfinite(F.psnr_avg(est, ref)[1])
    assert np.isinf(F.psnr_avg(F.crop_border(est, 10), F.crop_border(ref, 10))[1])


def test_psnr_kats():  # "psnr: identical, constant-offset, and the direct MSE oracle"
    ref = scene(2, 12, 12, 3)
    assert np.isinf(F.psnr_avg(ref, ref)[1])
    assert abs(F.psnr_avg(ref + 255.0, ref)[1]) < 1e-12
    est = scene(2, 12, 12, 4)
    per, avg = F.psnr_avg(est, ref)
    for b in range(2):
        mb = np.sum((est[b] - ref[b]) ** 2) / ref[b].size
        assert per[b] == pytest.approx(20.0 * np.log10(255.0 / np.sqrt(mb)), rel=1e-12)
    assert avg == pytest.approx(0.5 * (per[0] + per[1]), rel=1e-12)


def test_psnr_reg_kats():  # "regressed PSNR: affine invariance and fit optimality"
    ref = scene(2, 16, 16, 5)
    assert F.psnr_reg_avg(ref * 0.5 + 3.0, ref) > 200.0
    assert np.isinf(F.psnr_reg_avg(ref, ref))
    for t in range(100):
        est, noisy = scene(2, 8, 8, 700 + t), scene(2, 8, 8, 900 + t)
        assert F.psnr_reg_avg(est, noisy) >= F.psnr_avg(est, noisy)[1] - 1e-9
    target = scene(1, 8, 8, 6)
    const = np.full((1, 8, 8), 42.0)
    mse = np.mean((target[0] - target[0].mean()) ** 2)
    assert F.psnr_reg_avg(const, target) == pytest.approx(20.0 * np.log10(255.0 / np.sqrt(mse)), rel=1e-10)


def test_psnr_reg_grid_search():  # "regressed PSNR matches a grid-search oracle"
    ref, est = scene(1, 10, 10, 7), scene(1, 10, 10, 8)
    fast = F.psnr_reg_avg(est, ref)
    best = -1e300
    for a in np.arange(-2.0, 2.0 + 1e-12, 0.001):
        b = ref[0].mean() - a * est[0].mean()
        mse = np.mean((a * est[0] + b - ref[0]) ** 2)
        best = max(best, 20.0 * np.log10(255.0 / np.sqrt(mse)))
    assert fast >= best - 1e-9 and fast == pytest.approx(best, rel=0.01)


def test_ergas_sam_rase():  # "ergas, sam, rase: ideal values and oracles"
    ref = scene(3, 12, 12, 9)
    assert F.ergas(ref, ref, 4) == 0.0 and F.rase(ref, ref) == 0.0
    assert abs(F.sam_deg(ref, ref)) < 1e-6 and abs(F.sam_deg(3.0 * ref, ref)) < 1e-6
    est = scene(3, 12, 12, 10)
    mse = [np.mean((est[b] - ref[b]) ** 2) for b in range(3)]
    mu = [ref[b].mean() for b in range(3)]
    assert F.ergas(est, ref, 4) == pytest.approx(100.0 / 4 * np.sqrt(np.mean([m / u ** 2 for m, u in zip(mse, mu)])),
                                                 rel=1e-12)
    assert F.rase(est, ref) == pytest.approx(100.0 / np.mean(mu) * np.sqrt(np.mean(mse)), rel=1e-12)
    with pytest.raises(ValueError):
        F.ergas(est, np.zeros_like(ref), 4)
