"""Pins the CPU oracle (oracle/fbmp_oracle.cpp) to the reference's own known answers and
oracles (/root/reference/proj/tests/*.cpp, restated; inputs seeded with numpy instead of
std::mt19937_64) and to the independent numpy restatement (oracle/fbmp_numpy.py).
CPU only: no GPU needed.
"""
import itertools

import numpy as np
import pytest

import fbmp_numpy as fnp
from paper_2103_09943_b200 import synth


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def simplex_kernel(rng, n):
    k = rng.uniform(0, 1, (n, n))
    return k / k.sum()


def dense(op, h, w):
    """tests/test_util.cpp:47-60 -- materialise a linear operator by unit probes."""
    cols = []
    for j in range(h * w):
        e = np.zeros(h * w)
        e[j] = 1.0
        cols.append(np.ravel(op(e.reshape(h, w))))
    return np.stack(cols, 1)


# ---- ops (tests/test_tensor_core.cpp) ------------------------------------------------------

def test_conv_dirac_identity(orc):  # :10-16
    img = np.random.default_rng(1).uniform(0, 1, (8, 8))
    k = np.zeros((3, 3))
    k[1, 1] = 1
    assert np.abs(orc.conv(img, k) - img).max() <= 1e-13


def test_conv_constants_and_mean(orc):  # :18-28
    rng = np.random.default_rng(2)
    k = simplex_kernel(rng, 5)
    assert np.abs(orc.conv(np.full((8, 8), 5.0), k) - 5.0).max() < 1e-12
    img = rng.uniform(0, 1, (12, 12))
    assert abs(orc.conv(img, k).mean() - img.mean()) < 1e-12


def test_conv_shifted_dirac_wrap(orc):  # :30-42
    img = np.zeros((4, 4))
    img[0, 0] = 1
    k = np.zeros((3, 3))
    k[1, 2] = 1
    out = orc.conv(img, k)
    expect = np.zeros((4, 4))
    expect[0, 1] = 1
    assert np.abs(out - expect).max() < 1e-12
    assert np.abs(out - fnp.conv_direct(img, k)).max() < 1e-12


@pytest.mark.parametrize("trial", range(5))
def test_conv_vs_spatial_oracle(orc, trial):  # :44-58
    rng = np.random.default_rng(3 + trial)
    img = rng.uniform(-1, 2, (16, 16))
    k = simplex_kernel(rng, 5 if trial % 2 else 3)
    assert rel(orc.conv(img, k), fnp.conv_direct(img, k)) < 1e-9


def test_conv_kernel_too_large(orc):  # :60-63
    with pytest.raises(orc.OracleError) as e:
        orc.conv(np.ones((4, 4)), np.eye(5))
    assert e.value.code == 2


def test_conv_adjoint_pairing(orc):  # :65-73
    rng = np.random.default_rng(4)
    k = simplex_kernel(rng, 5)
    x, y = rng.uniform(-1, 1, (10, 10)), rng.uniform(-1, 1, (10, 10))
    assert abs(np.vdot(orc.conv(x, k), y) - np.vdot(x, orc.conv(y, k, adjoint=True))) < 1e-10


def test_downsample_phase(orc):  # :75-91
    img = np.arange(16, dtype=float).reshape(4, 4)
    assert np.array_equal(orc.downsample(img, 2), [[0, 2], [8, 10]])
    with pytest.raises(orc.OracleError):
        orc.downsample(np.ones((5, 4)), 2)
    a = np.random.default_rng(5).uniform(0, 1, (6, 6))
    assert np.array_equal(orc.downsample(a, 1), a)


def test_upsample_adjoint(orc):  # :93-110
    assert np.array_equal(orc.upsample_adjoint(np.array([[3.0]]), 2), [[3, 0], [0, 0]])
    rng = np.random.default_rng(6)
    x, y = rng.uniform(-1, 1, (8, 8)), rng.uniform(-1, 1, (4, 4))
    assert abs(np.vdot(orc.downsample(x, 2), y) - np.vdot(x, orc.upsample_adjoint(y, 2))) < 1e-12
    lr = rng.uniform(0, 1, (4, 4))
    assert np.array_equal(orc.downsample(orc.upsample_adjoint(lr, 2), 2), lr)


def test_diff_ops(orc):  # :112-141
    for which in (orc.GH, orc.GV, orc.LAP):
        assert np.all(orc.diff(np.full((6, 7), 3.25), which) == 0)
    img = np.zeros((5, 5))
    img[2, 2] = 1
    out = orc.laplacian(img)
    assert out[2, 2] == 4 and out[1, 2] == -1 and out[3, 2] == -1 and out[2, 1] == -1 and out[2, 3] == -1
    assert out[0, 0] == 0
    rng = np.random.default_rng(7)
    for which in (orc.GH, orc.GV, orc.LAP):
        x, y = rng.uniform(-1, 1, (9, 11)), rng.uniform(-1, 1, (9, 11))
        assert abs(np.vdot(orc.diff(x, which), y) - np.vdot(x, orc.diff(y, which, adjoint=True))) < 1e-10


def test_box_mean(orc):  # :143-159
    assert np.abs(orc.box_mean(np.full((5, 5), 2.5), 2) - 2.5).max() < 1e-14
    img = np.random.default_rng(8).uniform(0, 1, (7, 7))
    assert np.array_equal(orc.box_mean(img, 0), img)
    assert np.abs(orc.box_mean(img, 1) - fnp.box_mean(img, 1)).max() < 1e-12
    with pytest.raises(orc.OracleError) as e:
        orc.box_mean(np.ones((3, 3)), 2)
    assert e.value.code == 2


def test_circular_box_blur_vs_convolution(orc):  # :161-172
    img = np.random.default_rng(9).uniform(0, 1, (8, 8))
    box = np.full((5, 5), 1 / 25)
    assert np.abs(orc.circular_box_blur(img, 5) - orc.conv(img, box)).max() < 1e-11


# ---- pansharpen (tests/test_pansharpen.cpp) -----------------------------------------------

def regression_oracle(x, guide, r, eps):  # :25-54
    h, w = guide.shape
    N = (2 * r + 1) ** 2
    total = 0.0
    for kr in range(r, h - r):
        for kc in range(r, w - r):
            X = x[kr - r:kr + r + 1, kc - r:kc + r + 1]
            I = guide[kr - r:kr + r + 1, kc - r:kc + r + 1]
            xbar, ibar = X.mean(), I.mean()
            var = (I * I).mean() - ibar * ibar
            cov = (I * X).mean() - ibar * xbar
            a = N * cov / (N * var + eps)
            c = xbar - a * ibar
            total += eps * a * a + ((X - a * I - c) ** 2).sum()
    return total


def test_matting_constant_guide(orc):  # :63-69
    M = orc.Matting(np.full((3, 3), 4.2), 1, 1e-4)
    D = dense(M.apply, 3, 3)
    assert np.abs(D - (np.eye(9) - 1 / 9)).max() < 1e-12


def test_matting_nullspace_symmetric_psd(orc):  # :71-88
    rng = np.random.default_rng(61)
    M = orc.Matting(rng.uniform(0, 1, (7, 6)), 1, 1e-4)
    assert np.abs(M.apply(np.full((7, 6), 3.7))).max() < 1e-10
    D = M.csr().toarray()
    assert np.abs(D - D.T).max() < 1e-12
    for _ in range(100):
        v = rng.uniform(-1, 1, 42)
        assert v @ D @ v >= -1e-10


@pytest.mark.parametrize("trial", range(4))
def test_matting_quadratic_form(orc, trial):  # :90-101
    rng = np.random.default_rng(62 + 10 * trial)
    guide = rng.uniform(0, 1, (6, 6))
    eps = 1e-4 if trial % 2 else 1e-2
    x = rng.uniform(-1, 1, (6, 6))
    quad = float(np.vdot(x, orc.Matting(guide, 1, eps).apply(x)))
    assert quad == pytest.approx(regression_oracle(x, guide, 1, eps), rel=1e-8)


def test_matting_window_stats(orc):  # :103-111
    guide = np.random.default_rng(63).uniform(0, 1, (8, 8))
    mean, _ = orc.Matting(guide, 1, 1e-4).stats()
    np.testing.assert_allclose(mean[1:7, 1:7], fnp.box_mean(guide, 1)[1:7, 1:7], rtol=1e-12)


def test_matting_vs_numpy_and_matrix_free(orc):
    rng = np.random.default_rng(64)
    guide = rng.uniform(0, 1, (20, 17))
    x = rng.uniform(-1, 1, (20, 17))
    y = orc.Matting(guide, 1, 1e-4).apply(x)
    assert rel(y, (fnp.matting_matrix(guide, 1, 1e-4) @ x.ravel()).reshape(x.shape)) < 1e-12
    assert rel(y, fnp.matting_apply_free(x, guide, 1, 1e-4)) < 1e-10


def test_warmstart_constant_channel(orc):  # :113-126
    rng = np.random.default_rng(64)
    pan = rng.uniform(0, 1, (16, 16))
    M = orc.Matting(orc.laplacian(pan), 1, 1e-4)
    z0, _, _, _ = orc.warmstart_cg(np.full((8, 8), 0.37), simplex_kernel(rng, 5), 2, M, cg_tol=1e-10, max_iters=4000)
    assert np.abs(z0 - 0.37).max() <= 1e-5 * 0.37


def test_warmstart_dirac_tiny_lambda(orc):  # :128-142
    rng = np.random.default_rng(65)
    pan = rng.uniform(0, 1, (8, 8))
    M = orc.Matting(orc.laplacian(pan), 1, 1e-4)
    x = rng.uniform(0, 1, (8, 8))
    k = np.zeros((3, 3))
    k[1, 1] = 1
    z0, _, _, _ = orc.warmstart_cg(x, k, 1, M, lam=1e-12, cg_tol=1e-12, max_iters=4000)
    assert np.abs(z0 - x).max() <= 1e-6 * np.abs(x).max()


def test_warmstart_dense_solve(orc):  # :144-170
    rng = np.random.default_rng(66)
    pan = rng.uniform(0, 1, (8, 8))
    guide = orc.laplacian(pan)
    M = orc.Matting(guide, 1, 1e-4)
    k = simplex_kernel(rng, 3)
    x = rng.uniform(0, 1, (4, 4))
    z0, _, _, _ = orc.warmstart_cg(x, k, 2, M, lam=0.01, cg_tol=1e-13, max_iters=20000, error_on_cap=False)
    A = dense(lambda z: orc.conv(orc.upsample_adjoint(orc.downsample(orc.conv(z, k), 2), 2), k, adjoint=True)
              + orc.laplacian(M.apply(orc.laplacian(z))) * 0.01, 8, 8)
    rhs = orc.conv(orc.upsample_adjoint(x, 2), k, adjoint=True).ravel()
    sol = np.linalg.lstsq(A, rhs, rcond=None)[0]
    assert np.linalg.norm(z0.ravel() - sol) <= 1e-6 * np.linalg.norm(sol)


def test_warmstart_dense_solve_identity_prior(orc):  # :144-170 with PriorKind::identity (pansharpen.cpp:28-50)
    rng = np.random.default_rng(166)
    pan = rng.uniform(0, 1, (8, 8))
    M = orc.Matting(pan, 1, 1e-4)  # the identity prior's guide is pan_n itself
    k = simplex_kernel(rng, 3)
    x = rng.uniform(0, 1, (4, 4))
    z0, _, _, _ = orc.warmstart_cg(x, k, 2, M, lam=0.01, cg_tol=1e-13, max_iters=20000, error_on_cap=False, prior=1)
    A = dense(lambda z: orc.conv(orc.upsample_adjoint(orc.downsample(orc.conv(z, k), 2), 2), k, adjoint=True)
              + M.apply(z) * 0.01, 8, 8)
    rhs = orc.conv(orc.upsample_adjoint(x, 2), k, adjoint=True).ravel()
    sol = np.linalg.lstsq(A, rhs, rcond=None)[0]
    assert np.linalg.norm(z0.ravel() - sol) <= 1e-6 * np.linalg.norm(sol)


def test_solve_fft_identity_prior_normal_equations(orc):  # :265-279 with the identity prior's symbol 1
    rng = np.random.default_rng(171)
    for factor in (1, 2):
        x, v = rng.uniform(0, 1, (8 // factor, 8 // factor)), rng.uniform(-0.5, 0.5, (8, 8))
        k = simplex_kernel(rng, 3)
        z = orc.solve_channel_fft(x, k, factor, v, 0.05, prior=1)
        lhs = orc.conv(orc.upsample_adjoint(orc.downsample(orc.conv(z, k), factor), factor), k, adjoint=True) + z * 0.05
        rhs = orc.conv(orc.upsample_adjoint(x, factor), k, adjoint=True) + v * 0.05
        assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(rhs)


def test_pansharpen_identity_prior_equal_bands(orc):  # :350-361 with PriorKind::identity
    sc = synth.make_scene("C1", hr=32)
    lr = np.stack([sc.lrms[0]] * 3)
    k = simplex_kernel(np.random.default_rng(5), 5)
    out, _ = orc.pansharpen(lr, sc.pan, k, 4, prior=1, threads=1)
    outl, _ = orc.pansharpen(lr, sc.pan, k, 4, prior=0, threads=1)
    assert np.abs(out[0] - out[1]).max() == 0.0 and np.abs(out[0] - out[2]).max() == 0.0
    assert rel(out, outl) > 1e-6  # a different prior, a different HRMS


def test_warmstart_cap(orc):  # :172-183
    rng = np.random.default_rng(67)
    pan = rng.uniform(0, 1, (16, 16))
    M = orc.Matting(orc.laplacian(pan), 1, 1e-4)
    with pytest.raises(orc.OracleError, match="did not converge in 2 iterations") as e:
        orc.warmstart_cg(rng.uniform(0, 1, (8, 8)), simplex_kernel(rng, 5), 2, M, cg_tol=1e-14, max_iters=2)
    assert e.value.code == 3


def test_guided_closed_forms(orc):  # :185-206
    guide = np.random.default_rng(68).uniform(0, 1, (7, 7))
    m = orc.guided_coeffs(guide, guide, 1, 1e-2)
    np.testing.assert_allclose(m["a"], m["guide_var"] / (m["guide_var"] + 1e-2), rtol=1e-10)
    np.testing.assert_allclose(m["c"], (1 - m["a"]) * m["guide_mean"], rtol=1e-9, atol=1e-12)
    mc = orc.guided_coeffs(np.full((7, 7), 1.25), guide, 1, 1e-2)
    assert np.abs(mc["a"]).max() < 1e-12 and np.abs(mc["c"] - 1.25).max() < 1e-12


def test_guided_regression_oracle(orc):  # :208-236
    rng = np.random.default_rng(69)
    guide, inp = rng.uniform(0, 1, (7, 7)), rng.uniform(-1, 1, (7, 7))
    m = orc.guided_coeffs(inp, guide, 1, 1e-3)
    for pr, pc in itertools.product(range(7), range(7)):
        sl = np.s_[max(0, pr - 1):min(6, pr + 1) + 1, max(0, pc - 1):min(6, pc + 1) + 1]
        mu, pb = guide[sl].mean(), inp[sl].mean()
        var = (guide[sl] ** 2).mean() - mu * mu
        cov = (guide[sl] * inp[sl]).mean() - mu * pb
        a = cov / (var + 1e-3)
        assert m["a"][pr, pc] == pytest.approx(a, rel=1e-10)
        assert m["c"][pr, pc] == pytest.approx(pb - a * mu, rel=1e-10)


def test_guided_output(orc):  # :238-263
    rng = np.random.default_rng(70)
    guide = rng.uniform(0, 1, (7, 7))
    assert np.abs(orc.guided_output(np.zeros((7, 7)), np.full((7, 7), 5.0), guide, 1) - 5).max() < 1e-12
    assert np.abs(orc.guided_output(np.ones((7, 7)), np.zeros((7, 7)), guide, 1) - guide).max() < 1e-12
    a, c = rng.uniform(-1, 1, (7, 7)), rng.uniform(-1, 1, (7, 7))
    expect = fnp.box_mean(a, 1) * guide + fnp.box_mean(c, 1)
    np.testing.assert_allclose(orc.guided_output(a, c, guide, 1), expect, rtol=1e-11)


def test_solve_fft_c1_normal_equations(orc):  # :265-279
    rng = np.random.default_rng(71)
    x, v = rng.uniform(0, 1, (8, 8)), rng.uniform(-0.5, 0.5, (8, 8))
    k = simplex_kernel(rng, 3)
    z = orc.solve_channel_fft(x, k, 1, v, 0.05)
    lhs = orc.conv(orc.conv(z, k), k, adjoint=True) + orc.laplacian(orc.laplacian(z)) * 0.05
    rhs = orc.conv(x, k, adjoint=True) + orc.laplacian(v) * 0.05
    assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(rhs)


def test_solve_fft_identity_limit(orc):  # :281-289
    x = np.random.default_rng(72).uniform(0, 1, (8, 8))
    k = np.zeros((3, 3))
    k[1, 1] = 1
    z = orc.solve_channel_fft(x, k, 1, np.zeros((8, 8)), 1e-12)
    assert np.abs(z - x).max() <= 1e-6 * np.abs(x).max()


@pytest.mark.parametrize("factor", [1, 2])
def test_solve_fft_vs_cg(orc, factor):  # :291-327
    rng = np.random.default_rng(73 + factor)
    x = rng.uniform(0, 1, (8 // factor, 8 // factor))
    v = rng.uniform(-0.2, 0.2, (8, 8))
    k = simplex_kernel(rng, 3)
    z = orc.solve_channel_fft(x, k, factor, v, 2e-4)
    A = dense(lambda p: orc.conv(orc.upsample_adjoint(orc.downsample(orc.conv(p, k), factor), factor), k, adjoint=True)
              + orc.laplacian(orc.laplacian(p)) * 2e-4, 8, 8)
    rhs = (orc.conv(orc.upsample_adjoint(x, factor), k, adjoint=True) + orc.laplacian(v) * 2e-4).ravel()
    zc = np.linalg.solve(A, rhs)
    assert np.linalg.norm(z.ravel() - zc) <= 1e-7 * np.linalg.norm(zc)


def test_solve_fft_minimiser(orc):  # :329-348
    rng = np.random.default_rng(74)
    x, v = rng.uniform(0, 1, (4, 4)), rng.uniform(-0.2, 0.2, (8, 8))
    k = simplex_kernel(rng, 3)
    z = orc.solve_channel_fft(x, k, 2, v, 1e-3)

    def obj(p):
        r = orc.downsample(orc.conv(p, k), 2) - x
        q = orc.laplacian(p) - v
        return 0.5 * np.vdot(r, r) + 0.5e-3 * np.vdot(q, q)
    base = obj(z)
    for _ in range(20):
        assert obj(z + rng.uniform(-1, 1, (8, 8)) * 1e-3) >= base - 1e-12


def test_solve_fft_vs_numpy(orc):
    rng = np.random.default_rng(75)
    x, v = rng.uniform(0, 1, (16, 16)), rng.uniform(-0.5, 0.5, (64, 64))
    k = simplex_kernel(rng, 7)
    assert rel(orc.solve_channel_fft(x, k, 4, v, 2e-4), fnp.solve_channel_fft(x, k, 4, v, 2e-4)) < 1e-11


def test_pansharpen_equal_bands(orc):  # :350-361
    sc = synth.make_scene("C1", hr=32)
    lr = sc.lrms[0]
    out, _ = orc.pansharpen(np.stack([lr, lr, lr]), sc.pan, simplex_kernel(np.random.default_rng(1), 3), 4, threads=3)
    assert np.array_equal(out[1], out[0]) and np.array_equal(out[2], out[0])


def test_pansharpen_channel_annotation(orc):  # :389-403
    sc = synth.make_scene("C1", hr=32)
    with pytest.raises(orc.OracleError, match="channel") as e:
        orc.pansharpen(sc.lrms[:2], sc.pan, simplex_kernel(np.random.default_rng(76), 3), 4, cg_tol=1e-15,
                       cg_max_iter=1)
    assert e.value.code == 3


def test_pansharpen_validation(orc):  # :405-415
    sc = synth.make_scene("C1", hr=32)
    for kw in (dict(lam=0.0), dict(radius=0)):
        with pytest.raises(orc.OracleError) as e:
            orc.pansharpen(sc.lrms, sc.pan, np.ones((3, 3)) / 9, 4, **kw)
        assert e.value.code == 1


# ---- kernel estimator (tests/test_kernel_estimator.cpp) -----------------------------------

def test_observation_dirac_image(orc):  # :117-127
    y = np.zeros((6, 6))
    y[0, 0] = 1
    E = orc.observation_matrix(y, 1, 3)
    assert all((E[:, c] != 0).sum() == 1 for c in range(9))


def test_observation_dirac_kernel(orc):  # :129-138
    y = np.random.default_rng(41).uniform(0, 1, (8, 8))
    d = np.zeros(9)
    d[4] = 1
    np.testing.assert_allclose(orc.observation_matrix(y, 2, 3) @ d, orc.downsample(y, 2).ravel(), rtol=1e-12)


def test_observation_random_kernels(orc):  # :140-151
    rng = np.random.default_rng(42)
    y = rng.uniform(0, 1, (8, 8))
    E = orc.observation_matrix(y, 2, 3)
    for _ in range(20):
        k = simplex_kernel(rng, 3)
        np.testing.assert_allclose(E @ k.ravel(), orc.downsample(orc.conv(y, k), 2).ravel(), rtol=1e-9)


def test_gram_matches_E(orc):
    rng = np.random.default_rng(43)
    pan, obs = rng.uniform(0, 1, (16, 16)), rng.uniform(0, 1, (8, 8))
    E = orc.observation_matrix(pan, 2, 5)
    G, e = orc.gram(pan, obs, 2, 5)
    np.testing.assert_allclose(G, E.T @ E, rtol=1e-12)
    np.testing.assert_allclose(e, E.T @ obs.ravel(), rtol=1e-12)


def test_shrink2_kats(orc):  # :153-176
    row = lambda a, b: [np.array([[a]]), np.array([[b]])]  # noqa: E731
    assert [c[0, 0] for c in orc.shrink2(row(3.0, 4.0), 5.0)] == [0.0, 0.0]
    np.testing.assert_allclose([c[0, 0] for c in orc.shrink2(row(3.0, 4.0), 1.0)], [2.4, 3.2])
    np.testing.assert_allclose([c[0, 0] for c in orc.shrink2(row(3.0, 4.0), 0.0)], [3.0, 4.0])
    assert [c[0, 0] for c in orc.shrink2(row(0.0, 0.0), 0.5)] == [0.0, 0.0]


def brute_force_simplex(v):  # :84-113
    n = len(v)
    best, best_d = np.zeros(n), np.inf
    for mask in range(1, 1 << n):
        idx = [i for i in range(n) if mask >> i & 1]
        tau = (1 - v[idx].sum()) / len(idx)
        s = np.zeros(n)
        s[idx] = v[idx] + tau
        if (s[idx] < -1e-12).any():
            continue
        d = ((s - v) ** 2).sum()
        if d < best_d:
            best, best_d = s, d
    return best


def test_project_simplex(orc):  # :178-207
    np.testing.assert_allclose(orc.project_simplex(np.array([0.2, 0.8])), [0.2, 0.8])
    np.testing.assert_allclose(orc.project_simplex(np.array([2.0, 0.0])), [1.0, 0.0])
    np.testing.assert_allclose(orc.project_simplex(np.array([0.5, 0.7])), [0.4, 0.6])
    rng = np.random.default_rng(43)
    for n in (4, 9, 16 if False else 12):
        for _ in range(10):
            v = rng.uniform(-2, 2, n)
            f = orc.project_simplex(v)
            assert np.linalg.norm(f - brute_force_simplex(v)) < 1e-9
            assert f.sum() == pytest.approx(1.0, abs=1e-12) and f.min() >= 0


def test_solve_z(orc):  # :209-235
    anchor = np.arange(9) * 0.1 - 0.3
    z = orc.solve_z(np.zeros((6, 6)), np.zeros((3, 3)), 2, 3, 2.5, anchor)
    assert np.linalg.norm(z - anchor) < 1e-12
    rng = np.random.default_rng(44)
    pan, obs = rng.uniform(0, 1, (16, 16)), rng.uniform(0, 1, (8, 8))
    a2 = np.sin(np.arange(9) * 1.7)
    E = orc.observation_matrix(pan, 2, 3)
    slow = np.linalg.solve(E.T @ E + 100 * np.eye(9), E.T @ obs.ravel() + 100 * a2)
    assert np.linalg.norm(orc.solve_z(pan, obs, 2, 3, 100.0, a2) - slow) <= 1e-10 * np.linalg.norm(slow)


def up_dense(x, y, L1, L2, a1m1, a2m2, n):  # :31-76
    Dh = dense(lambda p: np.roll(p, -1, 1) - p, n, n)
    Dv = dense(lambda p: np.roll(p, -1, 0) - p, n, n)
    I = np.eye(n * n)
    d1 = a1m1 * (Dh.T @ Dh + Dv.T @ Dv)
    d2 = a1m1 * I + 0.5 * a2m2 * Dv.T @ Dv + a2m2 * Dh.T @ Dh
    d3 = a1m1 * I + 0.5 * a2m2 * Dh.T @ Dh + a2m2 * Dv.T @ Dv
    d4, d5, d6 = -a1m1 * Dh, -a1m1 * Dv, 0.5 * a2m2 * Dh.T @ Dv
    A = np.block([[d1, d4.T, d5.T], [d4, d2, d6.T], [d5, d6, d3]])
    x1, x2 = (x[0] - L1[0]).ravel(), (x[1] - L1[1]).ravel()
    y1, y2 = (y[0] - L2[0]).ravel(), (y[3] - L2[3]).ravel()
    yc = 0.5 * (y[1] - L2[1] + y[2] - L2[2]).ravel()
    rhs = np.concatenate([a1m1 * (Dh.T @ x1 + Dv.T @ x2), -a1m1 * x1 + a2m2 * (Dh.T @ y1 + Dv.T @ yc),
                          -a1m1 * x2 + a2m2 * (Dv.T @ y2 + Dh.T @ yc)])
    return np.linalg.lstsq(A, rhs, rcond=None)[0]


def test_solve_up_homogeneous_linear(orc):  # :237-264
    n = 4
    z = [np.zeros((n, n))]
    u, p1, p2 = orc.solve_up(z * 2, z * 4, z * 2, z * 4, 0.9, 0.31, 2.0, 3.0)
    assert max(np.abs(u).max(), np.abs(p1).max(), np.abs(p2).max()) < 1e-14
    rng = np.random.default_rng(45)
    cr = rng.uniform(-1, 1, (n, n))
    x = [rng.uniform(-1, 1, (n, n)) for _ in range(2)]
    y = [rng.uniform(-1, 1, (n, n)), cr, cr, rng.uniform(-1, 1, (n, n))]
    s1 = orc.solve_up(x, y, z * 2, z * 4, 0.9, 0.31, 2.0, 3.0)
    s3 = orc.solve_up([3 * a for a in x], [3 * a for a in y], z * 2, z * 4, 0.9, 0.31, 2.0, 3.0)
    assert np.linalg.norm(s3[0] - 3 * s1[0]) < 1e-10 * np.linalg.norm(s3[0]) + 1e-14


@pytest.mark.parametrize("trial", range(20))
def test_solve_up_vs_dense(orc, trial):  # :266-295
    n = 4
    rng = np.random.default_rng(46 + trial)
    u = lambda: rng.uniform(-1, 1, (n, n))  # noqa: E731
    x = [u(), u()]
    cr = u()
    y = [u(), cr, cr, u()]
    L1 = [u(), u()]
    lc = u()
    L2 = [u(), lc, lc, u()]
    fast = np.concatenate([a.ravel() for a in orc.solve_up(x, y, L1, L2, 1.0, 0.5, 1.5, 0.8)])
    slow = up_dense(x, y, L1, L2, 1.5, 0.4, n)
    assert np.linalg.norm(fast - slow) <= 1e-8 * np.linalg.norm(slow)


def test_degenerate_pan(orc):  # :297-305
    with pytest.raises(orc.OracleError, match="constant PAN") as e:
        orc.estimate_kernel_plane(np.ones((16, 16)), np.full((8, 8), 0.5), 2, 3)
    assert e.value.code == 3


def test_kernel_param_validation(orc):  # :307-317
    pan = np.random.default_rng(0).uniform(0, 1, (16, 16))
    for kw in (dict(rho=2.0), dict(alpha1=0.0)):
        with pytest.raises(orc.OracleError) as e:
            orc.estimate_kernel_plane(pan, pan[::2, ::2], 2, 3, **kw)
        assert e.value.code == 1
    with pytest.raises(orc.OracleError):
        orc.estimate_kernel_plane(pan, pan[::2, ::2], 2, 4)


def test_solve_up_along_admm(orc):  # :319-342 (hook point = state before the {u,p} solve)
    sc = synth.make_scene("C1", hr=32)
    obs = orc.combine_bands(sc.lrms, np.full(4, 0.25))
    for t in range(5):
        _, _, st = orc.estimate_kernel_plane(sc.pan, obs, 4, 5, hook_t=t, t_max=5, th=1e-14)
        fast = np.concatenate([a.ravel() for a in orc.solve_up(
            [st["x0"], st["x1"]], [st["y0"], st["y1"], st["y2"], st["y3"]], [st["L1_0"], st["L1_1"]],
            [st["L2_0"], st["L2_1"], st["L2_2"], st["L2_3"]], 1.0, 0.006, 100.0, 100.0)])
        slow = up_dense([st["x0"], st["x1"]], [st["y0"], st["y1"], st["y2"], st["y3"]], [st["L1_0"], st["L1_1"]],
                        [st["L2_0"], st["L2_1"], st["L2_2"], st["L2_3"]], 100.0, 0.6, 5)
        assert np.linalg.norm(fast - slow) <= 1e-8 * (np.linalg.norm(slow) + 1)


def texture(h, w, seed):
    """tests/test_util.cpp:62-90 in spirit: low-frequency waves plus random rectangles (numpy rng)."""
    rng = np.random.default_rng(seed)
    r, c = np.mgrid[0:h, 0:w]
    f1, f2, ph1, ph2 = 1 + 2 * rng.uniform(), 1 + 2 * rng.uniform(), 2 * np.pi * rng.uniform(), 2 * np.pi * rng.uniform()
    img = 0.5 + 0.25 * np.sin(2 * np.pi * f1 * r / h + ph1) + 0.25 * np.cos(2 * np.pi * f2 * c / w + ph2)
    for _ in range(6 + int(rng.uniform() * 6)):
        y0, x0 = rng.integers(0, h - 4), rng.integers(0, w - 4)
        img[y0:y0 + rng.integers(3, h // 3), x0:x0 + rng.integers(3, w // 3)] += rng.uniform(-0.3, 0.3)
    return img


def test_tv_degenerate_pan(orc):  # :297-305 (estimate_kernel_tv)
    with pytest.raises(orc.OracleError, match="constant PAN") as e:
        orc.estimate_kernel_plane_tv(np.ones((16, 16)), np.full((8, 8), 0.5), 2, 3)
    assert e.value.code == 3


def test_tv_recovers_noiseless_system(orc):  # :386-397 (KernelPrior::tv, alpha1 -> 0)
    pan = texture(32, 32, 9)
    rng = np.random.default_rng(9)
    truth = simplex_kernel(rng, 3)
    obs = (orc.observation_matrix(pan, 2, 3) @ truth.ravel()).reshape(16, 16)
    est, it = orc.estimate_kernel_plane_tv(pan, obs, 2, 3, alpha1=1e-6, t_max=4000, th=1e-9)
    assert 100 * np.linalg.norm(est - truth) / np.linalg.norm(truth) < 1.0
    assert abs(est.sum() - 1.0) < 1e-9 and est.min() >= 0.0


def test_tv_state_has_no_p(orc):  # :291-387 with with_p = false: p, y and L2 stay zero
    sc = synth.make_scene("C1", hr=32)
    obs = orc.combine_bands(sc.lrms, np.full(4, 0.25))
    k, it, st = orc.estimate_kernel_plane_tv(sc.pan, obs, 4, 5, want_state=True)
    for f in ("p1", "p2", "y0", "y1", "y2", "y3", "L2_0", "L2_1", "L2_2", "L2_3"):
        assert not st[f].any()
    kt, _ = orc.estimate_kernel_plane(sc.pan, obs, 4, 5)
    assert it > 1 and rel(k, kt) > 1e-6  # a different prior, a different kernel


def test_primal_residuals_at_convergence(orc):  # :357-384
    sc = synth.make_scene("C1", hr=32)
    obs = orc.combine_bands(sc.lrms, np.full(4, 0.25))
    _, _, s = orc.estimate_kernel_plane(sc.pan, obs, 4, 5, want_state=True, t_max=6000, th=1e-10)
    un = max(np.linalg.norm(s["u"]), 1e-30)
    r1 = np.hypot(np.linalg.norm(np.roll(s["u"], -1, 1) - s["u"] - s["p1"] - s["x0"]),
                  np.linalg.norm(np.roll(s["u"], -1, 0) - s["u"] - s["p2"] - s["x1"]))
    assert r1 < 1e-6 * un
    assert np.linalg.norm(s["u"] - s["z"]) < 1e-6 * un


def test_objective_init_invariance(orc):  # :430-457
    sc = synth.make_scene("C1", hr=40 * 4 // 4 if False else 32)
    obs = orc.combine_bands(sc.lrms, np.full(4, 0.25))
    k1, _, s1 = orc.estimate_kernel_plane(sc.pan, obs, 4, 5, want_state=True, t_max=20000, th=1e-10)
    k2, _, s2 = orc.estimate_kernel_plane(sc.pan, obs, 4, 5, want_state=True, t_max=20000, th=1e-10, init=1)
    s = orc.intensity_scale(sc.pan, 4)
    o1 = orc.tgv_objective(sc.pan * s, obs * s, 4, 5, s1["z"], s1["p1"], s1["p2"])
    o2 = orc.tgv_objective(sc.pan * s, obs * s, 4, 5, s2["z"], s2["p1"], s2["p2"])
    assert abs(o1 - o2) <= 1e-6 * max(o1, o2)
    assert np.linalg.norm(k1 - k2) / np.linalg.norm(k2) < 1e-3


# ---- spectral weights (tests/test_spectral_weights.cpp) ------------------------------------

def test_weights_single_band(orc):  # :46-61
    pan = np.random.default_rng(5).uniform(0, 1, (32, 32))
    degraded = orc.downsample(orc.circular_box_blur(pan, 9), 2)
    band = degraded / 0.4
    w = orc.solve_weights(band[None], pan, 4, 0.0, 2)
    a = orc.circular_box_blur(band, 5)
    assert w[0] == pytest.approx(np.vdot(a, degraded) / np.vdot(a, a), rel=1e-12)


def test_weights_dense_oracle(orc):  # :86-97
    rng = np.random.default_rng(32)
    lrms, pan = rng.uniform(0, 1, (4, 16, 16)), rng.uniform(0, 1, (32, 32))
    A = np.stack([orc.circular_box_blur(b, 5).ravel() for b in lrms], 1)
    b = orc.downsample(orc.circular_box_blur(pan, 9), 2).ravel()
    G = np.diff(np.eye(4), axis=0)
    expect = np.linalg.solve(A.T @ A + 10 * G.T @ G, A.T @ b)
    np.testing.assert_allclose(orc.solve_weights(lrms, pan, 4, 10.0, 2), expect, rtol=1e-9)
    np.testing.assert_allclose(fnp.solve_weights(lrms, pan, 4, 10.0, 2), expect, rtol=1e-9)


def test_weights_scale_invariance(orc):  # :128-141
    rng = np.random.default_rng(34)
    lrms, pan = rng.uniform(0, 1, (3, 16, 16)), rng.uniform(0, 1, (32, 32))
    np.testing.assert_allclose(orc.solve_weights(lrms, pan, 2, 0.0, 2),
                               orc.solve_weights(lrms * 7.5, pan * 7.5, 2, 0.0, 2), rtol=1e-9)


def test_weights_singular(orc):  # :143-147
    with pytest.raises(orc.OracleError) as e:
        orc.solve_weights(np.ones((2, 8, 8)), np.full((16, 16), 2.0), 2, 0.0, 2)
    assert e.value.code == 3


def test_weights_validation(orc):  # :149-154
    one = np.ones((1, 8, 8))
    for args, code in (((one, np.ones((15, 16)), 4, 10.0, 2), 2), ((one, np.ones((16, 16)), 0, 10.0, 2), 1),
                       ((one, np.ones((16, 16)), 4, -1.0, 2), 1)):
        with pytest.raises(orc.OracleError) as e:
            orc.solve_weights(*args)
        assert e.value.code == code


def test_combine_bands(orc):  # :156-164
    rng = np.random.default_rng(35)
    lrms = rng.uniform(0, 1, (2, 4, 4))
    np.testing.assert_allclose(orc.combine_bands(lrms, [0.25, 0.75]), 0.25 * lrms[0] + 0.75 * lrms[1])


# ---- end to end: C++ oracle vs the independent numpy restatement ---------------------------

def test_blind_oracle_vs_numpy(orc):
    """PR1 reference config. (Smaller scenes, e.g. 64^2 with n = 7, are CG-chaotic: the two
    restatements differ there by one iteration -- see DESIGN.md, CG trajectory sensitivity.)"""
    sc = synth.make_scene("C1")
    out_c, ic = orc.blind(sc.lrms, sc.pan, 4, 15, threads=4)
    out_n, inn = fnp.blind(sc.lrms, sc.pan, 4, 15)
    assert ic["admm_iters"] == inn["admm_iters"]
    assert rel(ic["kernel"], inn["kernel"]) < 1e-9
    assert list(ic["cg_iters"]) == list(inn["cg_iters"])
    assert rel(out_c, out_n) < 1e-6


# ---- the alias-group eigen-solver (Eigen::SelfAdjointEigenSolver at pansharpen.cpp:353) ------

@pytest.mark.parametrize("n,kind", [(3, "gram"), (9, "gram"), (16, "gram"), (16, "alias"), (16, "graded")])
def test_herm_eig_ql(orc, n, kind):
    """Householder + QL (used by the alias solve) agrees with LAPACK and with the Jacobi solver:
    eigenvalues to eps ||A||, A = V diag(ev) V^H, V unitary, eigenvalues ascending."""
    rng = np.random.default_rng(n * 7 + len(kind))
    for _ in range(4):
        if kind == "gram":
            B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
            A = B @ B.conj().T
        elif kind == "alias":  # b b^H / c^2 + lambda |l|^2 on the diagonal (the alias-group system)
            b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            A = np.outer(b.conj(), b) / n + np.diag(rng.uniform(1e-6, 2.0, n))
        else:  # widely graded spectrum (condition ~1e12)
            Qm, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
            A = (Qm * np.logspace(-12, 0, n)) @ Qm.conj().T
            A = 0.5 * (A + A.conj().T)
        ev, V = orc.herm_eig(A, 0)
        ev_j, _ = orc.herm_eig(A, 1)
        scale = np.abs(np.linalg.eigvalsh(A)).max()
        assert np.all(np.diff(ev) >= 0)
        assert np.abs(ev - np.linalg.eigvalsh(A)).max() < 1e-13 * scale
        assert np.abs(ev - ev_j).max() < 1e-13 * scale
        assert np.linalg.norm(V @ np.diag(ev) @ V.conj().T - A) < 1e-13 * np.linalg.norm(A)
        assert np.linalg.norm(V.conj().T @ V - np.eye(n)) < 1e-13
