"""GPU parity of the unit operators against the CPU oracle (through the C ABI).

Each check restates a reference test or compares one reference function
(/root/reference/proj/src/*.cpp) with its oracle restatement on seeded inputs.
Tolerances are fp64 round-off bounds (the GPU sums in a different order).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def simplex_kernel(rng, n):
    k = rng.uniform(0, 1, (n, n))
    return k / k.sum()


@pytest.mark.parametrize("shape,r", [((7, 7), 1), ((16, 20), 2), ((33, 31), 1), ((5, 5), 2)])
def test_box_mean(gpu, orc, shape, r):
    img = np.random.default_rng(8).uniform(0, 1, shape)
    assert rel(gpu.box_mean(img, r), orc.box_mean(img, r)) < 1e-13


def test_box_mean_errors(gpu):
    with pytest.raises(gpu.DimensionError):
        gpu.box_mean(np.ones((3, 3)), 2)  # tests/test_tensor_core.cpp:158


@pytest.mark.parametrize("n", [1, 3, 5, 7])
def test_convolve_and_adjoint(gpu, orc, n):
    rng = np.random.default_rng(3 + n)
    img = rng.uniform(-1, 2, (16, 12))
    k = simplex_kernel(rng, n)
    assert rel(gpu.circular_convolve(img, k), orc.conv(img, k)) < 1e-13
    assert rel(gpu.circular_convolve_adjoint(img, k), orc.conv(img, k, adjoint=True)) < 1e-13


def test_convolve_shifted_dirac(gpu):  # tests/test_tensor_core.cpp:30-42
    img = np.zeros((4, 4))
    img[0, 0] = 1.0
    k = np.zeros((3, 3))
    k[1, 2] = 1.0
    out = gpu.circular_convolve(img, k)
    expect = np.zeros((4, 4))
    expect[0, 1] = 1.0
    assert np.abs(out - expect).max() < 1e-15


def test_laplacian_kat(gpu):  # tests/test_tensor_core.cpp:120-130
    img = np.zeros((5, 5))
    img[2, 2] = 1.0
    out = gpu.apply_prior(img)
    assert out[2, 2] == 4.0 and out[1, 2] == -1.0 and out[3, 2] == -1.0
    assert out[2, 1] == -1.0 and out[2, 3] == -1.0 and out[0, 0] == 0.0


def test_laplacian_bitexact(gpu, orc):
    img = np.random.default_rng(1).uniform(0, 1, (37, 29))
    assert np.array_equal(gpu.apply_prior(img), orc.laplacian(img))


@pytest.mark.parametrize("shape,eps", [((6, 6), 1e-4), ((7, 6), 1e-2), ((40, 33), 1e-4), ((64, 64), 1e-4)])
def test_matting_apply_vs_assembled(gpu, orc, shape, eps):
    """Matrix-free M x vs the oracle's assembled CSR SpMV (pansharpen.cpp:117-202)."""
    rng = np.random.default_rng(61)
    guide = rng.uniform(0, 1, shape)
    x = rng.uniform(-1, 1, shape)
    M = orc.Matting(guide, 1, eps)
    assert rel(gpu.MattingMatrix(guide, 1, eps).apply(x), M.apply(x)) < 1e-11


def test_matting_constant_guide(gpu):  # tests/test_pansharpen.cpp:63-69
    M = gpu.MattingMatrix(np.full((3, 3), 4.2), 1, 1e-4)
    dense = np.stack([M.apply(e.reshape(3, 3)).ravel() for e in np.eye(9)], 1)
    assert np.abs(dense - (np.eye(9) - 1.0 / 9.0)).max() < 1e-12


def test_matting_nullspace_symmetry(gpu):  # tests/test_pansharpen.cpp:71-88
    guide = np.random.default_rng(61).uniform(0, 1, (7, 6))
    M = gpu.MattingMatrix(guide, 1, 1e-4)
    assert np.abs(M.apply(np.full((7, 6), 3.7))).max() < 1e-10
    dense = np.stack([M.apply(e.reshape(7, 6)).ravel() for e in np.eye(42)], 1)
    assert np.abs(dense - dense.T).max() < 1e-12
    assert np.linalg.eigvalsh(0.5 * (dense + dense.T)).min() >= -1e-10


def test_matting_radius2(gpu, orc):
    rng = np.random.default_rng(5)
    guide = rng.uniform(0, 1, (20, 24))
    x = rng.uniform(-1, 1, (20, 24))
    assert rel(gpu.MattingMatrix(guide, 2, 1e-3).apply(x), orc.Matting(guide, 2, 1e-3).apply(x)) < 1e-11


@pytest.mark.parametrize("H,W,n,c", [(8, 8, 3, 2), (16, 12, 5, 2), (64, 64, 15, 4), (40, 48, 17, 4), (12, 12, 3, 1)])
def test_data_term(gpu, orc, H, W, n, c):
    rng = np.random.default_rng(H * W + n)
    p = rng.uniform(-1, 1, (H, W))
    k = simplex_kernel(rng, n)
    expect = orc.conv(orc.upsample_adjoint(orc.downsample(orc.conv(p, k), c), c), k, adjoint=True)
    assert rel(gpu.data_apply(p, k, c), expect) < 1e-13


@pytest.mark.parametrize("H,W,n,c", [(8, 8, 3, 2), (64, 64, 15, 4), (48, 40, 7, 4),
                                     (65, 67, 3, 1), (96, 80, 5, 2), (128, 72, 11, 4), (128, 200, 21, 4),
                                     (64, 112, 17, 4),
                                     (512, 640, 17, 4),   # K_Q3: LR width 160 = two full bands + a partial one
                                     (512, 512, 21, 4), (768, 512, 7, 4)])
def test_cg_operator(gpu, orc, H, W, n, c):
    """Covers every operator variant: single-column / column-pair K_L (odd / even W, partial
    bands), register-tap and generic K_D, tile K_Q2, row-streaming K_Q3 (LR width >= 128)
    and generic K_Q, c in {1, 2, 4}."""
    rng = np.random.default_rng(7 * H + n)
    guide = orc.laplacian(rng.uniform(0, 1, (H, W)))
    p = rng.uniform(-1, 1, (H, W))
    k = simplex_kernel(rng, n)
    M = orc.Matting(guide, 1, 1e-4)
    data = orc.conv(orc.upsample_adjoint(orc.downsample(orc.conv(p, k), c), c), k, adjoint=True)
    expect = data + orc.laplacian(M.apply(orc.laplacian(p))) * 2e-4
    # the oracle's summed-area-table box means lose digits as the image grows
    assert rel(gpu.cg_operator(guide, p, k, c), expect) < (1e-12 if H * W < 100_000 else 1e-11)


@pytest.mark.parametrize("shape,r,eps", [((7, 7), 1, 1e-2), ((7, 7), 1, 1e-3), ((50, 45), 1, 1e-4), ((30, 30), 2, 1e-3)])
def test_guided_coeffs_and_output(gpu, orc, shape, r, eps):
    rng = np.random.default_rng(69)
    guide = rng.uniform(0, 1, shape)
    inp = rng.uniform(-1, 1, shape)
    g = gpu.guided_coeffs(inp, guide, r, eps)
    o = orc.guided_coeffs(inp, guide, r, eps)
    assert rel(g["a"], o["a"]) < 1e-10 and rel(g["c"], o["c"]) < 1e-10
    v = gpu.guided_output(g, guide, r)
    assert rel(v, orc.guided_output(o["a"], o["c"], guide, r)) < 1e-10
    assert rel(gpu.guided_filter(inp, guide, r, eps), v) < 1e-14


@pytest.mark.parametrize("shape", [(64, 64), (96, 130), (256, 192), (17, 64)])
def test_guided_filter_streaming(gpu, orc, shape):
    """The row-streaming guided filter (k_guided3: radius 1, even width >= 64) against the oracle's
    guided_output(guided_coeffs(.)) with summed-area-table box means (pansharpen.cpp:274-312)."""
    rng = np.random.default_rng(shape[0] + shape[1])
    guide = rng.uniform(0, 1, shape)
    inp = rng.uniform(-1, 1, shape)
    o = orc.guided_coeffs(inp, guide, 1, 1e-4)
    assert rel(gpu.guided_filter(inp, guide, 1, 1e-4), orc.guided_output(o["a"], o["c"], guide, 1)) < 1e-10


def test_guided_closed_forms(gpu):  # tests/test_pansharpen.cpp:185-206
    guide = np.random.default_rng(68).uniform(0, 1, (7, 7))
    m = gpu.guided_coeffs(np.full((7, 7), 1.25), guide, 1, 1e-2)
    assert np.abs(m["a"]).max() < 1e-12 and np.abs(m["c"] - 1.25).max() < 1e-12


@pytest.mark.parametrize("h,w,n,c,lam", [(8, 8, 3, 1, 0.05), (4, 4, 3, 2, 1e-3), (16, 16, 5, 4, 2e-4),
                                         (64, 64, 15, 4, 2e-4), (32, 24, 7, 2, 2e-4)])
def test_solve_channel_fft(gpu, orc, h, w, n, c, lam):
    rng = np.random.default_rng(71 + h + n)
    x = rng.uniform(0, 1, (h, w))
    v = rng.uniform(-0.5, 0.5, (h * c, w * c))
    k = simplex_kernel(rng, n)
    prm = gpu.PansharpenParams(lambda_=lam)
    assert rel(gpu.solve_channel_fft(x, k, c, v, prm), orc.solve_channel_fft(x, k, c, v, lam)) < 1e-10


def test_solve_channel_fft_identity(gpu):  # tests/test_pansharpen.cpp:281-289
    x = np.random.default_rng(72).uniform(0, 1, (8, 8))
    k = np.zeros((3, 3))
    k[1, 1] = 1
    z = gpu.solve_channel_fft(x, k, 1, np.zeros((8, 8)), gpu.PansharpenParams(lambda_=1e-12))
    assert np.abs(z - x).max() <= 1e-6 * np.abs(x).max()


def test_shrink2_kats(gpu):  # tests/test_kernel_estimator.cpp:153-176
    def row(a, b):
        return [np.array([[a]]), np.array([[b]])]
    out = gpu.shrink2(row(3.0, 4.0), 5.0)
    assert out[0][0, 0] == 0 and out[1][0, 0] == 0
    out = gpu.shrink2(row(3.0, 4.0), 1.0)
    assert abs(out[0][0, 0] - 2.4) < 1e-15 and abs(out[1][0, 0] - 3.2) < 1e-15
    out = gpu.shrink2(row(0.0, 0.0), 0.5)
    assert out[0][0, 0] == 0 and out[1][0, 0] == 0


def test_project_simplex(gpu, orc):  # tests/test_kernel_estimator.cpp:178-207
    np.testing.assert_allclose(gpu.project_simplex(np.array([0.5, 0.7])), [0.4, 0.6], atol=1e-15)
    np.testing.assert_allclose(gpu.project_simplex(np.array([2.0, 0.0])), [1.0, 0.0], atol=1e-15)
    rng = np.random.default_rng(43)
    for m in (4, 9, 16, 225, 289, 441):
        v = rng.uniform(-2, 2, m)
        g = gpu.project_simplex(v)
        assert np.abs(g - orc.project_simplex(v)).max() < 1e-14
        assert abs(g.sum() - 1) < 1e-12 and g.min() >= 0
    v = np.array([0.3, 0.3, 0.3, -1.0, 0.3])  # ties
    assert np.abs(gpu.project_simplex(v) - orc.project_simplex(v)).max() < 1e-15


@pytest.mark.parametrize("n,coupling", [(4, 0.0), (5, 0.0), (15, 100.0), (17, 100.0)])
def test_solve_up(gpu, orc, n, coupling):
    rng = np.random.default_rng(46 + n)
    cross = rng.uniform(-1, 1, (n, n))
    x = [rng.uniform(-1, 1, (n, n)) for _ in range(2)]
    y = [rng.uniform(-1, 1, (n, n)), cross, cross, rng.uniform(-1, 1, (n, n))]
    lc = rng.uniform(-1, 1, (n, n))
    L1 = [rng.uniform(-1, 1, (n, n)) for _ in range(2)]
    L2 = [rng.uniform(-1, 1, (n, n)), lc, lc, rng.uniform(-1, 1, (n, n))]
    anchor = rng.uniform(-1, 1, (n, n)) if coupling else None
    prm = gpu.KernelEstParams(alpha1=1.0, alpha2=0.5, mu1=1.5, mu2=0.8)
    g = gpu.solve_up(x, y, L1, L2, prm, coupling, anchor)
    o = orc.solve_up(x, y, L1, L2, 1.0, 0.5, 1.5, 0.8, coupling, anchor)
    for a, b in zip(g, o):
        assert np.abs(a - b).max() <= 1e-11 * (np.abs(b).max() + 1)


@pytest.mark.parametrize("H,c,n,mu3", [(16, 2, 3, 100.0), (64, 4, 7, 5.0), (128, 4, 15, 100.0)])
def test_solve_z_and_objective(gpu, orc, H, c, n, mu3):
    """Public ObservationSystem::solve_z / data_objective (kernel_estimator.cpp:79-87) on the device
    against the oracle's dense Cholesky solve and the direct 0.5 ||E u - f||^2."""
    rng = np.random.default_rng(H + n)
    pan = rng.uniform(0, 1, (H, H))
    obs = rng.uniform(0, 1, (H // c, H // c))
    anchor = rng.uniform(-1, 1, n * n)
    G, e = gpu.gram(pan, obs, c, n)
    z = gpu.solve_z(G, e, n, mu3, anchor)
    zo = orc.solve_z(pan, obs, c, n, mu3, anchor)
    assert rel(z, zo) < 1e-10
    u = rng.uniform(0, 1, n * n)
    E = orc.observation_matrix(pan, c, n)
    direct = 0.5 * float(np.sum((E @ u - obs.ravel()) ** 2))
    v = gpu.data_objective(G, e, n, float(obs.ravel() @ obs.ravel()), u)
    assert abs(v - direct) <= 1e-9 * max(abs(direct), 1.0)


@pytest.mark.parametrize("H,W,c,n", [(8, 8, 2, 3), (16, 16, 2, 5), (64, 64, 4, 15), (48, 64, 4, 17), (12, 12, 1, 3)])
def test_gram(gpu, orc, H, W, c, n):
    rng = np.random.default_rng(H + n)
    pan = rng.uniform(0, 1, (H, W))
    obs = rng.uniform(0, 1, (H // c, W // c))
    G, e = gpu.gram(pan, obs, c, n)
    Go, eo = orc.gram(pan, obs, c, n)
    assert rel(G, Go) < 1e-13 and rel(e, eo) < 1e-13


@pytest.mark.parametrize("nb,h,c,l,lam", [(1, 16, 2, 4, 0.0), (4, 16, 2, 4, 10.0), (4, 12, 2, 2, 10.0), (8, 32, 4, 4, 10.0)])
def test_solve_weights(gpu, orc, nb, h, c, l, lam):
    rng = np.random.default_rng(32 + nb)
    lrms = rng.uniform(0, 1, (nb, h, h))
    pan = rng.uniform(0, 1, (h * c, h * c))
    g = gpu.solve_weights(lrms, pan, gpu.SpectralWeightConfig(l=l, lambda_omega=lam, factor=c))
    assert rel(g, orc.solve_weights(lrms, pan, l, lam, c)) < 1e-10
    assert rel(gpu.combine_bands(lrms, g), orc.combine_bands(lrms, g)) < 1e-15


def test_solve_weights_singular(gpu):  # tests/test_spectral_weights.cpp:143-147
    with pytest.raises(gpu.NumericalError):
        gpu.solve_weights(np.ones((2, 8, 8)), np.full((16, 16), 2.0), gpu.SpectralWeightConfig(l=2, lambda_omega=0.0, factor=2))
