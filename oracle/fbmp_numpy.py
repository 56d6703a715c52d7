"""Independent numpy/scipy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

This is the second, independent CPU oracle named in SURVEY.md §8(c): it restates the
reference algorithms with numpy FFTs, scipy.sparse and ``numpy.linalg`` so the primary
C++ oracle (``oracle/fbmp_oracle.cpp``) can be cross-checked on small sizes. Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.

Every function cites the reference file:line it follows (paths relative to
``/root/reference/proj``).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class NumericalError(RuntimeError):
    pass


# ---------------------------------------------------------------------------------------
# ops.cpp / fft_util.cpp
# ---------------------------------------------------------------------------------------

def embed_kernel(k, h, w):
    """ops.cpp:9-22 -- centre tap at (0,0), wrap the rest."""
    n = k.shape[0]
    c = (n - 1) // 2
    out = np.zeros((h, w))
    for r in range(n):
        for q in range(n):
            out[(r - c) % h, (q - c) % w] += k[r, q]
    return out


def conv(img, khat):
    """fft_util.cpp:71-76 -- forward c2c, multiply by spectrum, backward /N real part."""
    return np.real(np.fft.ifft2(np.fft.fft2(img) * khat))


def conv_adj(img, khat):
    """fft_util.cpp:78-85 -- multiply by the conjugate spectrum."""
    return np.real(np.fft.ifft2(np.fft.fft2(img) * np.conj(khat)))


def conv_direct(img, k):
    """tests/test_util.cpp:13-27 -- naive spatial circular convolution."""
    n = k.shape[0]
    C = (n - 1) // 2
    out = np.zeros_like(img)
    for a in range(-C, C + 1):
        for b in range(-C, C + 1):
            out += k[a + C, b + C] * np.roll(img, (a, b), axis=(0, 1))
    return out


def conv_adj_direct(img, k):
    n = k.shape[0]
    C = (n - 1) // 2
    out = np.zeros_like(img)
    for a in range(-C, C + 1):
        for b in range(-C, C + 1):
            out += k[a + C, b + C] * np.roll(img, (-a, -b), axis=(0, 1))
    return out


def downsample(img, c):
    """ops.cpp:36-45 -- keep (c*i, c*j)."""
    return img[::c, ::c].copy()


def upsample_adjoint(img, c):
    """ops.cpp:47-54 -- zero insertion."""
    h, w = img.shape
    out = np.zeros((h * c, w * c))
    out[::c, ::c] = img
    return out


def laplacian(img):
    """ops.cpp:70-78 -- circular 5-point stencil 4x - N - S - W - E."""
    return (4.0 * img - np.roll(img, 1, 0) - np.roll(img, -1, 0)
            - np.roll(img, 1, 1) - np.roll(img, -1, 1))


def grad_h(img):
    """ops.cpp:60-64."""
    return np.roll(img, -1, 1) - img


def grad_v(img):
    """ops.cpp:65-69."""
    return np.roll(img, -1, 0) - img


def grad_h_adj(img):
    """ops.cpp:87-92 -- g(c-1) - g(c)."""
    return np.roll(img, 1, 1) - img


def grad_v_adj(img):
    """ops.cpp:93-97."""
    return np.roll(img, 1, 0) - img


def box_mean(img, r):
    """ops.cpp:104-128 -- clamped-window mean (computed directly, not via SAT)."""
    h, w = img.shape
    if r == 0:
        return img.copy()
    cs = np.zeros((h + 1, w + 1))
    cs[1:, 1:] = np.cumsum(np.cumsum(img, 0), 1)
    rr = np.arange(h)
    cc = np.arange(w)
    r0 = np.maximum(0, rr - r)
    r1 = np.minimum(h - 1, rr + r)
    c0 = np.maximum(0, cc - r)
    c1 = np.minimum(w - 1, cc + r)
    tot = (cs[r1[:, None] + 1, c1[None, :] + 1] - cs[r0[:, None], c1[None, :] + 1]
           - cs[r1[:, None] + 1, c0[None, :]] + cs[r0[:, None], c0[None, :]])
    cnt = (r1 - r0 + 1)[:, None] * (c1 - c0 + 1)[None, :]
    return tot / cnt


def circular_box_blur(img, window):
    """ops.cpp:130-155 -- separable circular box, taps at offsets [-lead, window-1-lead]."""
    lead = (window - 1) // 2
    rows = np.zeros_like(img)
    for t in range(-lead, window - lead):
        rows += np.roll(img, t, 1)
    rows /= window
    out = np.zeros_like(img)
    for t in range(-lead, window - lead):
        out += np.roll(rows, t, 0)
    return out / window


# ---------------------------------------------------------------------------------------
# pansharpen.cpp
# ---------------------------------------------------------------------------------------

def matting_matrix(guide, radius=1, eps=1e-4):
    """pansharpen.cpp:117-195 -- interior-window matting Laplacian as CSR."""
    h, w = guide.shape
    mu = box_mean(guide, radius)
    var = box_mean(guide * guide, radius) - mu * mu
    nw = 2 * radius + 1
    ws = float(nw * nw)
    rows, cols, vals = [], [], []
    kr, kc = np.mgrid[radius:h - radius, radius:w - radius]
    kr, kc = kr.ravel(), kc.ravel()
    m_k = mu[kr, kc]
    den = eps / ws + var[kr, kc]
    offs = [(dr, dc) for dr in range(-radius, radius + 1) for dc in range(-radius, radius + 1)]
    for (ar, ac) in offs:
        mr, mc = kr + ar, kc + ac
        im = guide[mr, mc] - m_k
        for (br, bc) in offs:
            nr, nc = kr + br, kc + bc
            inn = guide[nr, nc] - m_k
            v = -(1.0 + im * inn / den) / ws
            if ar == br and ac == bc:
                v = v + 1.0
            rows.append(mr * w + mc)
            cols.append(nr * w + nc)
            vals.append(v)
    M = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(h * w, h * w)).tocsr()
    M.sum_duplicates()
    return M


def matting_apply_free(x, guide, radius=1, eps=1e-4):
    """Matrix-free form of pansharpen.cpp:155-164."""
    h, w = guide.shape
    ws = float((2 * radius + 1) ** 2)
    mu = box_mean(guide, radius)
    var = box_mean(guide * guide, radius) - mu * mu
    xb = box_mean(x, radius)
    ix = box_mean(guide * x, radius)
    a = (ix - mu * xb) / (eps / ws + var)
    b = xb - a * mu
    inter = np.zeros((h, w), bool)
    inter[radius:h - radius, radius:w - radius] = True
    a = np.where(inter, a, 0.0)
    b = np.where(inter, b, 0.0)
    ones = inter.astype(float)
    nwin = np.zeros((h, w))
    sa = np.zeros((h, w))
    sb = np.zeros((h, w))
    for dr in range(-radius, radius + 1):
        for dc in range(-radius, radius + 1):
            nwin += np.roll(ones, (dr, dc), (0, 1))
            sa += np.roll(a, (dr, dc), (0, 1))
            sb += np.roll(b, (dr, dc), (0, 1))
    return nwin * x - guide * sa - sb


def warmstart_cg(x, khat, factor, Mop, lam, cg_tol, max_iters, error_on_cap=True,
                 dot=None, conv_f=None, conv_a=None):
    """pansharpen.cpp:208-264. Returns (z, iterations, converged)."""
    if dot is None:
        dot = lambda a, b: float(np.dot(a.ravel(), b.ravel()))
    cf = conv_f or (lambda z: conv(z, khat))
    ca = conv_a or (lambda z: conv_adj(z, khat))

    def A(z):
        d = ca(upsample_adjoint(downsample(cf(z), factor), factor))
        return d + laplacian(Mop(laplacian(z))) * lam

    rhs = ca(upsample_adjoint(x, factor))
    rhs_norm = np.sqrt(dot(rhs, rhs))
    z = np.zeros_like(rhs)
    if rhs_norm == 0.0:
        return z, 0, True
    r = rhs.copy()
    p = r.copy()
    rs = dot(r, r)
    conv_ok = False
    it = 0
    for it in range(max_iters):
        Ap = A(p)
        pAp = dot(p, Ap)
        if not pAp > 0:
            if np.sqrt(rs) <= 1e-12 * rhs_norm:
                conv_ok = True
                break
            raise NumericalError("warmstart: conjugate gradients hit a non-positive curvature direction")
        alpha = rs / pAp
        z = z + p * alpha
        r = r - Ap * alpha
        step = abs(alpha) * np.sqrt(dot(p, p))
        rs_new = dot(r, r)
        if step <= cg_tol * max(np.sqrt(dot(z, z)), 1e-300):
            conv_ok = True
            break
        p = r + p * (rs_new / rs)
        rs = rs_new
    iters = it + 1
    if not conv_ok and error_on_cap:
        raise NumericalError(f"warmstart: conjugate gradients did not converge in {max_iters} iterations")
    return z, iters, conv_ok


def guided_coeffs(inp, guide, radius, eps):
    """pansharpen.cpp:274-302."""
    mu = box_mean(guide, radius)
    im = box_mean(inp, radius)
    cgi = box_mean(guide * inp, radius)
    cgg = box_mean(guide * guide, radius)
    var = cgg - mu * mu
    cov = cgi - mu * im
    a = cov / (var + eps)
    c = im - a * mu
    return a, c


def guided_output(a, c, guide, radius):
    """pansharpen.cpp:304-312."""
    return box_mean(a, radius) * guide + box_mean(c, radius)


def lap_spectrum(H, W):
    """pansharpen.cpp:56-63."""
    cv = np.cos(2 * np.pi * np.arange(H) / H)[:, None]
    ch = np.cos(2 * np.pi * np.arange(W) / W)[None, :]
    return (4.0 - 2.0 * cv - 2.0 * ch).astype(complex)


def solve_channel_fft(x, k, factor, v, lam):
    """pansharpen.cpp:314-365 -- per alias group (c^2 x c^2) Hermitian solve via eigh."""
    H, W = v.shape
    h, w = x.shape
    c2 = factor * factor
    bhat = np.fft.fft2(embed_kernel(k, H, W))
    lhat = lap_spectrum(H, W)
    xhat = np.fft.fft2(x)
    vhat = np.fft.fft2(v)
    # group g = a*factor + b at index (kl + a*h, ll + b*w)
    B = bhat.reshape(factor, h, factor, w).transpose(1, 3, 0, 2).reshape(h, w, c2)
    Lh = lhat.reshape(factor, h, factor, w).transpose(1, 3, 0, 2).reshape(h, w, c2)
    V = vhat.reshape(factor, h, factor, w).transpose(1, 3, 0, 2).reshape(h, w, c2)
    A = np.conj(B)[..., :, None] * B[..., None, :] / c2
    idx = np.arange(c2)
    A[..., idx, idx] += lam * np.abs(Lh) ** 2
    rhs = np.conj(B) * xhat[..., None] + lam * np.conj(Lh) * V
    ev, vec = np.linalg.eigh(A)
    if not (np.all(ev[..., 0] > 0) and np.all(ev[..., -1] <= 1e14 * ev[..., 0])):
        raise NumericalError("solve_channel_fft: alias-group system condition number exceeds 1e14 "
                             "(prior transfer function too small)")
    sol = np.einsum("...ij,...j->...i", vec,
                    np.einsum("...ji,...j->...i", np.conj(vec), rhs) / ev)
    Z = sol.reshape(h, w, factor, factor).transpose(2, 0, 3, 1).reshape(H, W)
    return np.real(np.fft.ifft2(Z))


def pansharpen(lrms, pan, k, factor, lam=2e-4, radius=1, eps=1e-4, cg_tol=5e-5,
               cg_max_iter=2000, matrix_free=False, direct_conv=False, return_info=False):
    """pansharpen.cpp:367-424 (channels sequential here)."""
    peak = max(pan.max(), max(b.max() for b in lrms))
    scale = 1.0 / peak if peak > 0 else 1.0
    pan_n = pan * scale
    lpan = laplacian(pan_n)
    H, W = pan.shape
    if matrix_free:
        Mop = lambda z: matting_apply_free(z, lpan, radius, eps)
    else:
        M = matting_matrix(lpan, radius, eps)
        Mop = lambda z: (M @ z.ravel()).reshape(z.shape)
    khat = np.fft.fft2(embed_kernel(k, H, W))
    out, iters, z0s = [], [], []
    for b in lrms:
        xn = b * scale
        kw = {}
        if direct_conv:
            kw = dict(conv_f=lambda z: conv_direct(z, k), conv_a=lambda z: conv_adj_direct(z, k))
        z0, it, _ = warmstart_cg(xn, khat, factor, Mop, lam, cg_tol, cg_max_iter, **kw)
        a, c = guided_coeffs(laplacian(z0), lpan, radius, eps)
        v = guided_output(a, c, lpan, radius)
        z = solve_channel_fft(xn, k, factor, v, lam)
        out.append(z / scale)
        iters.append(it)
        z0s.append(z0 / scale)
    out = np.stack(out)
    if return_info:
        return out, dict(cg_iters=iters, z0=np.stack(z0s))
    return out


# ---------------------------------------------------------------------------------------
# spectral_weights.cpp
# ---------------------------------------------------------------------------------------

def solve_weights(lrms, pan, l=4, lambda_omega=10.0, factor=4):
    """spectral_weights.cpp:9-53."""
    nb = lrms.shape[0]
    A = np.stack([circular_box_blur(b, l + 1).ravel() for b in lrms], 1)
    b = downsample(circular_box_blur(pan, factor * l + 1), factor).ravel()
    normal = A.T @ A
    if nb > 1:
        G = np.zeros((nb - 1, nb))
        for i in range(nb - 1):
            G[i, i] = -1.0
            G[i, i + 1] = 1.0
        normal = normal + lambda_omega * (G.T @ G)
    rhs = A.T @ b
    if np.linalg.matrix_rank(normal) < nb:
        raise NumericalError("solve_weights: normal matrix is singular")
    omega = np.linalg.solve(normal, rhs)
    return omega


def combine_bands(lrms, omega):
    """spectral_weights.cpp:55-65."""
    out = np.zeros(lrms.shape[1:])
    for i in range(lrms.shape[0]):
        out += omega[i] * lrms[i]
    return out


# ---------------------------------------------------------------------------------------
# kernel_estimator.cpp (TGV^2 path)
# ---------------------------------------------------------------------------------------

def intensity_scale(pan, factor):
    """kernel_estimator.cpp:283-289."""
    m = np.abs(pan).max()
    if m <= 0:
        raise NumericalError("kernel estimation: PAN image is identically zero")
    hw = float(pan.shape[0] // factor) * (pan.shape[1] // factor)
    return np.sqrt(16384.0 / hw) / m


def observation_matrix(pan, factor, n):
    """kernel_estimator.cpp:57-68 -- E[(i,j),(tr,tc)] = pan[c*i-(tr-C), c*j-(tc-C)] (wrap)."""
    H, W = pan.shape
    h, w = H // factor, W // factor
    C = (n - 1) // 2
    ii = np.arange(h)[:, None, None, None]
    jj = np.arange(w)[None, :, None, None]
    tr = np.arange(n)[None, None, :, None]
    tc = np.arange(n)[None, None, None, :]
    rr = (factor * ii - (tr - C)) % H
    cc = (factor * jj - (tc - C)) % W
    return pan[rr, cc].reshape(h * w, n * n)


def shrink2(cols, t):
    """kernel_estimator.cpp:94-110."""
    nrm = np.sqrt(sum(c * c for c in cols))
    scale = np.where(nrm > t, (nrm - t) / np.where(nrm > 0, nrm, 1.0), 0.0)
    return [c * scale for c in cols]


def project_simplex(v):
    """kernel_estimator.cpp:112-128 -- tau from the LAST qualifying j."""
    u = np.sort(v)[::-1]
    css = np.cumsum(u)
    j = np.arange(1, len(u) + 1)
    cand = (1.0 - css) / j
    ok = np.nonzero(u + cand > 0)[0]
    if len(ok) == 0:
        raise NumericalError("project_simplex: empty support (non-finite input?)")
    tau = cand[ok[-1]]
    return np.maximum(v + tau, 0.0)


def _up_symbols(n, a1m1, a2m2, coupling):
    """kernel_estimator.cpp:174-195."""
    wv = 2 * np.pi * np.arange(n) / n
    dv = (np.cos(wv) + 1j * np.sin(wv) - 1.0)[:, None] * np.ones((1, n))
    dh = (np.cos(wv) + 1j * np.sin(wv) - 1.0)[None, :] * np.ones((n, 1))
    av2, ah2 = np.abs(dv) ** 2, np.abs(dh) ** 2
    d1 = a1m1 * (ah2 + av2) + coupling
    d2 = a1m1 + 0.5 * a2m2 * av2 + a2m2 * ah2
    d3 = a1m1 + 0.5 * a2m2 * ah2 + a2m2 * av2
    d4 = -a1m1 * dh
    d5 = -a1m1 * dv
    d6 = 0.5 * a2m2 * np.conj(dh) * dv
    return d1, d2, d3, d4, d5, d6


def solve_up_core(x, y, L1, L2, prm, coupling, anchor):
    """kernel_estimator.cpp:137-233 (Cramer branch; coupling > 0 so DC is regular)."""
    a1m1 = prm["alpha1"] * prm["mu1"]
    a2m2 = prm["alpha2"] * prm["mu2"]
    x1 = x[0] - L1[0]
    x2 = x[1] - L1[1]
    y1 = y[0] - L2[0]
    y2 = y[3] - L2[3]
    yc = (y[1] - L2[1] + y[2] - L2[2]) * 0.5
    B1 = (grad_h_adj(x1) + grad_v_adj(x2)) * a1m1
    B2 = x1 * -a1m1 + (grad_h_adj(y1) + grad_v_adj(yc)) * a2m2
    B3 = x2 * -a1m1 + (grad_v_adj(y2) + grad_h_adj(yc)) * a2m2
    if coupling > 0 and anchor is not None:
        B1 = B1 + anchor * coupling
    n = x1.shape[0]
    d1, d2, d3, d4, d5, d6 = _up_symbols(n, a1m1, a2m2, coupling)
    b1, b2, b3 = np.fft.fft2(B1), np.fft.fft2(B2), np.fft.fft2(B3)
    c = np.conj
    den = d1 * (d2 * d3 - np.abs(d6) ** 2) - c(d4) * (d4 * d3 - c(d6) * d5) + c(d5) * (d4 * d6 - d2 * d5)
    nu = b1 * (d2 * d3 - np.abs(d6) ** 2) - c(d4) * (b2 * d3 - c(d6) * b3) + c(d5) * (b2 * d6 - d2 * b3)
    np1 = d1 * (b2 * d3 - c(d6) * b3) - b1 * (d4 * d3 - c(d6) * d5) + c(d5) * (d4 * b3 - b2 * d5)
    np2 = d1 * (d2 * b3 - d6 * b2) - c(d4) * (d4 * b3 - b2 * d5) + b1 * (d4 * d6 - d2 * d5)
    tol = 1e-12 * np.abs(den).max()
    if np.any(np.abs(den) <= tol):
        raise NumericalError("singular {u,p} symbol (coupling must be > 0 in this restatement)")
    U = np.real(np.fft.ifft2(nu / den))
    P1 = np.real(np.fft.ifft2(np1 / den))
    P2 = np.real(np.fft.ifft2(np2 / den))
    return U, P1, P2


def estimate_kernel_tgv(pan, obs, factor, n, alpha1=1.0, alpha2=0.006, mu1=100.0, mu2=100.0,
                        mu3=100.0, rho=0.5, t_max=10000, th=1e-5):
    """kernel_estimator.cpp:291-387 + 438-455 (TGV^2 branch). Returns (kernel, iterations)."""
    mean = pan.mean()
    if np.abs(pan - mean).max() <= 1e-12 * max(1.0, abs(mean)):
        raise NumericalError("kernel estimation: constant PAN image is unidentifiable (E^T E has rank 1)")
    s = intensity_scale(pan, factor)
    pan_n = pan * s
    obs_n = obs * s
    E = observation_matrix(pan_n, factor, n)
    f = obs_n.ravel()
    Etf = E.T @ f
    EtE = E.T @ E
    reg = EtE + mu3 * np.eye(n * n)
    Lc = np.linalg.cholesky(reg)
    solve_z = lambda anc: np.linalg.solve(Lc.T, np.linalg.solve(Lc, Etf + mu3 * anc))
    prm = dict(alpha1=alpha1, alpha2=alpha2, mu1=mu1, mu2=mu2)
    u = np.zeros((n, n))
    u[(n - 1) // 2, (n - 1) // 2] = 1.0
    z = u.copy()
    p1 = np.zeros((n, n))
    p2 = np.zeros((n, n))
    x = [grad_h(u), grad_v(u)]
    y = [np.zeros((n, n)) for _ in range(4)]
    L1 = [np.zeros((n, n)) for _ in range(2)]
    L2 = [np.zeros((n, n)) for _ in range(4)]
    L3 = np.zeros((n, n))
    iters = 0
    for t in range(t_max):
        gx = [grad_h(u) - p1 + L1[0], grad_v(u) - p2 + L1[1]]
        x = shrink2(gx, 1.0 / mu1)
        cross = (grad_v(p1) + grad_h(p2)) * 0.5
        ep = [grad_h(p1), cross, cross, grad_v(p2)]
        y = shrink2([ep[j] + L2[j] for j in range(4)], 1.0 / mu2)
        z = project_simplex(solve_z((u + L3).ravel())).reshape(n, n)
        anchor = z - L3
        u_new, p1, p2 = solve_up_core(x, y, L1, L2, prm, mu3, anchor)
        L1[0] = L1[0] + (grad_h(u_new) - p1 - x[0]) * rho
        L1[1] = L1[1] + (grad_v(u_new) - p2 - x[1]) * rho
        cross = (grad_v(p1) + grad_h(p2)) * 0.5
        ep = [grad_h(p1), cross, cross, grad_v(p2)]
        for j in range(4):
            L2[j] = L2[j] + (ep[j] - y[j]) * rho
        L3 = L3 + (u_new - z) * rho
        delta = np.linalg.norm(u - u_new)
        scale = max(np.linalg.norm(u_new), 1e-300)
        u = u_new
        iters = t + 1
        if not (np.all(np.isfinite(u)) and np.all(np.isfinite(z))):
            raise NumericalError(f"kernel estimation diverged: non-finite at iteration {t}")
        if delta / scale < th:
            break
    return z, iters


def blind(lrms, pan, factor, n, l=4, lambda_omega=10.0, **kw):
    """SPEC.md:584-591 composition: solve_weights -> estimate_kernel_tgv -> pansharpen."""
    omega = solve_weights(lrms, pan, l, lambda_omega, factor)
    obs = combine_bands(lrms, omega)
    k, t = estimate_kernel_tgv(pan, obs, factor, n)
    out, info = pansharpen(lrms, pan, k, factor, return_info=True, **kw)
    info.update(omega=omega, kernel=k, admm_iters=t)
    return out, info


# ---------------------------------------------------------------------------------------------
# Evaluation metrics (proj/src/metrics.cpp:14-153) -- the checker of the device metrics.
# Sums are sequential (math.fsum-free Python loops would be slow; numpy's pairwise sums differ
# from the reference's sequential ones only by rounding).
# ---------------------------------------------------------------------------------------------
def crop_border(img, margin):  # metrics.cpp:46-58
    if margin < 0:
        raise ValueError("crop_border: negative margin")
    if margin == 0:
        return img
    if 2 * margin >= min(img.shape[-2:]):
        raise ValueError("crop_border: margin leaves no pixels")
    return img[..., margin:-margin, margin:-margin]


def _psnr_from_mse(mse):  # metrics.cpp:24-27
    return np.inf if mse <= 0.0 else 20.0 * np.log10(255.0 / np.sqrt(mse))


def psnr_avg(est, ref):  # metrics.cpp:66-79
    per = [_psnr_from_mse(np.mean((e - r) ** 2)) for e, r in zip(est, ref)]
    return per, sum(per) / len(per)


def psnr_reg_avg(est, ref):  # metrics.cpp:81-105
    s = 0.0
    for e, r in zip(est, ref):
        me, mr = e.mean(), r.mean()
        var = np.sum((e - me) * (e - me))
        cov = np.sum((e - me) * (r - mr))
        a, b = (cov / var, mr - cov / var * me) if var > 0.0 else (0.0, mr)
        s += _psnr_from_mse(np.mean((a * e + b - r) ** 2))
    return s / len(est)


def ergas(est, ref, factor):  # metrics.cpp:107-118
    acc = 0.0
    for e, r in zip(est, ref):
        mu = r.mean()
        if mu == 0.0:
            raise ValueError("ergas: reference band mean is zero")
        rmse = np.sqrt(np.mean((e - r) ** 2))
        acc += (rmse / mu) ** 2
    return 100.0 / factor * np.sqrt(acc / len(est))


def sam_deg(est, ref):  # metrics.cpp:120-141
    dot = np.sum(est * ref, axis=0)
    ne = np.sum(est * est, axis=0)
    nr = np.sum(ref * ref, axis=0)
    ok = (ne != 0.0) & (nr != 0.0)
    if not ok.any():
        return 0.0
    cosv = np.clip(dot[ok] / np.sqrt(ne[ok] * nr[ok]), -1.0, 1.0)
    return float(np.sum(np.arccos(cosv)) / ok.sum() * 180.0 / np.pi)


def rase(est, ref):  # metrics.cpp:143-153
    mu = np.mean([r.mean() for r in ref])
    if mu == 0.0:
        raise ValueError("rase: mean of reference image is zero")
    return 100.0 / mu * np.sqrt(np.mean([np.mean((e - r) ** 2) for e, r in zip(est, ref)]))
