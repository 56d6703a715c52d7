"""ctypes binding of the C++ CPU oracle (``oracle/liboracle.so``) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (CPU baseline / reference arm)
may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

D = C.POINTER(C.c_double)
I = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(
            os.path.join(_HERE, "fbmp_oracle.cpp")):
        subprocess.check_call(["make", "-C", _HERE, "-s"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_matting_build.restype = C.c_void_p
        _lib.orc_matting_build.argtypes = [D, C.c_int, C.c_int, C.c_int, C.c_double]
        _lib.orc_matting_free.argtypes = [C.c_void_p]
        _lib.orc_matting_apply.argtypes = [C.c_void_p, D, D]
        _lib.orc_matting_nnz.restype = C.c_longlong
        _lib.orc_matting_nnz.argtypes = [C.c_void_p]
        _lib.orc_matting_csr.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), D]
        _lib.orc_matting_stats.argtypes = [C.c_void_p, D, D]
        _lib.orc_intensity_scale.restype = C.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(D)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(st):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def conv(img, k, adjoint=False):
    img, k = _f(img), _f(k)
    out = np.empty_like(img)
    _check(lib().orc_conv(_p(img), img.shape[0], img.shape[1], _p(k), k.shape[0], int(adjoint), _p(out)))
    return out


def fft2(img):
    img = _f(img)
    out = np.empty(img.shape, np.complex128)
    _check(lib().orc_fft2(_p(img), img.shape[0], img.shape[1], out.ctypes.data_as(D)))
    return out


def downsample(img, c):
    img = _f(img)
    out = np.empty((img.shape[0] // c, img.shape[1] // c))
    _check(lib().orc_downsample(_p(img), img.shape[0], img.shape[1], c, _p(out)))
    return out


def upsample_adjoint(img, c):
    img = _f(img)
    out = np.empty((img.shape[0] * c, img.shape[1] * c))
    _check(lib().orc_upsample_adjoint(_p(img), img.shape[0], img.shape[1], c, _p(out)))
    return out


GH, GV, LAP = 0, 1, 2


def diff(img, which, adjoint=False):
    img = _f(img)
    out = np.empty_like(img)
    _check(lib().orc_diff(_p(img), img.shape[0], img.shape[1], which, int(adjoint), _p(out)))
    return out


def laplacian(img):
    return diff(img, LAP)


def box_mean(img, r):
    img = _f(img)
    out = np.empty_like(img)
    _check(lib().orc_box_mean(_p(img), img.shape[0], img.shape[1], r, _p(out)))
    return out


def circular_box_blur(img, window):
    img = _f(img)
    out = np.empty_like(img)
    _check(lib().orc_circular_box_blur(_p(img), img.shape[0], img.shape[1], window, _p(out)))
    return out


def embed_kernel(k, h, w):
    k = _f(k)
    out = np.empty((h, w))
    _check(lib().orc_embed_kernel(_p(k), k.shape[0], h, w, _p(out)))
    return out


class Matting:
    """pansharpen.hpp:33-60 -- assembled sparse matting matrix (CSR, Eigen row order)."""

    def __init__(self, guide, radius=1, eps=1e-4):
        guide = _f(guide)
        self.shape = guide.shape
        self.h = lib().orc_matting_build(_p(guide), guide.shape[0], guide.shape[1], radius, eps)
        if not self.h:
            raise OracleError(2, lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_matting_free(self.h)
            self.h = None

    def apply(self, x):
        x = _f(x)
        y = np.empty_like(x)
        _check(lib().orc_matting_apply(self.h, _p(x), _p(y)))
        return y

    def csr(self):
        import scipy.sparse as sp
        P = self.shape[0] * self.shape[1]
        nnz = lib().orc_matting_nnz(self.h)
        rp = np.empty(P + 1, np.int64)
        col = np.empty(nnz, np.int64)
        val = np.empty(nnz)
        _check(lib().orc_matting_csr(self.h, rp.ctypes.data_as(C.POINTER(C.c_longlong)),
                                     col.ctypes.data_as(C.POINTER(C.c_longlong)), _p(val)))
        return sp.csr_matrix((val, col, rp), shape=(P, P))

    def stats(self):
        m = np.empty(self.shape)
        v = np.empty(self.shape)
        _check(lib().orc_matting_stats(self.h, _p(m), _p(v)))
        return m, v


def warmstart_cg(x, k, factor, M: Matting, lam=2e-4, cg_tol=5e-5, max_iters=2000, error_on_cap=True, prior=0):
    """pansharpen.cpp:208-264 -> (z, iters, final_residual, converged); prior 0 Laplacian, 1 identity."""
    x, k = _f(x), _f(k)
    z = np.empty(M.shape)
    it = C.c_int(0)
    fr = C.c_double(0)
    cv = C.c_int(0)
    _check(lib().orc_warmstart_cg(_p(x), x.shape[0], x.shape[1], _p(k), k.shape[0], factor, C.c_void_p(M.h),
                                  C.c_double(lam), C.c_double(cg_tol), max_iters, int(error_on_cap), _p(z),
                                  C.byref(it), C.byref(fr), C.byref(cv), int(prior)))
    return z, it.value, fr.value, bool(cv.value)


def guided_coeffs(inp, guide, radius=1, eps=1e-4):
    inp, guide = _f(inp), _f(guide)
    outs = [np.empty_like(inp) for _ in range(5)]
    _check(lib().orc_guided_coeffs(_p(inp), _p(guide), inp.shape[0], inp.shape[1], radius, C.c_double(eps),
                                   *[_p(o) for o in outs]))
    return dict(a=outs[0], c=outs[1], guide_mean=outs[2], guide_var=outs[3], input_mean=outs[4])


def guided_output(a, c, guide, radius=1):
    a, c, guide = _f(a), _f(c), _f(guide)
    out = np.empty_like(guide)
    _check(lib().orc_guided_output(_p(a), _p(c), _p(guide), guide.shape[0], guide.shape[1], radius, _p(out)))
    return out


def solve_channel_fft(x, k, factor, v, lam=2e-4, prior=0):
    x, k, v = _f(x), _f(k), _f(v)
    out = np.empty_like(v)
    _check(lib().orc_solve_channel_fft(_p(x), x.shape[0], x.shape[1], _p(k), k.shape[0], factor, _p(v),
                                       C.c_double(lam), _p(out), int(prior)))
    return out


def pansharpen(lrms, pan, k, factor, lam=2e-4, radius=1, eps=1e-4, cg_tol=5e-5, cg_max_iter=2000, threads=0, prior=0):
    lrms, pan, k = _f(lrms), _f(pan), _f(k)
    N, h, w = lrms.shape
    out = np.empty((N, h * factor, w * factor))
    it = np.zeros(N, np.int32)
    _check(lib().orc_pansharpen(_p(lrms), N, h, w, _p(pan), _p(k), k.shape[0], factor, C.c_double(lam), radius,
                                C.c_double(eps), C.c_double(cg_tol), cg_max_iter, threads, _p(out),
                                it.ctypes.data_as(I), int(prior)))
    return out, it


def solve_weights(lrms, pan, l=4, lambda_omega=10.0, factor=4):
    lrms, pan = _f(lrms), _f(pan)
    nb, h, w = lrms.shape
    om = np.empty(nb)
    _check(lib().orc_solve_weights(_p(lrms), nb, h, w, _p(pan), pan.shape[0], pan.shape[1], l,
                                   C.c_double(lambda_omega), factor, _p(om)))
    return om


def combine_bands(lrms, omega):
    lrms, omega = _f(lrms), _f(omega)
    out = np.empty(lrms.shape[1:])
    _check(lib().orc_combine_bands(_p(lrms), lrms.shape[0], lrms.shape[1], lrms.shape[2], _p(omega), _p(out)))
    return out


def shrink2(cols, t):
    cols = _f(np.stack(cols))
    _check(lib().orc_shrink2(_p(cols), cols.shape[0], C.c_longlong(cols[0].size), C.c_double(t)))
    return list(cols)


def project_simplex(v):
    v = _f(v)
    out = np.empty_like(v)
    _check(lib().orc_project_simplex(_p(v), C.c_longlong(v.size), _p(out)))
    return out


def solve_up(x, y, L1, L2, alpha1=1.0, alpha2=0.006, mu1=100.0, mu2=100.0, coupling=0.0, anchor=None):
    fields = _f(np.stack(list(x) + list(y) + list(L1) + list(L2)))
    n = fields.shape[1]
    u, p1, p2 = (np.empty((n, n)) for _ in range(3))
    anc = None if anchor is None else _f(anchor)
    _check(lib().orc_solve_up(_p(fields), n, C.c_double(alpha1), C.c_double(alpha2), C.c_double(mu1),
                              C.c_double(mu2), C.c_double(coupling), None if anc is None else _p(anc),
                              _p(u), _p(p1), _p(p2)))
    return u, p1, p2


def gram(pan, obs, factor, n):
    pan, obs = _f(pan), _f(obs)
    EtE = np.empty((n * n, n * n))
    Etf = np.empty(n * n)
    _check(lib().orc_gram(_p(pan), pan.shape[0], pan.shape[1], _p(obs), factor, n, _p(EtE), _p(Etf)))
    return EtE, Etf


def solve_z(pan, obs, factor, n, mu3, anchor):
    pan, obs, anchor = _f(pan), _f(obs), _f(anchor)
    z = np.empty(n * n)
    _check(lib().orc_solve_z(_p(pan), pan.shape[0], pan.shape[1], _p(obs), factor, n, C.c_double(mu3),
                             _p(anchor), _p(z)))
    return z


KE_DEFAULTS = dict(alpha1=1.0, alpha2=0.006, mu1=100.0, mu2=100.0, mu3=100.0, rho=0.5, t_max=10000, th=1e-5,
                   init=0)
STATE_FIELDS = ("u", "p1", "p2", "x0", "x1", "y0", "y1", "y2", "y3", "z", "L1_0", "L1_1",
                "L2_0", "L2_1", "L2_2", "L2_3", "L3")


def estimate_kernel_plane(pan, obs, factor, n, want_state=False, hook_t=-1, **kw):
    """kernel_estimator.cpp:438-455 (TGV^2) -> (kernel, iterations[, state dict])."""
    p = dict(KE_DEFAULTS)
    p.update(kw)
    pan, obs = _f(pan), _f(obs)
    k = np.empty((n, n))
    it = C.c_int(0)
    st = np.empty((17, n, n)) if (want_state or hook_t >= 0) else None
    _check(lib().orc_estimate_kernel_plane(
        _p(pan), pan.shape[0], pan.shape[1], _p(obs), factor, n, C.c_double(p["alpha1"]), C.c_double(p["alpha2"]),
        C.c_double(p["mu1"]), C.c_double(p["mu2"]), C.c_double(p["mu3"]), C.c_double(p["rho"]), int(p["t_max"]),
        C.c_double(p["th"]), int(p["init"]), _p(k), C.byref(it), None if st is None else _p(st), hook_t))
    if st is not None:
        return k, it.value, dict(zip(STATE_FIELDS, st))
    return k, it.value


def estimate_kernel_plane_tv(pan, obs, factor, n, want_state=False, **kw):
    """kernel_estimator.cpp:438-455 with KernelPrior::tv (run_tgv_or_tv(false, ...), :291-387)
    -> (kernel, iterations[, state dict]); alpha2 / mu2 are unused by the TV branch."""
    p = dict(KE_DEFAULTS)
    p.update(kw)
    pan, obs = _f(pan), _f(obs)
    k = np.empty((n, n))
    it = C.c_int(0)
    st = np.empty((17, n, n)) if want_state else None
    _check(lib().orc_estimate_kernel_plane_tv(
        _p(pan), pan.shape[0], pan.shape[1], _p(obs), factor, n, C.c_double(p["alpha1"]), C.c_double(p["mu1"]),
        C.c_double(p["mu3"]), C.c_double(p["rho"]), int(p["t_max"]), C.c_double(p["th"]), int(p["init"]), _p(k),
        C.byref(it), None if st is None else _p(st)))
    if st is not None:
        return k, it.value, dict(zip(STATE_FIELDS, st))
    return k, it.value


def tgv_objective(pan, obs, factor, n, u, p1, p2, mu3=100.0, alpha1=1.0, alpha2=0.006):
    pan, obs, u, p1, p2 = map(_f, (pan, obs, u, p1, p2))
    v = C.c_double(0)
    _check(lib().orc_tgv_objective(_p(pan), pan.shape[0], pan.shape[1], _p(obs), factor, n, C.c_double(mu3),
                                   _p(u), _p(p1), _p(p2), C.c_double(alpha1), C.c_double(alpha2), C.byref(v)))
    return v.value


def intensity_scale(pan, factor):
    pan = _f(pan)
    return lib().orc_intensity_scale(_p(pan), pan.shape[0], pan.shape[1], factor)


def blind(lrms, pan, factor, n, l=4, lambda_omega=10.0, threads=0):
    """solve_weights -> estimate_kernel_tgv -> pansharpen (all bands)."""
    lrms, pan = _f(lrms), _f(pan)
    N, h, w = lrms.shape
    out = np.empty((N, h * factor, w * factor))
    k = np.empty((n, n))
    om = np.empty(N)
    ta = C.c_int(0)
    it = np.zeros(N, np.int32)
    _check(lib().orc_blind(_p(lrms), N, h, w, _p(pan), factor, n, l, C.c_double(lambda_omega), threads, _p(out),
                           _p(k), _p(om), C.byref(ta), it.ctypes.data_as(I)))
    return out, dict(kernel=k, omega=om, admm_iters=ta.value, cg_iters=it)


def blind_sampled(lrms, pan, factor, n, cg_cap, threads=0, admm_cap=0, post_rows=0):
    """Stage-timed blind pipeline on a bounded sample: every channel's CG capped at ``cg_cap``
    iterations, the ADMM at ``admm_cap`` (0 = the reference's t_max), the alias-group solve on LR
    rows [0, post_rows) (0 = all).

    Returns dict(times=[weights, fit_setup, admm, matting_build, cg, post_fixed, post_groups]
    seconds, cg_done=[...], admm_iters). Used only by bench.py's CPU baseline / reference arm.
    """
    lrms, pan = _f(lrms), _f(pan)
    N, h, w = lrms.shape
    t = np.zeros(7)
    done = np.zeros(N, np.int32)
    ta = C.c_int(0)
    _check(lib().orc_blind_sampled(_p(lrms), N, h, w, _p(pan), factor, n, threads, cg_cap, admm_cap, post_rows, _p(t),
                                   done.ctypes.data_as(I), C.byref(ta)))
    return dict(times=list(t), cg_done=list(done), admm_iters=ta.value)


def herm_eig(A, method=0):
    """Hermitian eigen-decomposition of the oracle (0: Householder + QL, 1: Jacobi)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    n = A.shape[0]
    ev = np.empty(n)
    V = np.empty((n, n), np.complex128)
    _check(lib().orc_herm_eig(n, A.ctypes.data_as(C.POINTER(C.c_double)), method, _p(ev),
                              V.ctypes.data_as(C.POINTER(C.c_double))))
    return ev, V


def observation_matrix(pan, factor, n):
    """E of kernel_estimator.cpp:57-68 (rows = LR pixels, cols = kernel taps)."""
    pan = _f(pan)
    p = (pan.shape[0] // factor) * (pan.shape[1] // factor)
    E = np.empty((p, n * n))
    _check(lib().orc_observation_matrix(_p(pan), pan.shape[0], pan.shape[1], factor, n, _p(E)))
    return E


def estimate_kernel_l2_plane(pan, obs, factor, n, alpha1=1.0, alpha2=0.006, mu3=100.0, rho=0.5, t_max=10000,
                             th=1e-5, init="dirac"):
    """kernel_estimator.cpp:389-428 (run_l2) behind estimate_kernel_plane's scaling (:438-455): dense
    K = E^T E + 2 alpha1 grad^T grad + (2 alpha2 + mu3) I assembled column by column from the
    circular difference operators, Cholesky solves (Eigen's LLT), the oracle's simplex projection.
    Returns (kernel, iterations). Test infrastructure (checker of the device l2 estimator)."""
    s = intensity_scale(pan, factor)
    pan_n, obs_n = _f(pan) * s, _f(obs) * s
    m = n * n
    EtE, Etf = gram(pan_n, obs_n, factor, n)
    K = EtE.copy()
    for j in range(m):
        e = np.zeros((n, n))
        e.flat[j] = 1.0
        g = diff(diff(e, 0), 0, adjoint=True) + diff(diff(e, 1), 1, adjoint=True)
        K[:, j] += 2.0 * alpha1 * g.ravel()
    K[np.diag_indices(m)] += 2.0 * alpha2 + mu3
    Lc = np.linalg.cholesky(K)
    solve = lambda r: np.linalg.solve(Lc.T, np.linalg.solve(Lc, r))  # noqa: E731
    u = np.zeros(m)
    if init == "dirac":
        u[(n // 2) * n + n // 2] = 1.0
    else:
        u[:] = 1.0 / m
    z, L = u.copy(), np.zeros(m)
    t = 0
    for t in range(t_max):
        un = solve(Etf + mu3 * (z - L))
        z = project_simplex(un + L)
        L = L + rho * (un - z)
        delta = np.linalg.norm(u - un) / max(np.linalg.norm(un), 1e-300)
        u = un
        if not (np.all(np.isfinite(u)) and np.all(np.isfinite(z))):
            raise OracleError(3, f"l2 kernel estimation diverged at iteration {t}")
        if delta < th:
            break
    return z.reshape(n, n), t + 1
