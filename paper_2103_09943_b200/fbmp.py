"""Python binding of the B200 C ABI (``include/fbmp_gpu.h``) with the reference's ``fbmp::`` names.

The functions below mirror the reference C++ API (``/root/reference/proj/include/fbmp/*.hpp``):
same names, same argument meaning, same exception taxonomy (``ParamError``,
``DimensionError``, ``NumericalError``; errors.hpp:8-33) and messages. Every call runs on the
GPU through ``lib/libfbmp_gpu.so``; there is no CPU path. If the library has not been built,
importing this module raises ``ImportError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FBMP_GPU_LIB") or os.path.join(_HERE, "lib", "libfbmp_gpu.so")  # env: A/B experiments
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2103_09943_b200.build` (or "
                      "__graft_entry__.build()) first; there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

D = C.POINTER(C.c_double)
I = C.POINTER(C.c_int)


class FbmpError(RuntimeError):
    """errors.hpp:11-13 (fbmp::Error)."""


class DimensionError(FbmpError):
    pass


class ParamError(FbmpError):
    pass


class NumericalError(FbmpError):
    pass


class DeviceError(FbmpError):
    """CUDA / cuFFT runtime failure (status 4)."""


_ERR = {1: ParamError, 2: DimensionError, 3: NumericalError, 4: DeviceError}


class _PsParams(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("radius", C.c_int), ("eps", C.c_double), ("cg_tol", C.c_double),
                ("cg_max_iter", C.c_int), ("threads", C.c_int), ("prior", C.c_int)]


class _KeParams(C.Structure):
    _fields_ = [("n", C.c_int), ("alpha1", C.c_double), ("alpha2", C.c_double), ("mu1", C.c_double),
                ("mu2", C.c_double), ("mu3", C.c_double), ("rho", C.c_double), ("t_max", C.c_int),
                ("th", C.c_double), ("init", C.c_int)]


class _SwParams(C.Structure):
    _fields_ = [("l", C.c_int), ("lambda_omega", C.c_double), ("factor", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("admm_iters", C.c_int), ("cg_iters", C.c_int * 64), ("ms_weights", C.c_double),
                ("ms_kernel_fit", C.c_double), ("ms_pansharpen", C.c_double), ("cg_channel_iters", C.c_longlong),
                ("n_channels", C.c_int)]


@dataclass
class PansharpenParams:
    """pansharpen.hpp:15-26; prior: "laplacian" (default) or "identity" (PriorKind, :11)."""
    lambda_: float = 2e-4
    radius: int = 1
    eps: float = 1e-4
    cg_tol: float = 5e-5
    cg_max_iter: int = 2000
    threads: int = 0
    prior: str = "laplacian"

    def c(self):
        kinds = {"laplacian": 0, "identity": 1, "custom": 2}
        if self.prior not in kinds:
            raise ParamError("pansharpen: unknown prior kind")
        return _PsParams(self.lambda_, self.radius, self.eps, self.cg_tol, self.cg_max_iter, self.threads,
                         kinds[self.prior])


@dataclass
class KernelEstParams:
    """kernel_estimator.hpp:16-31. init: 'dirac' or 'uniform'."""
    n: int = 29
    alpha1: float = 1.0
    alpha2: float = 0.006
    mu1: float = 100.0
    mu2: float = 100.0
    mu3: float = 100.0
    rho: float = 0.5
    t_max: int = 10000
    th: float = 1e-5
    init: str = "dirac"

    def c(self):
        return _KeParams(self.n, self.alpha1, self.alpha2, self.mu1, self.mu2, self.mu3, self.rho, self.t_max,
                         self.th, 0 if self.init == "dirac" else 1)


@dataclass
class SpectralWeightConfig:
    """spectral_weights.hpp:9-14 (band_indices are applied by slicing the input)."""
    l: int = 4
    lambda_omega: float = 10.0
    factor: int = 2

    def c(self):
        return _SwParams(self.l, self.lambda_omega, self.factor)


STATE_FIELDS = ("u", "p1", "p2", "x0", "x1", "y0", "y1", "y2", "y3", "z", "L1_0", "L1_1",
                "L2_0", "L2_1", "L2_2", "L2_3", "L3")

_lib.fbmp_gpu_last_error.restype = C.c_char_p
_lib.fbmp_gpu_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
_lib.fbmp_gpu_ctx_destroy.argtypes = [C.c_void_p]
_lib.fbmp_gpu_ctx_stream.restype = C.c_void_p
_lib.fbmp_gpu_ctx_stream.argtypes = [C.c_void_p]
_lib.fbmp_gpu_ctx_launches.restype = C.c_longlong
_lib.fbmp_gpu_ctx_launches.argtypes = [C.c_void_p]
_lib.fbmp_gpu_ctx_stats.argtypes = [C.c_void_p, C.POINTER(_Stats)]
_lib.fbmp_gpu_ctx_set_profile.argtypes = [C.c_void_p, C.c_int]
_lib.fbmp_gpu_ctx_cg_iters.restype = C.c_int
_lib.fbmp_gpu_ctx_cg_iters.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int]


def _check(status: int) -> None:
    if status != 0:
        raise _ERR.get(status, FbmpError)(_lib.fbmp_gpu_last_error().decode())


class Context:
    """One device context (workspace, cuFFT plans, stream) per host thread and device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_lib.fbmp_gpu_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            _lib.fbmp_gpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return _lib.fbmp_gpu_ctx_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return _lib.fbmp_gpu_ctx_launches(self.h)

    def set_profile(self, on: bool) -> None:
        _lib.fbmp_gpu_ctx_set_profile(self.h, int(on))

    def set_precision(self, bits: int) -> None:
        """64 (default, reference fp64) or 32 (fp32 mode of the HRMS CG: fp32 vectors and stencils,
        fp64 reductions and CG scalars; gate <= 1e-3 rel. L2 and <= 0.05 dB PSNR vs fp64)."""
        _check(_lib.fbmp_gpu_ctx_set_precision(self.h, int(bits)))

    @property
    def precision(self) -> int:
        return int(_lib.fbmp_gpu_ctx_precision(self.h))

    def set_comm(self, uid: bytes, nranks: int, rank: int) -> None:
        """Attach an NCCL communicator (row-strip solves); every rank calls this with the same id."""
        buf = (C.c_ubyte * 128).from_buffer_copy(bytes(uid).ljust(128, b"\0")[:128])
        _check(_lib.fbmp_gpu_ctx_set_comm(self.h, buf, nranks, rank))

    def kernel_profile(self) -> dict:
        ms = (C.c_double * 4)()
        n = (C.c_longlong * 4)()
        _check(_lib.fbmp_gpu_ctx_kernel_profile(self.h, ms, n))
        return {name: dict(total_ms=ms[i], launches=n[i]) for i, name in enumerate(("K_Q", "K_D", "K_L", "K_U"))}

    def stats(self) -> dict:
        s = _Stats()
        _check(_lib.fbmp_gpu_ctx_stats(self.h, C.byref(s)))
        n = _lib.fbmp_gpu_ctx_cg_iters(self.h, None, 0)
        if n < 0:
            raise FbmpError(_lib.fbmp_gpu_last_error().decode())
        its = (C.c_int * max(n, 1))()
        _lib.fbmp_gpu_ctx_cg_iters(self.h, its, n)
        return dict(admm_iters=s.admm_iters, cg_iters=list(its)[:n], ms_weights=s.ms_weights,
                    ms_kernel_fit=s.ms_kernel_fit, ms_pansharpen=s.ms_pansharpen,
                    cg_channel_iters=s.cg_channel_iters)


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _f(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(D) if a is not None else None


def _ctx(ctx):
    return (ctx or default_context()).h


# ---------------------------------------------------------------------------------------------
# pansharpen.hpp
# ---------------------------------------------------------------------------------------------

def pansharpen(lrms, pan, k, factor, params: PansharpenParams | None = None, ctx=None, return_iters=False):
    """pansharpen.hpp:95-96 -> HRMS (N, H, W)."""
    lrms, pan, k = _f(lrms), _f(pan), _f(k)
    N, h, w = lrms.shape
    if pan.shape != (h * factor, w * factor):
        raise DimensionError("pansharpen: PAN dimensions must be factor times the LRMS dimensions")
    prm = (params or PansharpenParams()).c()
    out = np.empty((N, h * factor, w * factor))
    it = np.zeros(N, np.int32)
    _check(_lib.fbmp_gpu_pansharpen(_ctx(ctx), _p(lrms), N, h, w, _p(pan), _p(k), k.shape[0], factor, C.byref(prm),
                                    _p(out), it.ctypes.data_as(I)))
    return (out, it) if return_iters else out


def apply_prior(img, params=None, ctx=None):
    """pansharpen.hpp:28 (Laplacian prior)."""
    img = _f(img)
    out = np.empty_like(img)
    _check(_lib.fbmp_gpu_apply_prior(_ctx(ctx), _p(img), img.shape[0], img.shape[1], _p(out)))
    return out


apply_prior_adjoint = apply_prior  # the 5-point stencil is symmetric (ops.cpp:98-99)


class MattingMatrix:
    """pansharpen.hpp:33-60, matrix-free: built on a guide, applied on the device."""

    def __init__(self, guide, radius=1, eps=1e-4, ctx=None):
        if radius < 1:
            raise ParamError("matting matrix: radius must be >= 1")
        self.guide = _f(guide)
        if 2 * radius + 1 > min(self.guide.shape):
            raise DimensionError("matting matrix: window larger than image")
        self.radius, self.eps, self.ctx = radius, eps, ctx

    @classmethod
    def build(cls, guide, radius, eps, ctx=None):
        return cls(guide, radius, eps, ctx)

    @property
    def height(self):
        return self.guide.shape[0]

    @property
    def width(self):
        return self.guide.shape[1]

    def apply(self, x):
        x = _f(x)
        if x.shape != self.guide.shape:
            raise DimensionError("matting matrix: plane shape mismatch")
        y = np.empty_like(x)
        _check(_lib.fbmp_gpu_llp_apply(_ctx(self.ctx), _p(self.guide), _p(x), x.shape[0], x.shape[1], self.radius,
                                       C.c_double(self.eps), _p(y)))
        return y


def build_matting_matrix(guide, radius, eps, ctx=None):
    return MattingMatrix(guide, radius, eps, ctx)


def data_apply(p, k, factor, ctx=None):
    """B^T U D B p (the data term of pansharpen.cpp:219-220)."""
    p, k = _f(p), _f(k)
    out = np.empty_like(p)
    _check(_lib.fbmp_gpu_data_apply(_ctx(ctx), _p(p), p.shape[0], p.shape[1], _p(k), k.shape[0], factor, _p(out)))
    return out


def cg_operator(guide, p, k, factor, params=None, ctx=None):
    """A(p) of pansharpen.cpp:218-223 with M built on ``guide``."""
    guide, p, k = _f(guide), _f(p), _f(k)
    prm = (params or PansharpenParams()).c()
    out = np.empty_like(p)
    _check(_lib.fbmp_gpu_cg_operator(_ctx(ctx), _p(guide), _p(p), p.shape[0], p.shape[1], _p(k), k.shape[0], factor,
                                     C.byref(prm), _p(out)))
    return out


def warmstart_cg(x, k, factor, M: MattingMatrix, params=None, max_iters=None, error_on_cap=True, ctx=None):
    """pansharpen.hpp:73-75 -> (z, iterations, final_residual)."""
    x, k = _f(x), _f(k)
    prm = params or PansharpenParams()
    if max_iters is None:
        max_iters = prm.cg_max_iter
    h, w = x.shape
    if h * factor != M.height or w * factor != M.width:
        raise DimensionError("warmstart: LR channel dimensions must be image/factor")
    z = np.empty((M.height, M.width))
    it = C.c_int(0)
    res = C.c_double(0)
    cp = prm.c()
    cp.radius, cp.eps = M.radius, M.eps
    _check(_lib.fbmp_gpu_warmstart_cg(_ctx(ctx or M.ctx), _p(x), h, w, _p(M.guide), _p(k), k.shape[0], factor,
                                      C.byref(cp), int(max_iters), int(error_on_cap), _p(z), C.byref(it),
                                      C.byref(res)))
    return z, it.value, res.value


def warmstart_channel(x, pan, k, factor, M: MattingMatrix, params=None, ctx=None):
    """pansharpen.hpp:68-69."""
    prm = params or PansharpenParams()
    _validate_ps(prm)
    if _f(pan).shape != (M.height, M.width):
        raise DimensionError("warmstart: matting matrix was not built on the PAN grid")
    return warmstart_cg(x, k, factor, M, prm, prm.cg_max_iter, True, ctx)[0]


def _validate_ps(p: PansharpenParams):
    """pansharpen.cpp:96-105."""
    if not p.lambda_ > 0:
        raise ParamError("pansharpen: lambda must be positive")
    if p.radius < 1:
        raise ParamError("pansharpen: radius must be >= 1")
    if not p.eps > 0:
        raise ParamError("pansharpen: eps must be positive")
    if not p.cg_tol > 0:
        raise ParamError("pansharpen: cg_tol must be positive")
    if p.cg_max_iter < 1:
        raise ParamError("pansharpen: cg_max_iter must be >= 1")
    if p.threads < 0:
        raise ParamError("pansharpen: threads must be >= 0")


def guided_coeffs(inp, guide, radius, eps, ctx=None):
    """pansharpen.hpp:83 -> dict(a, c)."""
    inp, guide = _f(inp), _f(guide)
    if inp.shape != guide.shape:
        raise DimensionError("guided_coeffs: shape mismatch")
    a, c, v = (np.empty_like(inp) for _ in range(3))
    _check(_lib.fbmp_gpu_guided_filter(_ctx(ctx), _p(inp), _p(guide), inp.shape[0], inp.shape[1], radius,
                                       C.c_double(eps), _p(a), _p(c), _p(v)))
    return dict(a=a, c=c)


def guided_output(coeffs, guide, radius, ctx=None):
    """pansharpen.hpp:84."""
    a, c, guide = _f(coeffs["a"]), _f(coeffs["c"]), _f(guide)
    if a.shape != guide.shape:
        raise DimensionError("guided_output: shape mismatch")
    out = np.empty_like(guide)
    _check(_lib.fbmp_gpu_guided_output(_ctx(ctx), _p(a), _p(c), _p(guide), guide.shape[0], guide.shape[1], radius,
                                       _p(out)))
    return out


def guided_filter(inp, guide, radius, eps, ctx=None):
    """guided_output(guided_coeffs(...)) fused in one kernel."""
    inp, guide = _f(inp), _f(guide)
    v = np.empty_like(inp)
    _check(_lib.fbmp_gpu_guided_filter(_ctx(ctx), _p(inp), _p(guide), inp.shape[0], inp.shape[1], radius,
                                       C.c_double(eps), None, None, _p(v)))
    return v


def solve_channel_fft(x, k, factor, v, params=None, ctx=None):
    """pansharpen.hpp:90-91."""
    x, k, v = _f(x), _f(k), _f(v)
    h, w = x.shape
    if v.shape != (h * factor, w * factor):
        raise DimensionError("solve_channel_fft: LR/HR dimensions inconsistent with factor")
    prm = (params or PansharpenParams()).c()
    out = np.empty_like(v)
    _check(_lib.fbmp_gpu_solve_channel_fft(_ctx(ctx), _p(x), h, w, _p(k), k.shape[0], factor, _p(v), C.byref(prm),
                                           _p(out)))
    return out


# ---------------------------------------------------------------------------------------------
# ops.hpp
# ---------------------------------------------------------------------------------------------

def box_mean(img, radius, ctx=None):
    img = _f(img)
    out = np.empty_like(img)
    _check(_lib.fbmp_gpu_box_mean(_ctx(ctx), _p(img), img.shape[0], img.shape[1], radius, _p(out)))
    return out


METRIC_PSNR, METRIC_PSNR_REG, METRIC_ERGAS, METRIC_SAM, METRIC_RASE = 1, 2, 4, 8, 16


def metrics(est, ref, factor=4, crop=0, which=31, ctx=None):
    """Evaluation metrics of metrics.hpp:11-51 on the device (inputs on the [0, 255] scale),
    after crop_border(crop) of both cubes: dict with psnr_per_band, psnr_avg, psnr_reg_avg,
    ergas, sam_deg, rase (None where `which` does not select it)."""
    est, ref = _f(est), _f(ref)
    if est.ndim == 2:
        est, ref = est[None], ref[None]
    if est.shape != ref.shape or est.ndim != 3:
        raise DimensionError("metrics: image shapes differ")
    N, H, W = est.shape
    pb, out = np.empty(N), np.empty(5)
    _check(_lib.fbmp_gpu_metrics(_ctx(ctx), _p(est), _p(ref), N, H, W, crop, factor, which, _p(pb), _p(out)))
    keys = ("psnr_avg", "psnr_reg_avg", "ergas", "sam_deg", "rase")
    res = {k: (float(out[i]) if which & (1 << i) else None) for i, k in enumerate(keys)}
    res["psnr_per_band"] = list(pb) if which & METRIC_PSNR else None
    return res


def psnr_avg(est, ref, ctx=None):  # metrics.hpp:31-33
    m = metrics(est, ref, which=METRIC_PSNR, ctx=ctx)
    return m["psnr_per_band"], m["psnr_avg"]


def psnr_reg_avg(est, ref, ctx=None):  # metrics.hpp:36-38
    return metrics(est, ref, which=METRIC_PSNR_REG, ctx=ctx)["psnr_reg_avg"]


def ergas(est, ref, factor, ctx=None):  # metrics.hpp:40
    return metrics(est, ref, factor=factor, which=METRIC_ERGAS, ctx=ctx)["ergas"]


def sam_deg(est, ref, ctx=None):  # metrics.hpp:41
    return metrics(est, ref, which=METRIC_SAM, ctx=ctx)["sam_deg"]


def rase(est, ref, ctx=None):  # metrics.hpp:42
    return metrics(est, ref, which=METRIC_RASE, ctx=ctx)["rase"]


def circular_convolve(img, k, ctx=None, adjoint=False):
    img, k = _f(img), _f(k)
    out = np.empty_like(img)
    _check(_lib.fbmp_gpu_convolve(_ctx(ctx), _p(img), img.shape[0], img.shape[1], _p(k), k.shape[0], int(adjoint),
                                  _p(out)))
    return out


def circular_convolve_adjoint(img, k, ctx=None):
    return circular_convolve(img, k, ctx, adjoint=True)


# ---------------------------------------------------------------------------------------------
# spectral_weights.hpp / kernel_estimator.hpp
# ---------------------------------------------------------------------------------------------

def solve_weights(lrms_subset, pan, cfg: SpectralWeightConfig | None = None, ctx=None):
    """spectral_weights.hpp:24-25 -> omega (nb,)."""
    lrms, pan = _f(lrms_subset), _f(pan)
    cfg = cfg or SpectralWeightConfig()
    nb, h, w = lrms.shape
    if pan.shape != (cfg.factor * h, cfg.factor * w):
        raise DimensionError("solve_weights: PAN dimensions must be factor times the LRMS dimensions")
    om = np.empty(nb)
    c = cfg.c()
    _check(_lib.fbmp_gpu_solve_weights(_ctx(ctx), _p(lrms), nb, h, w, _p(pan), C.byref(c), _p(om)))
    return om


def combine_bands(lrms_subset, omega, ctx=None):
    lrms, om = _f(lrms_subset), _f(omega)
    if om.size != lrms.shape[0]:
        raise DimensionError("combine_bands: weight count does not match band count")
    out = np.empty(lrms.shape[1:])
    _check(_lib.fbmp_gpu_combine_bands(_ctx(ctx), _p(lrms), lrms.shape[0], lrms.shape[1], lrms.shape[2], _p(om),
                                       _p(out)))
    return out


def estimate_kernel_plane(pan, observation, factor, params: KernelEstParams | None = None, want_state=False,
                          hook_t=-1, ctx=None):
    """kernel_estimator.hpp:109-112 (TGV^2) -> (kernel, iterations[, state])."""
    pan, obs = _f(pan), _f(observation)
    prm = params or KernelEstParams()
    n = prm.n
    if pan.shape[0] != factor * obs.shape[0] or pan.shape[1] != factor * obs.shape[1]:
        raise DimensionError("build_observation: PAN dimensions must be factor times the observation")
    k = np.empty((n, n))
    it = C.c_int(0)
    st = np.empty((17, n, n)) if (want_state or hook_t >= 0) else None
    cp = prm.c()
    _check(_lib.fbmp_gpu_estimate_kernel_plane(_ctx(ctx), _p(pan), pan.shape[0], pan.shape[1], _p(obs), factor,
                                               C.byref(cp), _p(k), C.byref(it), _p(st), int(hook_t)))
    if st is not None:
        return k, it.value, dict(zip(STATE_FIELDS, st))
    return k, it.value


def estimate_kernel_tv_plane(pan, observation, factor, params: KernelEstParams | None = None, want_state=False,
                             hook_t=-1, ctx=None):
    """estimate_kernel_plane with KernelPrior::tv (kernel_estimator.cpp:445-452, run_tgv_or_tv(false))
    -> (kernel, iterations[, state]); the TV ablation estimator of the paper's Table II."""
    pan, obs = _f(pan), _f(observation)
    prm = params or KernelEstParams()
    n = prm.n
    if pan.shape[0] != factor * obs.shape[0] or pan.shape[1] != factor * obs.shape[1]:
        raise DimensionError("build_observation: PAN dimensions must be factor times the observation")
    k = np.empty((n, n))
    it = C.c_int(0)
    st = np.empty((17, n, n)) if (want_state or hook_t >= 0) else None
    cp = prm.c()
    _check(_lib.fbmp_gpu_estimate_kernel_tv_plane(_ctx(ctx), _p(pan), pan.shape[0], pan.shape[1], _p(obs), factor,
                                                  C.byref(cp), _p(k), C.byref(it), _p(st), int(hook_t)))
    if st is not None:
        return k, it.value, dict(zip(STATE_FIELDS, st))
    return k, it.value


def estimate_kernel_tv(lrms_subset, pan, omega, factor, params: KernelEstParams | None = None, ctx=None):
    """kernel_estimator.hpp:120-123 -> (kernel, iterations)."""
    return estimate_kernel_tv_plane(pan, combine_bands(lrms_subset, omega, ctx), factor, params, ctx=ctx)


def estimate_kernel_l2_plane(pan, observation, factor, params: KernelEstParams | None = None, ctx=None):
    """estimate_kernel_plane with KernelPrior::l2 (kernel_estimator.cpp:389-428, :438-455): the l2 +
    simplex ablation estimator of the paper's Table II -> (kernel, iterations)."""
    pan, obs = _f(pan), _f(observation)
    prm = params or KernelEstParams()
    if pan.shape[0] != factor * obs.shape[0] or pan.shape[1] != factor * obs.shape[1]:
        raise DimensionError("build_observation: PAN dimensions must be factor times the observation")
    k = np.empty((prm.n, prm.n))
    it = C.c_int(0)
    cp = prm.c()
    _check(_lib.fbmp_gpu_estimate_kernel_l2_plane(_ctx(ctx), _p(pan), pan.shape[0], pan.shape[1], _p(obs), factor,
                                                  C.byref(cp), _p(k), C.byref(it)))
    return k, it.value


def estimate_kernel_tgv(lrms_subset, pan, omega, factor, params: KernelEstParams | None = None, ctx=None):
    """kernel_estimator.hpp:114-118 -> (kernel, iterations)."""
    return estimate_kernel_plane(pan, combine_bands(lrms_subset, omega, ctx), factor, params, ctx=ctx)


def estimation_intensity_scale(pan, factor):
    """kernel_estimator.cpp:283-289 (host arithmetic on the caller's array)."""
    pan = _f(pan)
    m = float(np.abs(pan).max())
    if m <= 0:
        raise NumericalError("kernel estimation: PAN image is identically zero")
    hw = float(pan.shape[0] // factor) * (pan.shape[1] // factor)
    return float(np.sqrt(16384.0 / hw) / m)


def shrink2(columns, t, ctx=None):
    cols = _f(np.stack([_f(c) for c in columns]))
    _check(_lib.fbmp_gpu_shrink2(_ctx(ctx), _p(cols), cols.shape[0], C.c_longlong(cols[0].size), C.c_double(t)))
    return list(cols)


def project_simplex(v, ctx=None):
    v = _f(v)
    out = np.empty_like(v)
    _check(_lib.fbmp_gpu_project_simplex(_ctx(ctx), _p(v), int(v.size), _p(out)))
    return out


def solve_up(x, y, L1, L2, params: KernelEstParams | None = None, coupling=0.0, anchor=None, ctx=None):
    """kernel_estimator.hpp:78-80 (+ optional mu3 coupling) -> (u, p1, p2)."""
    fields = _f(np.stack(list(x) + list(y) + list(L1) + list(L2)))
    n = fields.shape[1]
    prm = (params or KernelEstParams()).c()
    u, p1, p2 = (np.empty((n, n)) for _ in range(3))
    anc = None if anchor is None else _f(anchor)
    _check(_lib.fbmp_gpu_solve_up(_ctx(ctx), _p(fields), n, C.byref(prm), C.c_double(coupling), _p(anc), _p(u),
                                  _p(p1), _p(p2)))
    return u, p1, p2


def gram(pan, obs, factor, n, ctx=None):
    """E^T E and E^T f of kernel_estimator.cpp:57-71 (unscaled)."""
    pan, obs = _f(pan), _f(obs)
    EtE = np.empty((n * n, n * n))
    Etf = np.empty(n * n)
    _check(_lib.fbmp_gpu_gram(_ctx(ctx), _p(pan), pan.shape[0], pan.shape[1], _p(obs), factor, n, _p(EtE), _p(Etf)))
    return EtE, Etf


def solve_z(EtE, Etf, n, mu3, anchor, ctx=None):
    """ObservationSystem::solve_z (kernel_estimator.cpp:79-83) on the device for a Gram matrix from gram()."""
    EtE, Etf, anchor = _f(EtE), _f(Etf), _f(anchor)
    z = np.empty(n * n)
    _check(_lib.fbmp_gpu_solve_z(_ctx(ctx), _p(EtE), _p(Etf), n, C.c_double(mu3), _p(anchor), _p(z)))
    return z


def data_objective(EtE, Etf, n, ff, u, ctx=None):
    """ObservationSystem::data_objective (kernel_estimator.cpp:85-87) on the device."""
    EtE, Etf, u = _f(EtE), _f(Etf), _f(u)
    v = C.c_double(0)
    _check(_lib.fbmp_gpu_data_objective(_ctx(ctx), _p(EtE), _p(Etf), n, C.c_double(ff), _p(u), C.byref(v)))
    return v.value


# ---------------------------------------------------------------------------------------------
# blind pipeline
# ---------------------------------------------------------------------------------------------

def _out(out, shape):
    """Caller-provided output (e.g. pinned host memory: no pageable staging in the D2H copy)."""
    if out is None:
        return np.empty(shape)
    if out.shape != tuple(shape) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float64 array of shape {tuple(shape)}")
    return out


def blind(lrms, pan, factor, n, sw: SpectralWeightConfig | None = None, ke: KernelEstParams | None = None,
          ps: PansharpenParams | None = None, ctx=None, out=None):
    """solve_weights(all bands) -> estimate_kernel_tgv -> pansharpen. Returns (hrms, info)."""
    lrms, pan = _f(lrms), _f(pan)
    N, h, w = lrms.shape
    sw = sw or SpectralWeightConfig(l=4, lambda_omega=10.0, factor=factor)
    sw.factor = factor
    ke = ke or KernelEstParams(n=n)
    ke.n = n
    ps = ps or PansharpenParams()
    out = _out(out, (N, h * factor, w * factor))
    k = np.empty((n, n))
    om = np.empty(N)
    c1, c2, c3 = sw.c(), ke.c(), ps.c()
    cx = ctx or default_context()
    _check(_lib.fbmp_gpu_blind(cx.h, _p(lrms), N, h, w, _p(pan), C.byref(c1), C.byref(c2), C.byref(c3), _p(out),
                               _p(k), _p(om)))
    st = cx.stats()
    return out, dict(kernel=k, omega=om, admm_iters=st["admm_iters"], cg_iters=st["cg_iters"][:N],
                     ms_weights=st["ms_weights"], ms_kernel_fit=st["ms_kernel_fit"],
                     ms_pansharpen=st["ms_pansharpen"])


def blind_subset(lrms, pan, factor, n, ch0, nch, sw=None, ke=None, ps=None, ctx=None, out=None):
    """Blind solve of bands [ch0, ch0+nch) with weights / kernel / normalisation over all bands
    (one rank's share of a channel-sharded solve). Returns (hrms (nch, H, W), kernel)."""
    lrms, pan = _f(lrms), _f(pan)
    N, h, w = lrms.shape
    sw = sw or SpectralWeightConfig(l=4, lambda_omega=10.0, factor=factor)
    sw.factor = factor
    ke = ke or KernelEstParams(n=n)
    ke.n = n
    ps = ps or PansharpenParams()
    out = _out(out, (nch, h * factor, w * factor))
    k = np.empty((n, n))
    c1, c2, c3 = sw.c(), ke.c(), ps.c()
    _check(_lib.fbmp_gpu_blind_subset(_ctx(ctx), _p(lrms), N, h, w, _p(pan), C.byref(c1), C.byref(c2), C.byref(c3),
                                      int(ch0), int(nch), _p(out), _p(k)))
    return out, k


def blind_batch(lrms, pan, factor, n, sw=None, ke=None, ps=None, ctx=None, out=None):
    """S independent scenes: lrms (S, N, h, w), pan (S, H, W) -> (hrms (S, N, H, W), kernels (S, n, n))."""
    lrms, pan = _f(lrms), _f(pan)
    S, N, h, w = lrms.shape
    sw = sw or SpectralWeightConfig(l=4, lambda_omega=10.0, factor=factor)
    sw.factor = factor
    ke = ke or KernelEstParams(n=n)
    ke.n = n
    ps = ps or PansharpenParams()
    out = _out(out, (S, N, h * factor, w * factor))
    k = np.empty((S, n, n))
    c1, c2, c3 = sw.c(), ke.c(), ps.c()
    _check(_lib.fbmp_gpu_blind_batch(_ctx(ctx), _p(lrms), S, N, h, w, _p(pan), C.byref(c1), C.byref(c2),
                                     C.byref(c3), _p(out), _p(k)))
    return out, k


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0), to be broadcast to all ranks for Context.set_comm."""
    buf = (C.c_ubyte * 128)()
    _check(_lib.fbmp_gpu_nccl_unique_id(buf))
    return bytes(buf)


def blind_strips_dev(d_lrms: int, N: int, h: int, w: int, d_pan: int, d_out: int, d_k: int, factor: int, n: int,
                     ctx: Context, vstrips: int = 1, sw=None, ke=None, ps=None):
    """Row-strip blind solve (raw device pointers): across the context's NCCL ranks, or on
    `vstrips` virtual ranks in this process when the context has no communicator."""
    sw = sw or SpectralWeightConfig(l=4, lambda_omega=10.0, factor=factor)
    sw.factor = factor
    ke = ke or KernelEstParams(n=n)
    ke.n = n
    ps = ps or PansharpenParams()
    c1, c2, c3 = sw.c(), ke.c(), ps.c()
    _check(_lib.fbmp_gpu_blind_strips_dev(ctx.h, C.cast(C.c_void_p(d_lrms), D), N, h, w, C.cast(C.c_void_p(d_pan), D),
                                          C.byref(c1), C.byref(c2), C.byref(c3), vstrips,
                                          C.cast(C.c_void_p(d_out), D), C.cast(C.c_void_p(d_k), D)))


def blind_batch_dev(d_lrms: int, S: int, N: int, h: int, w: int, d_pan: int, d_out: int, d_k: int, factor: int,
                    n: int, ctx: Context, ch0: int = 0, nch: int = -1, sw=None, ke=None, ps=None):
    """Device-resident batch / channel-subset blind solve (raw device pointers)."""
    sw = sw or SpectralWeightConfig(l=4, lambda_omega=10.0, factor=factor)
    sw.factor = factor
    ke = ke or KernelEstParams(n=n)
    ke.n = n
    ps = ps or PansharpenParams()
    c1, c2, c3 = sw.c(), ke.c(), ps.c()
    _check(_lib.fbmp_gpu_blind_batch_dev(ctx.h, C.cast(C.c_void_p(d_lrms), D), S, N, h, w,
                                         C.cast(C.c_void_p(d_pan), D), C.byref(c1), C.byref(c2), C.byref(c3), ch0,
                                         nch, C.cast(C.c_void_p(d_out), D), C.cast(C.c_void_p(d_k), D)))


def blind_dev(d_lrms: int, N: int, h: int, w: int, d_pan: int, d_out: int, d_k: int, factor: int, n: int,
              ctx: Context, sw=None, ke=None, ps=None):
    """Device-resident blind solve: all arguments are raw device pointers (e.g. tensor.data_ptr())."""
    sw = sw or SpectralWeightConfig(l=4, lambda_omega=10.0, factor=factor)
    sw.factor = factor
    ke = ke or KernelEstParams(n=n)
    ke.n = n
    ps = ps or PansharpenParams()
    c1, c2, c3 = sw.c(), ke.c(), ps.c()
    _check(_lib.fbmp_gpu_blind_dev(ctx.h, C.cast(C.c_void_p(d_lrms), D), N, h, w, C.cast(C.c_void_p(d_pan), D),
                                   C.byref(c1), C.byref(c2), C.byref(c3), C.cast(C.c_void_p(d_out), D),
                                   C.cast(C.c_void_p(d_k), D)))


EXPORTED_SYMBOLS = (
    "fbmp_gpu_default_ps_params", "fbmp_gpu_default_ke_params", "fbmp_gpu_default_sw_params",
    "fbmp_gpu_ctx_create", "fbmp_gpu_ctx_destroy", "fbmp_gpu_last_error", "fbmp_gpu_ctx_stats", "fbmp_gpu_ctx_cg_iters",
    "fbmp_gpu_ctx_stream", "fbmp_gpu_ctx_launches", "fbmp_gpu_ctx_set_profile", "fbmp_gpu_ctx_kernel_profile",
    "fbmp_gpu_ctx_set_precision", "fbmp_gpu_ctx_precision",
    "fbmp_gpu_metrics", "fbmp_gpu_estimate_kernel_l2_plane", "fbmp_gpu_estimate_kernel_tv_plane",
    "fbmp_gpu_estimate_kernel_tv",
    "fbmp_gpu_blind_batch_dev", "fbmp_gpu_blind_strips_dev", "fbmp_gpu_nccl_unique_id", "fbmp_gpu_ctx_set_comm",
    "fbmp_gpu_pansharpen", "fbmp_gpu_estimate_kernel_tgv",
    "fbmp_gpu_estimate_kernel_plane", "fbmp_gpu_solve_weights", "fbmp_gpu_combine_bands", "fbmp_gpu_blind",
    "fbmp_gpu_blind_dev", "fbmp_gpu_blind_batch", "fbmp_gpu_blind_subset", "fbmp_gpu_apply_prior", "fbmp_gpu_llp_apply",
    "fbmp_gpu_data_apply", "fbmp_gpu_cg_operator", "fbmp_gpu_warmstart_cg", "fbmp_gpu_guided_filter",
    "fbmp_gpu_guided_output", "fbmp_gpu_solve_channel_fft", "fbmp_gpu_box_mean", "fbmp_gpu_convolve",
    "fbmp_gpu_shrink2", "fbmp_gpu_project_simplex", "fbmp_gpu_solve_up", "fbmp_gpu_gram",
    "fbmp_gpu_solve_z", "fbmp_gpu_data_objective",
)
