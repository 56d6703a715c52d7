"""Shared by make_golden.py (fixture writer) and the GPU parity tests (fixture reader).

Whole-cube relative L2 without the cube: every band x is summarised by PROJ projections
y_j = <s_j, x> onto seeded Rademacher (+-1) vectors s_j. For a difference e = x_gpu - x_ref,
E[<s_j, e>^2] = ||e||^2, so mean_j (y_j(gpu) - y_j(ref))^2 estimates ||e||^2 with relative
standard deviation sqrt(2 / PROJ) (25 % at PROJ = 32): a rel-L2 gate of 1e-6 checked this way
has orders of magnitude of margin against results that differ at the 1e-9 level, yet fails on
any error that the whole-cube rel-L2 would reveal.
"""
import zlib

import numpy as np

PROJ = 32   # projections per band
CROP = 64   # crop side


def fixture_name(spec: str) -> str:
    return spec.lower().replace("@", "_") + "_blind.npz"


def crop_origins(H: int):
    """Four crops: centre, top-left corner (periodic-wrap region), and two off-centre."""
    c = CROP
    return [(H // 2 - c // 2, H // 2 - c // 2), (0, 0), (H // 4, 3 * H // 4 - c), (3 * H // 4 - c, H // 8)]


def _signs(seed: int, n: int) -> np.ndarray:
    bits = np.random.default_rng(seed).integers(0, 2, size=n, dtype=np.int8)
    return (2 * bits - 1).astype(np.float64)


def projections(cube: np.ndarray, spec: str) -> np.ndarray:
    """(bands, PROJ) projections of every band onto seeded sign vectors."""
    N = cube.shape[0]
    out = np.empty((N, PROJ))
    base = zlib.crc32(spec.encode())
    flat = cube.reshape(N, -1)
    for j in range(PROJ):
        s = _signs(base * 1000 + j, flat.shape[1])
        out[:, j] = flat @ s
    return out


def cube_rel_l2_estimate(proj_test: np.ndarray, proj_ref: np.ndarray, ref_norms: np.ndarray) -> float:
    """Estimated ||x_test - x_ref|| / ||x_ref|| over the whole cube from the projections."""
    err2 = np.mean((proj_test - proj_ref) ** 2, axis=1).sum()
    return float(np.sqrt(err2) / np.linalg.norm(ref_norms))
