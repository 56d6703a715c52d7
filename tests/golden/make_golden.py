"""Generate the committed golden fixtures (tests/golden/*.npz) with the CPU oracle.

The reference itself cannot be built in this image (no Eigen3 / FFTW3), so the
fixtures are produced by the oracle restatement (oracle/fbmp_oracle.cpp), which is pinned to
the reference's known answers (tests/test_oracle_kats.py) and cross-checked here against the
independent numpy restatement (oracle/fbmp_numpy.py) where that is affordable.

Each fixture stores the blind-pipeline result of one seeded BASELINE scene compactly:
kernel, spectral weights, ADMM / CG iteration counts, a central crop of every HRMS band, the
per-row sums of every band (a full-field linear checksum) and the band norms.

    python tests/golden/make_golden.py            # C1 (+ numpy cross-check)
    python tests/golden/make_golden.py C2         # C2 (~2 min on 4 cores)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle  # noqa: E402
import fbmp_numpy  # noqa: E402
from paper_2103_09943_b200 import synth  # noqa: E402

CROP = {"C1": 64, "C2": 128}


def make(cfg_name: str, crosscheck: bool):
    cfg = synth.CONFIGS[cfg_name]
    sc = synth.make_scene(cfg, 0)
    out, info = oracle.blind(sc.lrms, sc.pan, cfg.ratio, cfg.support, threads=min(4, os.cpu_count() or 1))
    if crosscheck:
        out_n, info_n = fbmp_numpy.blind(sc.lrms, sc.pan, cfg.ratio, cfg.support)
        assert info_n["admm_iters"] == info["admm_iters"]
        assert list(info_n["cg_iters"]) == list(info["cg_iters"])
        rel = np.linalg.norm(out_n - out) / np.linalg.norm(out)
        assert rel < 1e-6, rel
        print(f"{cfg_name}: numpy restatement agrees (rel L2 {rel:.2e})")
    H = cfg.hr
    c = CROP[cfg_name]
    lo = H // 2 - c // 2
    np.savez_compressed(
        os.path.join(HERE, f"{cfg_name.lower()}_blind.npz"),
        config=cfg_name, seed=sc.seed, kernel=info["kernel"], omega=info["omega"],
        admm_iters=info["admm_iters"], cg_iters=np.asarray(info["cg_iters"]),
        crop=out[:, lo:lo + c, lo:lo + c], crop_origin=lo, row_sums=out.sum(axis=2),
        band_norms=np.linalg.norm(out.reshape(out.shape[0], -1), axis=1),
        pan_checksum=float(sc.pan.sum()), lrms_checksum=float(sc.lrms.sum()))
    print(f"{cfg_name}: ADMM {info['admm_iters']} it, CG {list(info['cg_iters'])} it -> written")


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1"]
    for nm in names:
        make(nm, crosscheck=(nm == "C1"))
