"""Generate the committed golden fixtures (tests/golden/*.npz) with the CPU oracle.

The reference itself cannot be built in this image (no Eigen3 / FFTW3), so the
fixtures are produced by the oracle restatement (oracle/fbmp_oracle.cpp), which is pinned to
the reference's known answers (tests/test_oracle_kats.py) and cross-checked here against the
independent numpy restatement (oracle/fbmp_numpy.py) where that is affordable.

Each fixture stores the blind-pipeline result of one seeded BASELINE scene compactly:
kernel, spectral weights, ADMM / CG iteration counts, four crops of every HRMS band, per-row and
per-column sums of every band (full-field linear checksums), the band norms, and PROJ random
sign projections of every band (fixture_checks.projections): the mean squared projection of a
difference estimates its squared L2 norm (Johnson-Lindenstrauss), so a test can bound the
relative L2 error of the WHOLE cube without the cube being committed.

    python tests/golden/make_golden.py                 # C1 (+ numpy cross-check)
    python tests/golden/make_golden.py C2 C3 C5@2048   # C5@2048: the C5 generator at side 2048
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)

import oracle  # noqa: E402
import fbmp_numpy  # noqa: E402
from fixture_checks import CROP, crop_origins, fixture_name, projections  # noqa: E402
from paper_2103_09943_b200 import synth  # noqa: E402


def make(spec: str, crosscheck: bool):
    cfg_name, _, side = spec.partition("@")
    cfg = synth.CONFIGS[cfg_name]
    hr = int(side) if side else None
    sc = synth.make_scene(cfg, 0, hr=hr)
    t0 = time.time()
    threads = min(cfg.bands, os.cpu_count() or 1)
    out, info = oracle.blind(sc.lrms, sc.pan, cfg.ratio, cfg.support, threads=threads)
    t_solve = time.time() - t0
    if crosscheck:
        out_n, info_n = fbmp_numpy.blind(sc.lrms, sc.pan, cfg.ratio, cfg.support)
        assert info_n["admm_iters"] == info["admm_iters"]
        assert list(info_n["cg_iters"]) == list(info["cg_iters"])
        rel = np.linalg.norm(out_n - out) / np.linalg.norm(out)
        assert rel < 1e-6, rel
        print(f"{spec}: numpy restatement agrees (rel L2 {rel:.2e})")
    H = out.shape[1]
    c = CROP
    origins = crop_origins(H)
    np.savez_compressed(
        os.path.join(HERE, fixture_name(spec)),
        config=cfg_name, side=H, seed=sc.seed, kernel=info["kernel"], omega=info["omega"],
        admm_iters=info["admm_iters"], cg_iters=np.asarray(info["cg_iters"]),
        crops=np.stack([out[:, y:y + c, x:x + c] for y, x in origins]), crop_origins=np.asarray(origins),
        row_sums=out.sum(axis=2), col_sums=out.sum(axis=1),
        band_norms=np.linalg.norm(out.reshape(out.shape[0], -1), axis=1),
        projections=projections(out, spec),
        pan_checksum=float(sc.pan.sum()), lrms_checksum=float(sc.lrms.sum()),
        oracle_seconds=t_solve, oracle_threads=threads)
    print(f"{spec}: ADMM {info['admm_iters']} it, CG {list(info['cg_iters'])} it, oracle {t_solve:.1f}s "
          f"-> {fixture_name(spec)}")


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["C1"]:
        make(nm, crosscheck=(nm == "C1"))
