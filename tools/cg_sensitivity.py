"""CG trajectory sensitivity of the warm start ("CG trajectory sensitivity").

The warm-start CG stops on a relative step (pansharpen.cpp:248-253, cg_tol 5e-5). Two equally
valid CPU restatements -- FFT vs direct circular convolution for B, and assembled CSR vs
matrix-free matting -- differ only in rounding, yet on a white-noise PAN the trajectories drift
apart and may stop one iteration apart; on the BASELINE generator's scenes they agree.

    python tools/cg_sensitivity.py            # white noise 64^2 (n = 7) and the C1 generator scene
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import fbmp_numpy as fnp  # noqa: E402

from paper_2103_09943_b200 import synth  # noqa: E402


def run(pan, x, k, c, label):
    H, W = pan.shape
    guide = fnp.laplacian(pan / pan.max())
    khat = np.fft.fft2(fnp.embed_kernel(k, H, W))
    M = fnp.matting_matrix(guide)
    a = fnp.warmstart_cg(x, khat, c, lambda v: (M @ v.ravel()).reshape(v.shape), 2e-4, 5e-5, 2000)
    b = fnp.warmstart_cg(x, khat, c, lambda v: fnp.matting_apply_free(v, guide), 2e-4, 5e-5, 2000,
                         conv_f=lambda z: fnp.conv_direct(z, k), conv_a=lambda z: fnp.conv_adj_direct(z, k))
    d = np.linalg.norm(a[0] - b[0]) / np.linalg.norm(a[0])
    print(f"{label:34s} iterations FFT+CSR {a[1]:4d} | direct+matrix-free {b[1]:4d} | rel. diff of z {d:.1e}")


if __name__ == "__main__":
    rng = np.random.default_rng(64)
    pan = rng.uniform(0, 1, (64, 64))
    k = synth.make_kernel(rng, 7, 2.0)
    x = fnp.downsample(fnp.conv_direct(pan, k), 4) * 0.8
    run(pan, x, k, 4, "white-noise PAN 64^2, n = 7")
    sc = synth.make_scene("C1")
    kk = synth.make_kernel(np.random.default_rng(1), 15, 2.0)
    run(sc.pan, sc.lrms[1] / sc.pan.max(), kk, 4, "C1 generator scene 256^2, n = 15")
