"""Blind solve of a config: print the CG iteration counts and the HRMS relative difference to the
oracle fixture; optionally save the HRMS (debug driver for K_Q variants; env selects the variant).
usage: python tools/c1_iters.py [C1|C2] [n] [save.npy]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_09943_b200 import fbmp, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
sc = synth.make_scene(name)
out, info = fbmp.blind(sc.lrms, sc.pan, 4, n)
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         f"{name.lower()}_blind.npz"))
lo, c = int(g["crop_origin"]), g["crop"].shape[1]
crop = out[:, lo:lo + c, lo:lo + c]
per = [float(np.linalg.norm(crop[b] - g["crop"][b]) / np.linalg.norm(g["crop"][b])) for b in range(crop.shape[0])]
print(os.environ.get("TAG", ""), "cg", list(info["cg_iters"]), "golden", list(g["cg_iters"]),
      "crop rel per band", ["%.2e" % v for v in per], flush=True)
if len(sys.argv) > 3:
    np.save(sys.argv[3], out)
