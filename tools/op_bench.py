"""Repeated single-channel CG-operator applications on a C2-sized plane (ncu timing driver)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_09943_b200 import fbmp, synth  # noqa: E402

sc = synth.make_scene("C2", 0)
rng = np.random.default_rng(0)
guide = fbmp.apply_prior(sc.pan / sc.pan.max())
p = rng.uniform(-1, 1, guide.shape)
k = synth.make_kernel(rng, 17, 3.0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    fbmp.cg_operator(guide, p, k, 4)
print("ok")
