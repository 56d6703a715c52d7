"""One warm-up + one measured blind solve of a config (driver for ncu / compute-sanitizer)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2103_09943_b200 import fbmp, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sc = synth.make_scene(cfg, 0)
ctx = fbmp.Context(0)
N, h, w = sc.lrms.shape
d_l = torch.from_numpy(sc.lrms).cuda()
d_p = torch.from_numpy(sc.pan).cuda()
d_o = torch.empty((N,) + sc.pan.shape, dtype=torch.float64, device="cuda")
d_k = torch.empty((cfg.support, cfg.support), dtype=torch.float64, device="cuda")
for i in range(reps):
    t = time.perf_counter()
    fbmp.blind_dev(d_l.data_ptr(), N, h, w, d_p.data_ptr(), d_o.data_ptr(), d_k.data_ptr(), cfg.ratio, cfg.support, ctx)
    torch.cuda.synchronize()
    st = ctx.stats()
    print(f"solve {i}: {1e3 * (time.perf_counter() - t):.2f} ms  fit {st['ms_kernel_fit']:.2f} ms  "
          f"hrms {st['ms_pansharpen']:.2f} ms  admm {st['admm_iters']}  cg {st['cg_iters'][:N]}", flush=True)
    if os.environ.get("RUN_ONE_SLEEP"):
        time.sleep(float(os.environ["RUN_ONE_SLEEP"]))
