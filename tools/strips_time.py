"""Time the row-strip blind solve on virtual ranks (one process): python tools/strips_time.py C2 2 [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2103_09943_b200 import fbmp, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sc = synth.make_scene(cfg, 0)
ctx = fbmp.Context(0)
N, h, w = sc.lrms.shape
d_l, d_p = torch.from_numpy(sc.lrms).cuda(), torch.from_numpy(sc.pan).cuda()
d_o = torch.empty((N,) + sc.pan.shape, dtype=torch.float64, device="cuda")
d_k = torch.empty((cfg.support, cfg.support), dtype=torch.float64, device="cuda")
for i in range(reps):
    t = time.perf_counter()
    fbmp.blind_strips_dev(d_l.data_ptr(), N, h, w, d_p.data_ptr(), d_o.data_ptr(), d_k.data_ptr(), cfg.ratio, cfg.support,
                          ctx, vstrips=G)
    torch.cuda.synchronize()
    st = ctx.stats()
    print(f"strips G={G} solve {i}: {1e3 * (time.perf_counter() - t):.2f} ms  hrms {st['ms_pansharpen']:.2f} ms  "
          f"cg {st['cg_iters'][:N]}  launches {ctx.launches}", flush=True)
