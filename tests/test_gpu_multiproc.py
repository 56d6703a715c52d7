"""The multi-GPU job split that bench.py runs, exercised with two real processes
(torch.distributed, gloo for the gather) calling the device-resident entry points exactly as
bench.py's ranks do: scene batches (C4 mode) and channel shards (C3 mode) through
fbmp.blind_batch_dev, results gathered on rank 0 with shard.gather_blocks and compared
bit-for-bit with a single-process solve of the whole job.

Both ranks run on cuda:0 of the one B200 the test box has. That is sound here because these
modes have no data-path collective -- neither rank's kernels wait on the other's -- so sharing
the device changes the timing only, not the work or the bits.
"""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank_share(cfg_name, hr, world, rank, n_scenes):
    """One rank's share of the job, with bench.py's calls (device-resident inputs and outputs)."""
    import torch
    from paper_2103_09943_b200 import fbmp, shard, synth

    cfg = synth.CONFIGS[cfg_name]
    ctx = fbmp.Context(0)
    if n_scenes > 1:  # scene-batch
        mine = shard.partition(n_scenes, world, rank)
        scenes = [synth.make_scene(cfg, i, hr=hr) for i in mine]
        ch0, nch = 0, -1
    else:             # channel-shards
        scenes = [synth.make_scene(cfg, 0, hr=hr)]
        part = shard.partition(cfg.bands, world, rank)
        ch0, nch = part.start, len(part)
    S = len(scenes)
    N, h, w = scenes[0].lrms.shape
    NO = N if nch < 0 else nch
    dev = torch.device("cuda", 0)
    d_l = torch.from_numpy(np.stack([s.lrms for s in scenes])).to(dev)
    d_p = torch.from_numpy(np.stack([s.pan for s in scenes])).to(dev)
    d_o = torch.empty((S, NO, h * cfg.ratio, w * cfg.ratio), dtype=torch.float64, device=dev)
    d_k = torch.empty((S, cfg.support, cfg.support), dtype=torch.float64, device=dev)
    fbmp.blind_batch_dev(d_l.data_ptr(), S, N, h, w, d_p.data_ptr(), d_o.data_ptr(), d_k.data_ptr(), cfg.ratio,
                         cfg.support, ctx, ch0=ch0, nch=nch)
    torch.cuda.synchronize()
    out = d_o.cpu().numpy()
    return out if n_scenes > 1 else out[0]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2103_09943_b200 import shard, synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    # C4 mode: 3 scenes of the C4 generator (side 256) over 2 ranks (2 + 1)
    n_sc = 3
    counts = [len(shard.partition(n_sc, world, r)) for r in range(world)]
    res["scenes"] = shard.gather_blocks(_rank_share("C4", 256, world, rank, n_sc), counts)
    # C3 mode: the 8 bands of the C3 generator (side 256) over 2 ranks (4 + 4)
    counts = [len(shard.partition(8, world, r)) for r in range(world)]
    res["channels"] = shard.gather_blocks(_rank_share("C3", 256, world, rank, 1), counts)
    if rank == 0:
        from paper_2103_09943_b200 import fbmp
        scenes = [synth.make_scene("C4", i, hr=256) for i in range(n_sc)]
        ref_sc, _ = fbmp.blind_batch(np.stack([s.lrms for s in scenes]), np.stack([s.pan for s in scenes]), 4, 15)
        c3 = synth.make_scene("C3", 0, hr=256)
        ref_ch, _ = fbmp.blind(c3.lrms, c3.pan, 4, 15)
        q.put((np.array_equal(res["scenes"], ref_sc), np.array_equal(res["channels"], ref_ch)))
    dist.destroy_process_group()


def test_bench_job_split_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok == (True, True)
