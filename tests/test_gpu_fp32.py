"""fp32 mode of the HRMS CG (BASELINE.json north_star: "in an fp32 mode, <= 1e-3 relative L2 and
<= 0.05 dB PSNR deviation"). The CG vectors, taps, guide and window maps are fp32, every reduction
and CG scalar fp64; the kernel fit, guided filter and alias-group solve stay fp64. The deviation is
measured against the fp64 solve of the same scene, which itself matches the CPU oracle to 1e-9
(test_gpu_pipeline.py: live oracle on C1, golden fixtures on C2 / C3 / C5@2048) -- on C1 the
oracle is also compared directly. PSNR as metrics.cpp:24-27, 67-78 (peak 255, data x 255) after a
10-pixel border crop (the paper's evaluation)."""
import numpy as np
import pytest

from paper_2103_09943_b200 import synth

pytestmark = pytest.mark.gpu

REL_GATE = 1e-3    # north_star fp32 relative L2
PSNR_GATE = 0.05   # north_star fp32 PSNR deviation (dB)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def psnr(gpu, est, truth):
    return gpu.metrics(est * 255.0, truth * 255.0, crop=10, which=gpu.METRIC_PSNR)["psnr_avg"]


def solve(gpu, sc, cfg, bits):
    ctx = gpu.Context(0)
    ctx.set_precision(bits)
    assert ctx.precision == bits
    return gpu.blind(sc.lrms, sc.pan, cfg.ratio, cfg.support, ctx=ctx)


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5@1024"])
def test_fp32_gate(gpu, name):
    cfg_name, _, side = name.partition("@")
    cfg = synth.CONFIGS[cfg_name]
    sc = synth.make_scene(cfg, 0, hr=int(side) if side else None)
    o64, i64 = solve(gpu, sc, cfg, 64)
    o32, i32 = solve(gpu, sc, cfg, 32)
    assert i32["admm_iters"] == i64["admm_iters"]          # the kernel fit is fp64 in both modes
    assert rel(i32["kernel"], i64["kernel"]) < 1e-12
    assert rel(o32, o64) <= REL_GATE
    d = abs(psnr(gpu, o32, sc.hrms) - psnr(gpu, o64, sc.hrms))
    assert d <= PSNR_GATE
    # CG counts stay close (the stop rule is a relative step of 5e-5, far above fp32 rounding)
    assert max(abs(a - b) for a, b in zip(i32["cg_iters"], i64["cg_iters"])) <= 0.1 * max(i64["cg_iters"])


def test_fp32_c1_against_oracle(gpu, orc):
    cfg = synth.CONFIGS["C1"]
    sc = synth.make_scene(cfg, 0)
    out_o, _ = orc.blind(sc.lrms, sc.pan, 4, 15, threads=4)
    o32, _ = solve(gpu, sc, cfg, 32)
    assert rel(o32, out_o) <= REL_GATE
    assert abs(psnr(gpu, o32, sc.hrms) - psnr(gpu, out_o, sc.hrms)) <= PSNR_GATE


def test_fp32_batch_and_subset(gpu):
    """The fp32 mode through the batched (C4-style) and channel-subset (C3-style) entry points:
    a scene solved alone, in a batch, or as a band subset gives the same fp32 result."""
    cfg = synth.CONFIGS["C4"]
    scenes = [synth.make_scene(cfg, i, hr=256) for i in range(3)]
    ctx = gpu.Context(0)
    ctx.set_precision(32)
    lr = np.stack([s.lrms for s in scenes])
    pa = np.stack([s.pan for s in scenes])
    ob, _ = gpu.blind_batch(lr, pa, 4, cfg.support, ctx=ctx)
    for i, s in enumerate(scenes):
        o1, _ = gpu.blind(s.lrms, s.pan, 4, cfg.support, ctx=ctx)
        assert rel(ob[i], o1) == 0.0
    osub, _ = gpu.blind_subset(scenes[0].lrms, scenes[0].pan, 4, cfg.support, 1, 2, ctx=ctx)
    o1, _ = gpu.blind(scenes[0].lrms, scenes[0].pan, 4, cfg.support, ctx=ctx)
    assert rel(osub, o1[1:3]) == 0.0


def test_fp32_errors(gpu):
    ctx = gpu.Context(0)
    with pytest.raises(gpu.ParamError):
        ctx.set_precision(16)
    ctx.set_precision(32)
    sc = synth.make_scene("C1", hr=64)
    rng = np.random.default_rng(1)
    odd = rng.uniform(0, 1, (4, 15, 15))  # 60 x 60 HR: below the specialised operator's 64 x 64
    with pytest.raises(gpu.ParamError):
        gpu.pansharpen(odd, rng.uniform(0, 1, (60, 60)), np.full((7, 7), 1 / 49.0), 4, ctx=ctx)
    ctx.set_precision(64)
    gpu.blind(sc.lrms, sc.pan, 4, 7, ctx=ctx)
