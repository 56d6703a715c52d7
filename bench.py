#!/usr/bin/env python
"""Benchmark of the blind-pansharpening hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

One step = one full blind solve of one scene (spectral weights -> TGV^2 kernel fit ->
HRMS estimation of every band) on synthetic data of the config's shape (BASELINE.json
configs[1] = C2 by default). Multi-GPU (torchrun): every rank solves its own scene
(scene index = rank) with no data-path collective -> weak scaling.

`value`  : whole-job Mpixel*bands/s with inputs resident in HBM (CUDA events on the
           library's stream, L2 flushed with a 512 MB write before every step).
`e2e`    : the same metric through the public host-pointer C ABI (fbmp_gpu_blind), with
           the H2D upload of PAN + LRMS and the D2H download of the HRMS inside the step.
`roofline`: dominant CG kernel, algorithmic bytes / CUDA-event duration (profile pass).
`cpu_baseline`: the CPU oracle (oracle/, C++ restatement of the reference) on a bounded
           sample of the same scene, extrapolated to the full iteration counts.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2103_09943_b200 import synth  # noqa: E402

METRIC = "HRMS Mpixel·bands/s per blind-pansharpen solve, 1–8 B200; % HBM roofline"
UNIT = "Mpixel*bands/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(cfg: synth.SceneConfig) -> dict:
    return {"workload": f"{cfg.name}: {cfg.bands}-band scene, PAN {cfg.hr}x{cfg.hr}, r={cfg.ratio} "
                        f"(LRMS {cfg.lr}x{cfg.lr}x{cfg.bands}), blur {cfg.support}x{cfg.support}, "
                        f"shift +-{cfg.shift:g} px; blind solve = spectral weights + TGV^2 kernel fit "
                        f"(n={cfg.support}) + LLP HRMS solve of every band",
            "config": cfg.name, "pan": cfg.hr, "bands": cfg.bands, "ratio": cfg.ratio, "kernel_n": cfg.support,
            "l2": "flushed before every timed step (512 MB write)", "precision": "fp64 (reference precision)"}


# ----------------------------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
# CPU baseline / reference arm (oracle restatement of the reference, bounded sample)
# ----------------------------------------------------------------------------------------------
CG_CAP = 2      # CG iterations per band in a sample
ADMM_CAP = 20   # ADMM iterations in a sample
POST_DIV = 8    # the alias-group solve runs on 1/POST_DIV of the LR rows in a sample


def cpu_sample(scene, cfg, threads, cg_full=None, admm_full=None):
    """One bounded sample of the blind solve on the CPU oracle: CG capped at CG_CAP iterations per
    band, ADMM at ADMM_CAP iterations, the alias-group solve on the first 1/POST_DIV of the LR rows.
    Each capped phase is extrapolated linearly to the full solve (iteration counts of the full
    solve are identical on the oracle and the GPU, tests/test_gpu_pipeline.py). Returns (seconds
    for the full solve, description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # test infrastructure: the checker, timed here as the CPU baseline only
    cg_full = cg_full or REF_CG_ITERS.get(cfg.name)
    admm_full = admm_full or REF_ADMM_ITERS.get(cfg.name)
    h = cfg.hr // cfg.ratio
    post_rows = max(1, h // POST_DIV)
    r = oracle.blind_sampled(scene.lrms, scene.pan, cfg.ratio, cfg.support, CG_CAP, threads=threads,
                             admm_cap=ADMM_CAP if admm_full else 0, post_rows=post_rows)
    tw, tsetup, tadmm, tmat, tcg, tpost, tgroups = r["times"]
    admm_x = admm_full / r["admm_iters"] if admm_full else 1.0
    cg_x = max(cg_full) / CG_CAP if cg_full else 1.0
    grp_x = h / post_rows
    est = tw + tsetup + tadmm * admm_x + tmat + tcg * cg_x + tpost + tgroups * grp_x
    sample = (f"oracle (C++ restatement of the reference; FFT = own radix-2, alias solve = Householder + QL as "
              f"Eigen's SelfAdjointEigenSolver) on {cfg.name} scene 0, {threads} threads for the per-band phases: "
              f"weights {tw:.2f}s + fit setup {tsetup:.2f}s + ADMM {r['admm_iters']} it {tadmm:.2f}s (x{admm_x:.1f}) + "
              f"matting build {tmat:.2f}s + CG {CG_CAP} it/band {tcg:.2f}s (x{cg_x:.1f}) + guided/FFT {tpost:.2f}s + "
              f"alias groups of {post_rows}/{h} LR rows {tgroups:.2f}s (x{grp_x:.0f}); estimated full solve {est:.1f}s")
    return est, sample


def reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    scene = synth.make_scene(cfg, 0)
    threads = min(os.cpu_count() or 1, cfg.bands)
    times = []
    desc = ""
    for i in range(args.warmup + args.steps):
        est, desc = cpu_sample(scene, cfg, threads)
        if i >= args.warmup:
            times.append(est)
    T = sum(times)
    P = cfg.hr * cfg.hr
    value = args.steps * P * cfg.bands / T / 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator of BASELINE.json configs)",
            "config": workload(cfg), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# CG / ADMM iteration counts of scene 0 of each config (GPU; oracle == GPU at C1/C2/C4 in
# tests/test_gpu_pipeline.py); used only to extrapolate the bounded CPU sample.
REF_CG_ITERS = {"C1": [160, 157, 157, 158], "C2": [124, 125, 124, 125], "C4": [148, 147, 147, 147],
                "C3": [124, 123, 121, 120, 123, 123, 123, 121]}
REF_ADMM_ITERS = {"C1": 153, "C2": 179, "C4": 161, "C3": 167}


# ----------------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------------
def our_arm(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2103_09943_b200 import fbmp

    ctx = fbmp.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    # how the job is split over the ranks:
    #   scene batch (C4): the 64 scenes are partitioned, each rank solves its block as one batch;
    #   channel shards (C3 on > 1 GPU): every rank repeats the per-scene setup, solves its bands;
    #   replicas (C1, C2, C5, C3 on 1 GPU): each rank solves its own scene of the config (weak).
    from paper_2103_09943_b200 import shard
    if cfg.scenes > 1:
        mode, scaling = "scene-batch", "strong"
        mine = shard.partition(cfg.scenes, world, rank)
        scenes = [synth.make_scene(cfg, i) for i in mine]
        ch0, nch = 0, -1
    elif cfg.name == "C3" and world > 1:
        mode, scaling = "channel-shards", "strong"
        scenes = [synth.make_scene(cfg, 0)]
        part = shard.partition(cfg.bands, world, rank)
        ch0, nch = part.start, len(part)
    elif cfg.name == "C5" and world > 1:
        # one 8192^2 scene on row strips: r-halo exchange + allreduces over NCCL every CG iteration
        mode, scaling = "row-strips", "strong"
        scenes = [synth.make_scene(cfg, 0)]
        ch0, nch = 0, -1
        uid = [fbmp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_comm(uid[0], world, rank)
    else:
        mode, scaling = "replicas", "weak"
        scenes = [synth.make_scene(cfg, rank)]
        ch0, nch = 0, -1
    scene = scenes[0]
    S = len(scenes)
    N, h, w = scene.lrms.shape
    H, W = scene.pan.shape
    n = cfg.support
    NO = N if nch < 0 else nch          # bands reconstructed on this rank (per scene)
    dev = torch.device("cuda", local)
    lrms_np = np.stack([sc.lrms for sc in scenes])
    pan_np = np.stack([sc.pan for sc in scenes])
    d_lrms = torch.from_numpy(lrms_np).to(dev)
    d_pan = torch.from_numpy(pan_np).to(dev)
    d_out = torch.empty((S, NO, H, W), dtype=torch.float64, device=dev)
    d_k = torch.empty((S, n, n), dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def step():
        if mode == "row-strips":
            fbmp.blind_strips_dev(d_lrms.data_ptr(), N, h, w, d_pan.data_ptr(), d_out.data_ptr(), d_k.data_ptr(),
                                  cfg.ratio, n, ctx)
        else:
            fbmp.blind_batch_dev(d_lrms.data_ptr(), S, N, h, w, d_pan.data_ptr(), d_out.data_ptr(),
                                 d_k.data_ptr(), cfg.ratio, n, ctx, ch0=ch0, nch=nch)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev[i][0].record(stream)
            step()
            with torch.cuda.stream(stream):
                ev[i][1].record(stream)
        barrier()
    launches = ctx.launches - launches0
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    stats = ctx.stats()

    # e2e through the public host-pointer API (H2D + solve + D2H inside each step)
    lrms_h = torch.from_numpy(lrms_np).pin_memory().numpy()
    pan_h = torch.from_numpy(pan_np).pin_memory().numpy()

    # pinned host output (the C ABI writes into caller-owned buffers; pageable memory would add a
    # staging copy and first-touch page faults to every step)
    out_h = torch.empty((S, NO, H, W), dtype=torch.float64).pin_memory().numpy()

    def e2e_step():
        if mode == "row-strips":  # H2D of the (replicated) inputs, solve, D2H of the cube on rank 0
            with torch.cuda.stream(stream):
                d_lrms.copy_(torch.from_numpy(lrms_h), non_blocking=True)
                d_pan.copy_(torch.from_numpy(pan_h), non_blocking=True)
            step()
            with torch.cuda.stream(stream):
                if rank == 0:
                    d_out.cpu()
            return None
        if mode == "scene-batch":
            return fbmp.blind_batch(lrms_h, pan_h, cfg.ratio, n, ctx=ctx, out=out_h)
        if mode == "channel-shards":
            return fbmp.blind_subset(lrms_h[0], pan_h[0], cfg.ratio, n, ch0, nch, ctx=ctx, out=out_h[0])
        return fbmp.blind(lrms_h[0], pan_h[0], cfg.ratio, n, ctx=ctx, out=out_h[0])

    e2e_step()  # warm the host-pointer path
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    t_e2e = (time.perf_counter() - t0) * 1e3
    barrier()

    # roofline of the dominant CG kernel (profile pass: events bracket each kernel)
    ctx.set_profile(True)
    step()
    prof = ctx.kernel_profile()
    prof_ch_iters = ctx.stats()["cg_channel_iters"]
    ctx.set_profile(False)

    tt = torch.tensor([t_ms, t_e2e], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms, t_e2e = float(tt[0]), float(tt[1])
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    P = H * W
    # whole-job units per step: all pixel-bands of every scene the job solves
    job_units = {"scene-batch": cfg.scenes * P * N, "channel-shards": P * N, "replicas": world * P * N,
                 "row-strips": P * N}[mode]
    units = args.steps * job_units
    value = units / (t_ms / 1e3) / 1e6
    e2e = units / (t_e2e / 1e3) / 1e6
    s = 8
    p = h * w
    NC = S * NO  # channels in one launch of the CG kernels on this rank
    # algorithmic bytes per launch: only channels that are still iterating do work, so a launch
    # moves (channel-iterations / launches) channels' worth (converged channels exit at once);
    # the guide, mu_k and g_k maps are read per scene
    prof = {k: v for k, v in prof.items() if v["launches"] > 0}
    nlaunch = max(v["launches"] for v in prof.values())
    act = prof_ch_iters / max(nlaunch, 1)  # mean active channels per launch
    alg = {"K_Q": (3 * s * P + s * p) * act,        # read r, p_old; write p_new, q
           "K_D": (s * P + s * p) * act,            # read q; write d = B^T U q
           "K_L": 3 * s * P * act + 3 * s * P * S,  # read p, d, guide/mu/g (per scene); write Ap
           "K_U": 6 * s * P * act}                  # read z, r, p, Ap; write z, r
    dom = max(prof, key=lambda k: prof[k]["total_ms"])
    d = prof[dom]
    avg_ms = d["total_ms"] / max(d["launches"], 1)
    bytes_per_launch = alg[dom]
    achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9
    peak, kind = peaks()
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            if tj.get("config", "C2") == cfg.name:  # the capture's own config only
                traffic = tj.get(dom)
        except Exception:
            traffic = None
    cg_total = sum(v["total_ms"] for v in prof.values())
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom, "peak_kind": kind,
                "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
                "kernel_share_of_cg": {k: v["total_ms"] / cg_total for k, v in prof.items()} if cg_total else None,
                "cg_kernels": {k: {"launches": v["launches"], "avg_ms": v["total_ms"] / max(v["launches"], 1),
                                   "GB/s": alg[k] / (v["total_ms"] / max(v["launches"], 1) / 1e3) / 1e9}
                               for k, v in prof.items()}}
    h2d = S * (N * p + P) * 8
    d2h = S * (NO * P + n * n) * 8 + (N * 8 if mode == "replicas" else 0)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator of BASELINE.json configs)",
            "config": workload(cfg) | {"parallelism": f"{mode} x{world}", "scenes_per_rank": S,
                                       "bands_per_rank": NO},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "roofline": roofline, "clocks": clk.summary(),
            "stages_ms": {"weights": stats["ms_weights"], "kernel_fit": stats["ms_kernel_fit"],
                          "pansharpen": stats["ms_pansharpen"]},
            "iterations": {"admm": stats["admm_iters"], "cg": stats["cg_iters"][:NO]}}
    if world == 1 and not args.no_cpu_baseline and cfg.hr <= 2048:
        est, desc = cpu_sample(scene, cfg, min(os.cpu_count() or 1, N), cg_full=stats["cg_iters"][:N],
                               admm_full=stats["admm_iters"])
        cv = P * N / est / 1e6  # sample of one scene (the unit rate of the job)
        line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": min(os.cpu_count() or 1, N), "kind": "port",
                                "sample": desc}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        our_arm(args, cfg)


if __name__ == "__main__":
    main()
