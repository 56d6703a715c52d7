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
`roofline`: the dominant CG operator (K_A = K_Q + K_L on the fused chain, K_Q + K_D + K_L otherwise;
           or K_U = K_DU / K_U), SURVEY 8(d) algorithmic bytes / CUDA-event duration (profile pass,
           one CG chain), the whole iteration (CG_iter, 11 s P) and the whole-solve fraction.
`cpu_baseline`: the CPU oracle (oracle/, C++ restatement of the reference): one complete solve
           of the same scene for C1/C2; a labelled estimate from a bounded sample for C3.
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
PRECISION = 64  # --precision: 64 (reference arithmetic, the headline) or 32 (north_star's fp32 mode)
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
            "l2": "flushed before every timed step (512 MB write)",
            "precision": "fp64 (reference precision)" if PRECISION == 64 else
                         "fp32 mode (HRMS CG vectors / stencils fp32, reductions and CG scalars fp64; fit, "
                         "guided filter and alias solve fp64)"}


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
# CPU baseline / reference arm (the oracle: C++ restatement of the reference, timed whole)
# ----------------------------------------------------------------------------------------------
FULL_SOLVE_MAX_HR = 1024  # C1 / C2: complete solves are timed (1 warm-up, median of 3)
CG_CAP = 2      # larger configs (C3 - C5, labelled estimates): CG iterations per band in a sample
ADMM_CAP = 20   # ADMM iterations in a sample
POST_DIV = 8    # the alias-group solve runs on 1/POST_DIV of the LR rows in a sample
ORACLE_DESC = ("oracle (C++ restatement of the reference; FFT = own radix-2 with FFTW's c2c conventions, "
               "alias solve = Householder + QL as Eigen's SelfAdjointEigenSolver, matting = assembled CSR SpMV)")


def ref_threads(cfg) -> int:
    """Threads the reference path uses: min(hardware_concurrency, N) channel workers for the HRMS
    stage (pansharpen.cpp:410-412); the weights and the kernel fit run on one core."""
    return max(1, min(os.cpu_count() or 1, cfg.bands))


def cpu_full_solve(scene, cfg, threads) -> float:
    """Seconds of one complete blind solve (solve_weights -> estimate_kernel_tgv -> pansharpen) of
    the scene on the CPU oracle, wall clock around the single library call."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # test infrastructure: the checker, timed here as the CPU baseline only
    t0 = time.perf_counter()
    oracle.blind(scene.lrms, scene.pan, cfg.ratio, cfg.support, threads=threads)
    return time.perf_counter() - t0


def cpu_sample(scene, cfg, threads, cg_full, admm_full):
    """ESTIMATE for configs whose complete CPU solve runs for many minutes (C3 - C5): CG capped at
    CG_CAP iterations per band, ADMM at ADMM_CAP, the alias-group solve on 1/POST_DIV of the LR
    rows, each capped phase scaled linearly to the iteration counts of the GPU solve of the same
    scene (cg_full, admm_full). Returns (estimated seconds, description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    h = cfg.hr // cfg.ratio
    post_rows = max(1, h // POST_DIV)
    r = oracle.blind_sampled(scene.lrms, scene.pan, cfg.ratio, cfg.support, CG_CAP, threads=threads,
                             admm_cap=ADMM_CAP, post_rows=post_rows)
    tw, tsetup, tadmm, tmat, tcg, tpost, tgroups = r["times"]
    admm_x = admm_full / r["admm_iters"]
    cg_x = max(cg_full) / CG_CAP
    grp_x = h / post_rows
    est = tw + tsetup + tadmm * admm_x + tmat + tcg * cg_x + tpost + tgroups * grp_x
    sample = (f"ESTIMATE from a bounded sample of the {ORACLE_DESC} on {cfg.name} scene 0, {threads} threads: "
              f"weights {tw:.2f}s + fit setup {tsetup:.2f}s + ADMM {r['admm_iters']} it {tadmm:.2f}s (x{admm_x:.1f}) + "
              f"matting build {tmat:.2f}s + CG {CG_CAP} it/band {tcg:.2f}s (x{cg_x:.1f}, GPU counts) + guided/FFT "
              f"{tpost:.2f}s + alias groups of {post_rows}/{h} LR rows {tgroups:.2f}s (x{grp_x:.0f}); "
              f"estimated full solve {est:.1f}s")
    return est, sample


def reference_arm(args, cfg):
    """The reference's CPU path (the oracle port: the reference itself cannot be built here or on
    the GPU box) on this arm's workload. C1/C2: complete solves, min(W, 1) warm-up
    and min(K, 3) timed solves (1 warm-up, median of 3), so the whole run takes a
    few minutes; `steps` / `warmup` report the solves actually run."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    scene = synth.make_scene(cfg, 0)
    threads = ref_threads(cfg)
    P = cfg.hr * cfg.hr
    if cfg.hr <= FULL_SOLVE_MAX_HR:
        warm, steps = min(args.warmup, 1), max(1, min(args.steps, 3))
        for _ in range(warm):
            cpu_full_solve(scene, cfg, threads)
        times = [cpu_full_solve(scene, cfg, threads) for _ in range(steps)]
        T = statistics.median(times)
        desc = (f"{ORACLE_DESC}: complete blind solves of {cfg.name} scene 0 (weights + TGV fit + HRMS of "
                f"{cfg.bands} bands), {threads} channel threads (pansharpen.cpp:410-412; weights and kernel fit "
                f"on 1 core), host nproc {os.cpu_count()}; {warm} warm-up + median of {steps}: "
                f"{', '.join(f'{t:.2f}s' for t in times)}")
    else:
        warm, steps = 0, 1
        T, desc = cpu_sample(scene, cfg, threads, REF_CG_ITERS[cfg.name], REF_ADMM_ITERS[cfg.name])
    value = P * cfg.bands / T / 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "requested": {"steps": args.steps, "warmup": args.warmup},
            "ms_per_step": 1e3 * T, "higher_is_better": True, "scaling": job_mode(cfg, world)[1],
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator of BASELINE.json configs)",
            "config": job_config(cfg, world), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
                             "host_nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# CG / ADMM iteration counts of scene 0 of the large configs (GPU == oracle where both ran); used
# only to scale the bounded CPU sample of C3 - C5 in the reference arm.
REF_CG_ITERS = {"C3": [124, 123, 121, 120, 123, 123, 123, 121], "C4": [148, 147, 147, 147],
                "C5": [103, 105, 103, 103, 105, 105, 103, 102]}
REF_ADMM_ITERS = {"C3": 167, "C4": 161, "C5": 274}


def job_mode(cfg, world):
    """How the job is split over the ranks; shared by both arms."""
    if cfg.scenes > 1:
        return "scene-batch", "strong"
    if cfg.name == "C3" and world > 1:
        return "channel-shards", "strong"
    if cfg.name == "C5" and world > 1:
        return "row-strips", "strong"
    return "replicas", "weak"


def job_config(cfg, world) -> dict:
    """The `config` dict of the JSON line (identical in both arms)."""
    mode, _ = job_mode(cfg, world)
    return workload(cfg) | {"parallelism": f"{mode} x{world}"}


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
    ctx.set_precision(PRECISION)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    # how the job is split over the ranks:
    #   scene batch (C4): the 64 scenes are partitioned, each rank solves its block as one batch;
    #   channel shards (C3 on > 1 GPU): every rank repeats the per-scene setup, solves its bands;
    #   replicas (C1, C2, C5, C3 on 1 GPU): each rank solves its own scene of the config (weak).
    from paper_2103_09943_b200 import shard
    mode, scaling = job_mode(cfg, world)
    ch0, nch = 0, -1
    if mode == "scene-batch":
        scenes = [synth.make_scene(cfg, i) for i in shard.partition(cfg.scenes, world, rank)]
    elif mode == "channel-shards":   # every rank repeats the per-scene setup and solves its bands
        scenes = [synth.make_scene(cfg, 0)]
        part = shard.partition(cfg.bands, world, rank)
        ch0, nch = part.start, len(part)
    elif mode == "row-strips":       # one 8192^2 scene: r-halo exchange + allreduces every CG iteration
        scenes = [synth.make_scene(cfg, 0)]
        uid = [fbmp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_comm(uid[0], world, rank)
    else:                            # replicas: each rank solves its own scene of the config (weak)
        scenes = [synth.make_scene(cfg, rank)]
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
    s = 8 if PRECISION == 64 else 4  # bytes per CG-vector element
    p = h * w
    # SURVEY 8(d) algorithmic bytes (compulsory HBM traffic of an ideally fused implementation).
    # Only channels that are still iterating do work, so a launch moves (channel-iterations /
    # launches) channels' worth (converged channels exit at their first instruction):
    #   K_A = K_Q + K_D + K_L (the operator application): read r, p_old, I; write p, Ap -> 5 s P
    #   K_U (axpys + norms): read z, r, p, Ap; write z, r                               -> 6 s P
    prof = {k: v for k, v in prof.items() if v["launches"] > 0}
    nlaunch = max(v["launches"] for v in prof.values())
    act = prof_ch_iters / max(nlaunch, 1)  # mean active channels per launch
    avg = {k: v["total_ms"] / max(v["launches"], 1) for k, v in prof.items()}
    # Fused path (no K_D launch): K_L writes w = L M L p instead of Ap, and K_U is K_DU, which forms
    # d = B^T U q in registers while it updates z and r. The operator split of the bytes is
    # unchanged (K_Q + K_L: r, p_old, I -> p, w; K_DU: z, r, p, w -> z, r) and the kernels together
    # move exactly the 11 s P of SURVEY 8(d), reported as CG_iter.
    fused = "K_D" not in avg
    ops = {"K_A": [k for k in ("K_Q", "K_D", "K_L") if k in avg], "K_U": ["K_U"],
           "CG_iter": [k for k in ("K_Q", "K_D", "K_L", "K_U") if k in avg]}
    alg = {"K_A": 5 * s * P * act, "K_U": 6 * s * P * act, "CG_iter": 11 * s * P * act}
    op_ms = {o: sum(avg[k] for k in ks) for o, ks in ops.items()}
    dom = max(("K_A", "K_U"), key=lambda o: op_ms[o])
    achieved = alg[dom] / (op_ms[dom] / 1e3) / 1e9
    peak, kind = peaks()
    traffic, traffic_src = None, None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            if tj.get("config", "C2") == cfg.name and all(k in tj for k in ops[dom]):  # the capture's own config
                traffic = sum(tj[k] for k in ops[dom])
                traffic_src = tj.get("source")
        except Exception:
            traffic = None
    cg_total = sum(v["total_ms"] for v in prof.values())
    # whole solve: B = s P (5 S + sum_c (13 + 11 K_c)) over this rank's scenes and channels
    K_all = stats["cg_iters"]
    B_solve = s * P * (5 * S + sum(13 + 11 * k for k in K_all))
    T_step = t_ms / args.steps / 1e3
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": f"{dom} ({' + '.join(ops[dom])})", "peak_kind": kind,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": alg[dom], "avg_launch_ms": op_ms[dom],
                "active_channels_per_launch": act,
                "operators": {o: {"kernels": ks, "avg_ms": op_ms[o], "algorithmic_bytes": alg[o],
                                  "GB/s": alg[o] / (op_ms[o] / 1e3) / 1e9,
                                  "frac": alg[o] / (op_ms[o] / 1e3) / 1e9 / peak} for o, ks in ops.items()},
                "cg_path": ("fused: K_Q3 -> K_L (w = L M L p, p.Ap = |q|^2 + lambda p.w) -> K_DU (K_U slot: data term "
                            "gather + update; d and Ap never stored)") if fused else "K_Q -> K_D -> K_L -> K_U",
                "kernel_avg_ms": avg,
                "kernel_share_of_cg": {k: v["total_ms"] / cg_total for k, v in prof.items()} if cg_total else None,
                "whole_solve": {"algorithmic_bytes": B_solve, "GB/s": B_solve / T_step / 1e9,
                                "frac": B_solve / T_step / 1e9 / peak}}
    h2d = S * (N * p + P) * 8
    d2h = S * (NO * P + n * n) * 8 + (N * 8 if mode == "replicas" else 0)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64" if PRECISION == 64 else "f32", "data": "synthetic (seeded generator of BASELINE.json configs)",
            "config": job_config(cfg, world),
            "job": {"scenes_per_rank": S, "bands_per_rank": NO},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "roofline": roofline, "clocks": clk.summary(),
            "stages_ms": {"weights": stats["ms_weights"], "kernel_fit": stats["ms_kernel_fit"],
                          "pansharpen": stats["ms_pansharpen"]},
            "iterations": {"admm": stats["admm_iters"], "cg": stats["cg_iters"][:S * NO]}}
    if world == 1 and not args.no_cpu_baseline and cfg.hr <= 2048:
        th = ref_threads(cfg)
        if cfg.hr <= FULL_SOLVE_MAX_HR:  # one complete CPU solve of the same scene
            est = cpu_full_solve(scene, cfg, th)
            desc = (f"{ORACLE_DESC}: one complete blind solve of {cfg.name} scene {rank} ({cfg.bands} bands), "
                    f"{th} channel threads (weights and kernel fit on 1 core), host nproc {os.cpu_count()}: "
                    f"{est:.2f}s")
        else:
            est, desc = cpu_sample(scene, cfg, th, stats["cg_iters"][:N], stats["admm_iters"])
        cv = P * N / est / 1e6  # one scene (the unit rate of the job)
        line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": th, "kind": "port", "sample": desc,
                                "host_nproc": os.cpu_count()}
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
    ap.add_argument("--precision", type=int, default=64, choices=[32, 64])
    args = ap.parse_args()
    global PRECISION
    PRECISION = args.precision
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        our_arm(args, cfg)


if __name__ == "__main__":
    main()
