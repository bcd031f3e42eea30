#!/usr/bin/env python
"""Benchmark: CNSF fan-beam forward + back-projection pairs per second.

One step = one FP+BP pair over one image of the configured workload (default
config 2: 512^2 Shepp-Logan, 720 views, 1024 bins, SID 500 / SDD 1000 mm):
  y_g = A_g c            (cbp_forward over this rank's view shard)
  c'  = sum_g A_g^T y_g  (cbp_back over the shard, then NCCL all_reduce)
With N GPUs the views are sharded (strong scaling: the pair's work is fixed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2]
  python bench.py --impl reference ...   # the FP64 CPU oracle arm

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream,
per step, L2 flushed (256 MiB write) between steps outside the events, max
over ranks.  See DESIGN.md section 6 for the roofline arithmetic.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "fwd+back projection pairs/sec at 512²×720 views×1024 dets; % FP32/HBM roofline"
FLOPS_PER_WEIGHT = 32  # canonical FP32 flops per nonzero weight
WORKLOADS = {
    "1": "config1: 64x64 Shepp-Logan, 90 views, 128 bins, SID 500 / SDD 1000 mm",
    "2": "config2: 512x512 Shepp-Logan, 720 views, 1024 bins, SID 500 / SDD 1000 mm",
    "3": "config3: 1024x1024 Shepp-Logan, 1440 views, 2048 bins, SID 500 / SDD 1000 mm",
    "4": "config4: batch of 64 512x512 jittered Shepp-Logan slices, 720 views, 1024 bins",
    "5": "config5: 2048x2048 Shepp-Logan, 2880 views, 4096 bins (one pair of the SART/CGLS loop)",
    # the general path (no view symmetry) and the paper's own timing shapes
    "2v721": "config2 geometry with 721 views (no 4-/8-fold view symmetry: the direct kernels)",
    "p256": "paper timing shape (P:512-515): 256x256 all-ones, h 1 mm, 360 views, 815 bins, D_po = D_so = 400 mm",
    "p512": "paper timing shape (P:512-515): 512x512 all-ones, h 1 mm, 360 views, 1627 bins, D_po = D_so = 800 mm",
    "p1024": "paper timing shape (P:512-515): 1024x1024 all-ones, h 1 mm, 360 views, 3250 bins, "
             "D_po = D_so = 1600 mm",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="cnsf", choices=["cnsf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--views", default=None,
                    help="a:b -- project views [a, b) only (a view sub-range: the direct kernels)")
    return ap.parse_args()


def view_range(args, g):
    """(v0, nv) of the projected views: all, or the --views sub-range"""
    if not args.views:
        return 0, g["n_views"]
    a, b = (int(x) for x in args.views.split(":"))
    if not 0 <= a < b <= g["n_views"]:
        raise SystemExit(f"--views {args.views}: outside [0, {g['n_views']})")
    return a, b - a


def batch_of(cfg: str) -> int:
    return W.BATCH.get(cfg, 1)


def host_image(cfg: str, n: int, batch: int):
    if cfg.startswith("p"):
        return W.ones(n)  # the paper's timing images
    return W.shepp_logan(n) if batch == 1 else W.jittered_batch(n, batch, seed=7)


def bench_config(args, g, world: int, mode: str, slice_shard: bool) -> dict:
    """the `config` dict of the JSON line -- identical for the CUDA arm and the
    reference arm of the same command"""
    v0, nv = view_range(args, g)
    total_batch = batch_of(args.config)
    par = (f"slices/{world}" if slice_shard else (f"views/{world}" if world > 1 else "single"))
    par += {"orbit": " (4-fold rotational symmetry)", "dihedral": " (8-fold dihedral symmetry)"}.get(mode, "")
    cfg = {"workload": WORKLOADS[args.config], "n": g["n"], "n_views": g["n_views"],
           "n_det": g["n_det"], "pixel_mm": g["pixel"], "det_pitch_mm": g["det_pitch"],
           "det_width_mm": g["det_width"], "sid_mm": g["sid"], "sdd_mm": g["sdd"], "batch": total_batch,
           "parallelism": par,
           "l2": "flushed between steps (256 MiB write, outside the timed events)"}
    if args.views:
        cfg["views"] = f"{v0}:{v0 + nv}"
    return cfg


def weight_counts(cfg: str):
    cfg = {"4": "2"}.get(cfg, cfg)  # config 4 = 64 slices in the geometry of config 2
    path = os.path.join(ROOT, "tests", "golden", "weight_counts.json")
    try:
        return json.load(open(path))[cfg]["per_view"]
    except (OSError, KeyError):
        return None


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


def traffic_table():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/cbp_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        busy = [s for s in sm if s > 0]
        return {"sm_mhz": statistics.median(busy) if busy else 0.0, "sm_max_mhz": max(mx),
                "power_w_max": max(pw), "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------- reference arm
def _shard_mode(args, g, world):
    from paper_1907_10526_b200.sharded import make_shard
    batch = batch_of(args.config)
    slice_shard = batch > 1 and world > 1
    if slice_shard or args.views or world == 1:
        return "block", slice_shard
    return make_shard(g["n_views"], 0, world, batch, dihedral=True).mode, False


def run_reference(args, rank, world):
    """The FP64 CPU oracle as it stands (bench's reference arm: there is no
    reference implementation to install).  Each step is the
    oracle's FP+BP over a bounded, rotating sample of the workload's views,
    sized so the whole --warmup + --steps run takes about a minute;
    `ms_per_step` is the measured time of such a step and `value` the pairs
    per second it implies (views done / views per pair / time)."""
    if rank != 0:
        return
    import oracle as O
    g = W.geometry(args.config)
    v0, nv = view_range(args, g)
    batch = batch_of(args.config)
    img = host_image(args.config, g["n"], 1).astype(np.float64)  # the oracle has no batch sharing: per slice
    cores = os.cpu_count() or 1
    O.build()
    probe = min(nv, max(8, cores))
    t0 = time.perf_counter()
    y = O.forward(g, img, view_begin=v0, view_count=probe, threads=cores)
    O.back(g, y, view_begin=v0, threads=cores)
    per_view = (time.perf_counter() - t0) / probe
    budget = 60.0 / max(1, args.steps + args.warmup)
    nvs = int(max(min(nv, cores), min(nv, budget / max(per_view, 1e-6))))
    times = []
    for k in range(args.warmup + args.steps):
        a = v0 + (k * 37) % (nv - nvs + 1)
        t0 = time.perf_counter()
        y = O.forward(g, img, view_begin=a, view_count=nvs, threads=cores)
        O.back(g, y, view_begin=a, threads=cores)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    t_step = sum(times) / len(times)
    pairs_per_step = nvs / nv  # of one slice's pair
    value = pairs_per_step / t_step
    sample = (f"each step: oracle FP+BP of one slice over {nvs} of the pair's {nv} views (rotating), "
              f"{pairs_per_step:.3f} of a pair in {t_step:.2f} s; {cores} OpenMP threads")
    mode, slice_shard = _shard_mode(args, g, world)
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "pairs_per_step": pairs_per_step,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, g, world, mode, slice_shard),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if batch > 1:
        line["note"] = f"per slice of the {batch}-slice batch (the oracle evaluates every weight per slice)"
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg: str, v0: int, nv: int, target_s: float = 12.0):
    """oracle FP+BP on a bounded view sample of the same workload (rank 0,
    N=1), plus one whole config-1 pair on a single thread."""
    import oracle as O
    g = W.geometry(cfg)
    img = host_image(cfg, g["n"], 1).astype(np.float64)
    cores = os.cpu_count() or 1
    O.build()
    probe = min(nv, max(8, cores))
    t0 = time.perf_counter()
    y = O.forward(g, img, view_begin=v0, view_count=probe, threads=cores)
    O.back(g, y, view_begin=v0, threads=cores)
    per_view = (time.perf_counter() - t0) / probe
    nvs = int(max(probe, min(nv, target_s / max(per_view, 1e-6))))
    t0 = time.perf_counter()
    y = O.forward(g, img, view_begin=v0, view_count=nvs, threads=cores)
    O.back(g, y, view_begin=v0, threads=cores)
    dt = time.perf_counter() - t0
    g1 = W.geometry("1")
    img1 = W.shepp_logan(g1["n"]).astype(np.float64)
    t1 = time.perf_counter()
    O.back(g1, O.forward(g1, img1, threads=1), threads=1)
    t1 = time.perf_counter() - t1
    return {"value": nvs / (dt * nv), "unit": "pairs/s", "cores": cores,
            "kind": "oracle",
            "sample": f"FP+BP over views {v0}..{v0 + nvs - 1} of the pair's {nv} ({dt:.1f} s wall), "
                      f"scaled to one full pair",
            "config1_single_thread_pair_s": t1}


# -------------------------------------------------------------------- CUDA arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1907_10526_b200 as cbp
    from paper_1907_10526_b200.sharded import MulticastImage, Shard, back_sharded, make_shard, view_shard

    assert args.warmup >= 3, "at least 3 warm-up steps"
    # CBP_BENCH_BACKEND=gloo (a logic check, not a measurement): the ranks may
    # share GPUs (device = local rank mod the device count) and the BP partials
    # are summed through gloo, so the N > 1 code path runs on a one-GPU box
    backend = os.environ.get("CBP_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    g = W.geometry(args.config)
    n, ns = g["n"], g["n_det"]
    batch = batch_of(args.config)
    rv0, rnv = view_range(args, g)
    # view shard of this rank: the orbits of a block of base views under the
    # 8 frames (one image, n_views % 8 == 0: the BP keeps one weight per 8
    # views on every rank), else the 4 rotated copies of a block of base views
    # (n_views % 4 == 0), else a contiguous block
    # A batch (config 4) shards SLICES instead: each rank projects its slices
    # over all views (replicas of the single-GPU path, no communication;
    # SURVEY 8(e)).
    slice_shard = batch > 1 and world > 1
    total_batch = batch
    s0 = 0
    if slice_shard:
        s0, batch = view_shard(total_batch, rank, world)
        sh = make_shard(g["n_views"], 0, 1)
    elif args.views:  # a view sub-range: contiguous blocks of it (the direct kernels)
        a, c = view_shard(rnv, rank, world)
        sh = Shard("block", rv0 + a, c, g["n_views"])
    else:
        sh = make_shard(g["n_views"], rank, world, batch, dihedral=True)
    views = sh.views()
    nv = len(views)
    orbit = sh.mode == "orbit"
    dihedral = sh.mode == "dihedral"

    host_img = host_image(args.config, n, total_batch)
    if total_batch > 1:
        host_img = host_img[s0:s0 + batch]
    img = torch.from_numpy(np.ascontiguousarray(host_img)).to(dev)
    bshape = () if total_batch == 1 else (batch,)
    sshape = (4, sh.count, ns) if orbit else ((g["n_views"], ns) if dihedral else bshape + (nv, ns))
    sino = torch.zeros(sshape, dtype=torch.float32, device=dev)
    out = torch.empty(bshape + (n, n), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def _graph_call(fn, a, b, st):
        nonlocal stream
        saved = stream
        stream = st
        try:
            fn(a, b)
        finally:
            stream = saved

    def fwd(image, y):
        if orbit:
            cbp.forward_orbit(g, image, sh.begin, sh.count, sino=y, stream=stream)
        elif dihedral:
            cbp.forward_dihedral(g, image, sh.begin, sh.count, sino=y, stream=stream)
        else:
            cbp.forward(g, image, y, view_begin=sh.begin, view_count=sh.count, stream=stream)

    def bwd(y, image):
        if orbit:
            cbp.back_orbit(g, y, sh.begin, image=image, stream=stream)
        elif dihedral:
            cbp.back_dihedral(g, y, sh.begin, sh.count, image=image, stream=stream)
        else:
            cbp.back(g, y, image, view_begin=sh.begin, stream=stream)

    # The timed step replays the FP and the BP as two CUDA graphs captured from
    # the same library calls (the library's kernels, scratch allocations and
    # programmatic-launch edges become graph nodes): the device timing then
    # does not depend on how fast this Python loop enqueues -- with eager
    # launches, host jitter (the clock sampler's driver queries, GC) left the
    # GPU idle inside a few steps' BP interval (0.5-20 ms outliers; round 2).
    # CBP_BENCH_EAGER=1 times eager launches instead.
    graphs, graph_kernels = None, (0, 0)
    # N > 1, view shards: the BP's partial images are summed by the BP itself
    # through an NVLink multicast image (CBP_ACC_MULTIMEM, sharded.MulticastImage)
    # when the system has one and a first step agrees with the NCCL all-reduce;
    # else (or CBP_BENCH_NCCL=1) by NCCL's all_reduce after the BP
    mm, reduce_note = None, (f"{backend} all_reduce after the BP" if world > 1 and not slice_shard else "none")
    if world > 1 and not slice_shard and os.environ.get("CBP_BENCH_NCCL") != "1" and backend == "nccl":
        why = ""
        try:
            mm = MulticastImage(n, device=dev)
        except Exception as exc:  # noqa: BLE001
            mm, why = None, str(exc)[:100]
        # every rank agrees before any multicast barrier runs
        ok = torch.tensor([1.0 if mm is not None else 0.0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 1.0:
            fwd(img, sino)
            bwd(sino, out)
            dist.all_reduce(out)
            ref = out.clone()
            try:  # a failure here votes no (every rank still reaches the vote below)
                res = back_sharded(g, sino, sh, multimem=mm, stream=stream)
                torch.cuda.synchronize()
                err = float((res - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
            except Exception as exc:  # noqa: BLE001
                err, why = float("inf"), f"multicast BP failed: {str(exc)[:80]}"
            ok.fill_(1.0 if err <= 1e-5 else 0.0)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            why = why or f"multicast BP disagreed with NCCL on some rank (here {err:.1e})"
        if ok.item() == 1.0:
            reduce_note = f"fused into the BP epilogue through NVLink multicast (checked against NCCL: {err:.1e})"
        else:
            mm = None
            reduce_note = f"NCCL all_reduce after the BP ({why or 'multicast unavailable on some rank'})"

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        if graphs:
            graphs[0].replay()
        else:
            fwd(img, sino)
        if ev:
            ev[1].record(stream)
        if mm is not None:  # the BP adds into every rank's copy; zero + barriers before / after
            back_sharded(g, sino, sh, multimem=mm, stream=stream)
        elif graphs:
            graphs[1].replay()
        else:
            bwd(sino, out)
        if ev:
            ev[2].record(stream)
        if world > 1 and not slice_shard and mm is None:
            dist.all_reduce(out)
        if ev:
            ev[3].record(stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if os.environ.get("CBP_BENCH_EAGER") != "1":
        try:
            gfp, gbp = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            c0 = cbp.launch_count()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(gfp, stream=cap):
                    _graph_call(fwd, img, sino, cap)
                c1 = cbp.launch_count()
                with torch.cuda.graph(gbp, stream=cap):
                    _graph_call(bwd, sino, out, cap)
            stream.wait_stream(cap)
            torch.cuda.synchronize()
            # the library's kernels captured in each graph: every replay launches them again
            graph_kernels = (c1 - c0, cbp.launch_count() - c1)
            graphs = (gfp, gbp)
            for _ in range(3):  # warm the graphs
                flush.zero_()
                step()
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001 -- fall back to eager launches, say so in the line
            graphs, graph_kernels = None, (0, 0)
            graph_note = f"graph capture failed ({type(exc).__name__}: {str(exc)[:120]}); eager launches"
        else:
            graph_note = "FP and BP each replayed as a CUDA graph of the library calls"
    else:
        graph_note = "eager launches (CBP_BENCH_EAGER=1)"

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clocks:
        clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = cbp.launch_count()
    for k in range(args.steps):
        flush.zero_()  # L2 flush, outside the timed events
        step(evs[k])
    torch.cuda.synchronize()
    # eager library calls count themselves; graph replays launch the captured kernels
    launches = cbp.launch_count() - launches0
    if graphs:
        launches += args.steps * (graph_kernels[0] + (graph_kernels[1] if mm is None else 0))
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None

    fp_ms = [e[0].elapsed_time(e[1]) for e in evs]
    bp_ms = [e[1].elapsed_time(e[2]) for e in evs]
    ar_ms = [e[2].elapsed_time(e[3]) for e in evs]
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    value = args.steps * total_batch / (total_ms * 1e-3)  # FP+BP pairs (one per slice, all ranks) per second

    # ---- roofline of the dominant kernel (ALU / FP32-pipe bound)
    # units = nonzero (view, bin, pixel) weights of this rank's views x slices;
    # each weight is EVALUATED once per `fold` units (4 views by symmetry, or
    # S slices of a batch), at 30 flops, plus 2 flops per unit accumulated
    counts = weight_counts(args.config)
    nw = int(sum(counts[v] for v in views)) if counts else None
    # views (symmetry) or slices (batch) per weight evaluation, FP and BP
    sym = 4 if orbit else (8 if dihedral else cbp.symmetry_fold(g, batch, sh.begin, sh.count))
    fp_mirror = bool(os.environ.get("CBP_FP_MIRROR"))
    slices = 4 if batch >= 4 else (2 if batch >= 2 else 1)
    if batch > 1:  # FP: weights shared by the batch's slices; BP: symmetry per image
        folds = {"fp": slices, "bp": sym if sym > 1 else slices}
    else:
        folds = {"fp": sym if (sym != 8 or fp_mirror) else 4, "bp": sym}
    units = nw * batch if nw else None
    props = torch.cuda.get_device_properties(dev)
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0)
    peak_tflops = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12
    fp_avg, bp_avg = statistics.mean(fp_ms), statistics.mean(bp_ms)
    kernels = {}
    for name, ms in (("fp", fp_avg), ("bp", bp_avg)):
        evals = units / folds[name] if units else None
        flops = evals * (FLOPS_PER_WEIGHT - 2) + units * 2 if units else None
        ach = flops / (ms * 1e-3) / 1e12 if flops else None
        per = fp_ms if name == "fp" else bp_ms
        kernels[name] = {"ms": ms, "ms_median": statistics.median(per), "ms_min": min(per), "ms_max": max(per),
                         "tflops": ach, "frac": ach / peak_tflops if ach else None,
                         "weights_per_launch": units, "weight_evaluations": evals,
                         "views_or_slices_per_evaluation": folds[name],
                         "effective_tflops_per_view_weight": units * FLOPS_PER_WEIGHT / (ms * 1e-3) / 1e12
                         if units else None}
    dom = "bp" if bp_avg >= fp_avg else "fp"
    ttab = traffic_table().get(args.config, {})
    cap = traffic_table().get("_capture", {})
    traffic = ttab.get(dom)
    eff = kernels[dom]["effective_tflops_per_view_weight"]
    step_s = statistics.mean(step_ms) * 1e-3
    alg_bytes = 2 * 4 * batch * (n * n + nv * ns)  # image + sinogram, FP and BP
    roof = {"bound": "alu", "kernel": f"cbp_{dom}_kernel", "achieved": kernels[dom]["tflops"],
            "peak": peak_tflops, "unit": "TFLOP/s", "frac": kernels[dom]["frac"],
            "traffic": traffic,
            # the three fractions of the dominant kernel, labelled
            "fractions": {
                "frac_executed_flops": {
                    "value": kernels[dom]["frac"],
                    "basis": "executed work: weight evaluations x 30 flop + view-weights x 2 flop, "
                             "over the kernel's event-timed duration, / peak (this run)"},
                "fma_pipe_util_ncu": {
                    "value": ttab.get(f"{dom}_fma_pipe"),
                    "basis": "SURVEY 8(d)(i): ncu sm__pipe_fma_cycles_active of this kernel in the "
                             "committed capture of this command",
                    "capture": cap.get("file"), "capture_head": cap.get("head")},
                "effective_view_weight_rate": {
                    "value": eff / peak_tflops if eff else None,
                    "basis": "SURVEY 8(d)(ii): nonzero view-weights x 32 flop / duration / peak -- effective, "
                             f"includes the {folds[dom]}-fold sharing of each weight evaluation "
                             "(symmetry / batch), so it can exceed 1; not a utilisation"}},
            "issue_active_ncu": ttab.get(f"{dom}_issue"),
            "peak_basis": f"{props.multi_processor_count} SMs x 128 FP32 lanes x 2 flop x "
                          f"{sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "work": f"{units} nonzero view-weights per launch ({nw} x {batch} slices), each weight "
                    f"evaluated once per {folds[dom]} views/slices (symmetry / batch): "
                    f"{kernels[dom]['weight_evaluations']:.4g} evaluations x {FLOPS_PER_WEIGHT - 2} flop"
                    f" + {units} x 2 flop accumulation" if units else None,
            "hbm_gbs_algorithmic": alg_bytes / step_s / 1e9,
            "hbm_basis": f"2 x 4 B x (n^2 + views x bins) x slices = {alg_bytes} B per step / step time"}

    # ---- end to end through the C ABI with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        h_img = torch.from_numpy(host_img).pin_memory()
        h_sino = torch.empty(sshape, dtype=torch.float32).pin_memory()
        h_out = torch.empty(bshape + (n, n), dtype=torch.float32).pin_memory()
        d_img = torch.empty_like(img)
        d_out = torch.empty(bshape + (n, n), dtype=torch.float32, device=dev)
        ke = max(3, min(args.steps, 50))
        piped = world == 1 and not args.views  # cbp_normal_stream covers all views
        if piped:  # one pinned input and output per step: at most ~512 MiB each
            ke = max(3, min(ke, (1 << 29) // max(1, host_img.nbytes)))

        def e2e_step():
            if piped:
                # cbp_normal on host buffers: the library stages H2D image, runs the
                # FP+BP pair (the sinogram stays on the device), D2H the result image
                cbp.normal(g, h_img, h_out)
            else:
                d_img.copy_(h_img, non_blocking=True)  # H2D image
                fwd(d_img, sino)
                if mm is not None:
                    h_out.copy_(back_sharded(g, sino, sh, multimem=mm, stream=stream))  # D2H image
                else:
                    bwd(sino, d_out)
                    if world > 1 and not slice_shard:
                        dist.all_reduce(d_out)
                    h_out.copy_(d_out)  # D2H image
                torch.cuda.synchronize()

        def e2e_sino_step():  # the same pair with the sinogram through host memory too
            hs = h_sino.view(nv, ns) if orbit else h_sino
            cbp.forward(g, h_img, hs, view_begin=sh.begin, view_count=sh.count)
            cbp.back(g, hs, h_out, view_begin=sh.begin)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        unpiped = None
        if piped:
            # ke DISTINCT inputs in pinned host memory (one per step: the workload's image
            # scaled by 1 + 0.01 k) through cbp_normal_stream: H2D of step i+1 and D2H of
            # step i-1 overlap step i's FP+BP on the device
            scale = (1.0 + 0.01 * np.arange(ke, dtype=np.float32)).reshape((ke,) + (1,) * host_img.ndim)
            h_imgs = torch.from_numpy(np.ascontiguousarray(host_img[None] * scale))
            h_imgs = h_imgs.pin_memory()
            h_outs = torch.empty_like(h_imgs).pin_memory()
            cbp.normal_stream(g, h_imgs[:3], h_outs[:3])  # warm-up
            torch.cuda.synchronize()
            e0.record()
            cbp.normal_stream(g, h_imgs, h_outs)
            e1.record()
            e1.synchronize()
            # A^T A is linear: step k's result is (1 + 0.01 k) x step 0's (to FP32 rounding)
            r0, rk = h_outs[0].numpy().astype(np.float64), h_outs[-1].numpy().astype(np.float64)
            if np.linalg.norm(rk - scale.ravel()[-1] * r0) > 1e-5 * np.linalg.norm(rk):
                raise RuntimeError("normal_stream: the steps' results are inconsistent")
            # informational: one synchronous cbp_normal call per step (no overlap)
            for _ in range(3):
                e2e_step()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
            for _ in range(ke):
                e2e_step()
            eb.record()
            eb.synchronize()
            unpiped = {"value": ke * total_batch / (ea.elapsed_time(eb) * 1e-3),
                       "path": "cbp_normal per step on pinned host buffers (synchronous, no overlap)"}
        else:
            for _ in range(3):
                e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0.record()
            for _ in range(ke):
                e2e_step()
            e1.record()
            e1.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": ke * total_batch / (float(et.item()) * 1e-3), "unit": "pairs/s",
               "h2d_bytes_per_step": 4 * batch * n * n,
               "d2h_bytes_per_step": 4 * batch * n * n,
               "path": f"cbp_normal_stream (A^T A) over {ke} distinct inputs in pinned host memory: the "
                       "library's copy/compute/copy pipeline (the sinogram stays on the device)" if piped
               else f"pinned H2D/D2H + {sh.mode} shards (cbp_forward_{sh.mode}/cbp_back_{sh.mode} or view "
                    f"ranges)" + ((" + multicast BP" if mm is not None else " + NCCL all_reduce")
                                   if world > 1 and not slice_shard else ""),
               "note": "a pipeline figure: steps follow each other without the L2 flush that separates the "
                       "device-timed steps of `value`, and PCIe copies overlap compute, so it can exceed "
                       "`value`" if piped else "synchronous steps"}
        if unpiped:
            e2e["unpipelined"] = unpiped
        if world == 1:  # informational: the sinogram also crosses PCIe both ways
            for _ in range(3):
                e2e_sino_step()
            e0.record()
            for _ in range(ke):
                e2e_sino_step()
            e1.record()
            e1.synchronize()
            e2e["with_host_sinogram"] = {
                "value": ke * batch / (e0.elapsed_time(e1) * 1e-3),
                "h2d_bytes_per_step": 4 * batch * (n * n + nv * ns),
                "d2h_bytes_per_step": 4 * batch * (nv * ns + n * n),
                "path": "cbp_forward then cbp_back on pinned host buffers"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, rv0, rnv)  # per slice: the oracle has no batch sharing

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": bench_config(args, g, world, sh.mode if not slice_shard else "block", slice_shard),
            "roofline": roof,
            "kernels": kernels,
            "timing": graph_note,
            "bp_reduction": reduce_note,
            "allreduce_ms": statistics.mean(ar_ms) if world > 1 else 0.0,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if backend == "gloo" and world > 1:
            line["note"] = "CBP_BENCH_BACKEND=gloo: a logic check of the N > 1 path (ranks may share a GPU), not a measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
