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
    return ap.parse_args()


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
def run_reference(args, rank, world):
    """The FP64 CPU oracle as it stands, on a bounded view sample per step."""
    if rank != 0:
        return
    import oracle as O
    g = W.geometry(args.config)
    img = W.shepp_logan(g["n"]).astype(np.float64)
    cores = os.cpu_count() or 1
    O.build()
    # size each step so the whole run takes about a minute; at least one view
    # per core (the oracle's FP is parallel over views)
    probe = min(g["n_views"], max(8, cores))
    t0 = time.perf_counter()
    y = O.forward(g, img, view_begin=0, view_count=probe, threads=cores)
    O.back(g, y, view_begin=0, threads=cores)
    per_view = (time.perf_counter() - t0) / probe
    budget = 60.0 / max(1, args.steps + args.warmup)
    nvs = int(max(min(g["n_views"], cores), min(g["n_views"], budget / max(per_view, 1e-6))))
    times = []
    for k in range(args.warmup + args.steps):
        v0 = (k * 37) % (g["n_views"] - nvs + 1)
        t0 = time.perf_counter()
        y = O.forward(g, img, view_begin=v0, view_count=nvs, threads=cores)
        O.back(g, y, view_begin=v0, threads=cores)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    t_pair = sum(times) / len(times) * g["n_views"] / nvs  # extrapolated full pair
    value = 1.0 / t_pair
    sample = (f"{nvs} of {g['n_views']} views per step (FP+BP, views rotated), "
              f"extrapolated x{g['n_views'] / nvs:.1f} to one pair")
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_pair * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "n": g["n"], "n_views": g["n_views"],
                   "n_det": g["n_det"], "parallelism": "cpu-openmp"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg: str, target_s: float = 12.0):
    """oracle FP+BP on a bounded view sample of the same workload (rank 0, N=1)."""
    import oracle as O
    g = W.geometry(cfg)
    img = W.shepp_logan(g["n"]).astype(np.float64)
    cores = os.cpu_count() or 1
    O.build()
    probe = min(g["n_views"], max(8, cores))
    t0 = time.perf_counter()
    y = O.forward(g, img, view_begin=0, view_count=probe, threads=cores)
    O.back(g, y, view_begin=0, threads=cores)
    per_view = (time.perf_counter() - t0) / probe
    nvs = int(max(probe, min(g["n_views"], target_s / max(per_view, 1e-6))))
    t0 = time.perf_counter()
    y = O.forward(g, img, view_begin=0, view_count=nvs, threads=cores)
    O.back(g, y, view_begin=0, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": nvs / (dt * g["n_views"]), "unit": "pairs/s", "cores": cores,
            "kind": "oracle",
            "sample": f"FP+BP over views 0..{nvs - 1} of {g['n_views']} ({dt:.1f} s wall), "
                      f"scaled to one full pair"}


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
    from paper_1907_10526_b200.sharded import make_shard, view_shard

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
    batch = W.BATCH[args.config]
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
    else:
        sh = make_shard(g["n_views"], rank, world, batch, dihedral=True)
    views = sh.views()
    nv = len(views)
    orbit = sh.mode == "orbit"
    dihedral = sh.mode == "dihedral"

    host_img = W.shepp_logan(n) if total_batch == 1 else W.jittered_batch(n, total_batch, seed=7)[s0:s0 + batch]
    img = torch.from_numpy(np.ascontiguousarray(host_img)).to(dev)
    bshape = () if total_batch == 1 else (batch,)
    sshape = (4, sh.count, ns) if orbit else ((g["n_views"], ns) if dihedral else bshape + (nv, ns))
    sino = torch.zeros(sshape, dtype=torch.float32, device=dev)
    out = torch.empty(bshape + (n, n), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

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

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        fwd(img, sino)
        if ev:
            ev[1].record(stream)
        bwd(sino, out)
        if ev:
            ev[2].record(stream)
        if world > 1 and not slice_shard:
            dist.all_reduce(out)
        if ev:
            ev[3].record(stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()

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
    launches = cbp.launch_count() - launches0
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
        kernels[name] = {"ms": ms, "tflops": ach, "frac": ach / peak_tflops if ach else None,
                         "weights_per_launch": units, "weight_evaluations": evals,
                         "views_or_slices_per_evaluation": folds[name],
                         "effective_tflops_per_view_weight": units * FLOPS_PER_WEIGHT / (ms * 1e-3) / 1e12
                         if units else None}
    dom = "bp" if bp_avg >= fp_avg else "fp"
    ttab = traffic_table().get(args.config, {})
    traffic = ttab.get(dom)
    roof = {"bound": "alu", "kernel": f"cbp_{dom}_kernel", "achieved": kernels[dom]["tflops"],
            "peak": peak_tflops, "unit": "TFLOP/s", "frac": kernels[dom]["frac"],
            "traffic": traffic,
            # the FP32 (FMA) pipe utilisation ncu measured for this kernel in the
            # committed capture of this command (profiles/traffic.json), and its issue-slot use
            "fma_pipe_util_ncu": ttab.get(f"{dom}_fma_pipe"),
            "issue_active_ncu": ttab.get(f"{dom}_issue"),
            "peak_basis": f"{props.multi_processor_count} SMs x 128 FP32 lanes x 2 flop x "
                          f"{sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "work": f"{units} nonzero view-weights per launch ({nw} x {batch} slices), each weight "
                    f"evaluated once per {folds[dom]} views/slices (symmetry / batch): "
                    f"{kernels[dom]['weight_evaluations']:.4g} evaluations x {FLOPS_PER_WEIGHT - 2} flop"
                    f" + {units} x 2 flop accumulation" if units else None,
            "hbm_gbs_algorithmic": 4 * batch * (n * n + nv * ns) / (ms_to_s(statistics.mean(step_ms))) / 1e9}

    # ---- end to end through the C ABI with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        h_img = torch.from_numpy(host_img).pin_memory()
        h_sino = torch.empty(sshape, dtype=torch.float32).pin_memory()
        h_out = torch.empty(bshape + (n, n), dtype=torch.float32).pin_memory()
        d_img = torch.empty_like(img)
        d_out = torch.empty(bshape + (n, n), dtype=torch.float32, device=dev)
        ke = max(3, min(args.steps, 50))
        if world == 1:  # one pinned input and output per step: at most ~512 MiB each
            ke = max(3, min(ke, (1 << 29) // max(1, host_img.nbytes)))

        def e2e_step():
            if world == 1:
                # cbp_normal on host buffers: the library stages H2D image, runs the
                # FP+BP pair (the sinogram stays on the device), D2H the result image
                cbp.normal(g, h_img, h_out)
            else:
                d_img.copy_(h_img, non_blocking=True)  # H2D image
                fwd(d_img, sino)
                bwd(sino, d_out)
                if not slice_shard:
                    dist.all_reduce(d_out)
                h_out.copy_(d_out)  # D2H image
                torch.cuda.synchronize()

        def e2e_sino_step():  # the same pair with the sinogram through host memory too
            cbp.forward(g, h_img, h_sino.view(nv, ns) if orbit else h_sino)
            cbp.back(g, h_sino.view(nv, ns) if orbit else h_sino, h_out)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        unpiped = None
        if world == 1:
            # ke inputs in pinned host memory (one per step) through cbp_normal_stream:
            # H2D of step i+1 and D2H of step i-1 overlap step i's FP+BP on the device
            h_imgs = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(host_img, (ke,) + host_img.shape)))
            h_imgs = h_imgs.pin_memory()
            h_outs = torch.empty_like(h_imgs).pin_memory()
            cbp.normal_stream(g, h_imgs[:3], h_outs[:3])  # warm-up
            torch.cuda.synchronize()
            e0.record()
            cbp.normal_stream(g, h_imgs, h_outs)
            e1.record()
            e1.synchronize()
            if not np.array_equal(h_outs[-1].numpy(), h_outs[0].numpy()):
                raise RuntimeError("normal_stream: the steps' results differ")
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
               "path": f"cbp_normal_stream (A^T A) over {ke} steps' inputs in pinned host memory: the "
                       "library's copy/compute/copy pipeline (the sinogram stays on the device; L2 is not "
                       "flushed between these steps, unlike `value`)" if world == 1
               else f"pinned H2D/D2H + {sh.mode} shards (cbp_forward_{sh.mode}/cbp_back_{sh.mode} or view "
                    f"ranges) + NCCL all_reduce"}
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
        cpu = cpu_baseline(args.config)  # per slice: the oracle has no batch sharing

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "n": n, "n_views": g["n_views"],
                       "n_det": ns, "pixel_mm": g["pixel"], "det_pitch_mm": g["det_pitch"],
                       "sid_mm": g["sid"], "sdd_mm": g["sdd"], "batch": total_batch,
                       "parallelism": (f"slices/{world}" if slice_shard else
                                       (f"views/{world}" if world > 1 else "single"))
                       + (" (4-fold rotational symmetry)" if orbit else "")
                       + (" (8-fold dihedral symmetry)" if dihedral else ""),
                       "l2": "flushed between steps (256 MiB write, outside the timed events)"},
            "roofline": roof,
            "kernels": kernels,
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


def ms_to_s(ms: float) -> float:
    return ms * 1e-3


if __name__ == "__main__":
    main()
