"""Benchmark: probe-traced Mrays/s (and frames/s) of the B200 grid tracer.

    python bench.py [--gpus N --steps K --warmup W --config c2|c1|c3]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # CPU reference arm (oracle port)

A step renders one batch of synthetic frames with the config's probe grid.
Weak scaling: every rank owns a fixed share (one config batch) of a global
batch of N config batches; the global batch's 8x16 tiles are interleaved
over the ranks, each rank traces its tiles against its own probe-set replica
and rank 0 gathers the framebuffer over NCCL (the only collective) and
untiles it. Inputs (probe set, camera parameters) are resident before the
timed region; L2 (126 MB) is flushed between steps by writing 512 MiB
outside the timed events, since the C2 probe set (28 MB) would otherwise
stay L2-resident across steps.
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

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "probe-traced Mrays/s and frames/s at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Mrays/s"

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting",
            0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
            0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.gpu_id),
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
               "clocks_event_reasons.active", "--format=csv,noheader,nounits",
               "-lms", "50"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self

        def read():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 4:
                    self.rows.append(parts)
        self.thread = threading.Thread(target=read, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread is not None:
                self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                mask = int(r[3], 16)
            except ValueError:
                continue
            for bit, name in _REASONS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def gpu_smi_id(torch, dev_index):
    try:
        p = torch.cuda.get_device_properties(dev_index)
        return "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id,
                                      p.pci_device_id)
    except Exception:
        return dev_index


def build_config(name, views):
    from paper_2507_14624_b200 import configs
    if name == "c1":
        return configs.c1()
    if name == "c2":
        return configs.c2(n_views=views)
    if name == "c3":
        return configs.c3(n_views=views)
    raise SystemExit(f"unknown config {name}")


def config_views(name):
    return {"c1": 1, "c2": 1, "c3": 64}[name]


def config_record(cfg, name, world, per_rank_views):
    cam = cfg.cameras[0]
    ps = cfg.grid.probe_set
    return {
        "workload": f"{name.upper()}: {cfg.description}",
        "probes": int(ps.dist_hi.shape[0]),
        "res_hi": int(ps.dist_hi.shape[1]), "res_lo": int(ps.dist_lo.shape[1]),
        "frame": [cam.width, cam.height],
        "views_per_gpu": per_rank_views,
        "global_views": per_rank_views * world,
        "rays_per_step": per_rank_views * world * cam.width * cam.height,
        "parallelism": f"tile-sharded x{world} (interleaved 8x16 tiles), "
                       "probe set replicated" + (", NCCL gather to rank 0"
                                                 if world > 1 else ""),
        "l2": "flushed between steps (512 MiB write, outside timed events)",
        "seeds": "configs.py (scene/bake/camera seeds fixed)",
    }


# --------------------------------------------------------------------------
# CPU reference arm / baseline (the oracle port -- test infrastructure)
# --------------------------------------------------------------------------

def cpu_sample(cfg, stride):
    """Seeded pixel subsample of the config's first view: every `stride`-th
    ray of the frame (row-major), f64 directions computed as render.py does."""
    from oracle import oracle
    cam = cfg.cameras[0]
    basis, tv, th = oracle.camera_params(cam)
    dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
    return np.asarray(cam.eye, np.float64), np.ascontiguousarray(dirs[::stride])


def run_cpu(cfg, eye, dirs, threads=None):
    from oracle import oracle
    if threads:
        oracle.set_num_threads(threads)
    g = cfg.grid
    t0 = time.perf_counter()
    res = oracle.trace_rays(g.probe_set, g.grid_origin, g.cell_size, g.dims,
                            eye, dirs)
    return time.perf_counter() - t0, res


def cpu_baseline(cfg, budget_s=12.0, stride=1):
    """Oracle port on all host threads over repeated passes of a bounded
    sample, ~budget_s of CPU time."""
    from oracle import oracle
    threads = os.cpu_count() or 1
    oracle.set_num_threads(threads)
    eye, dirs = cpu_sample(cfg, stride)
    run_cpu(cfg, eye, dirs[:4096])   # warm (page-in, thread pool)
    total_t, total_n, reps = 0.0, 0, 0
    while total_t < budget_s or reps == 0:
        dt, _ = run_cpu(cfg, eye, dirs)
        total_t += dt
        total_n += len(dirs)
        reps += 1
        if reps >= 50:
            break
    return {"value": total_n / total_t / 1e6, "unit": UNIT, "cores": threads,
            "kind": "port",
            "sample": f"{reps} pass(es) over every {stride}-th pixel of view 0 "
                      f"({len(dirs)} rays/pass), C oracle (oracle/lfp_oracle.c"
                      f", OpenMP {threads} threads)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = build_config(args.config, 1)
    from oracle import oracle
    threads = os.cpu_count() or 1
    oracle.set_num_threads(threads)
    stride = {"c1": 1, "c2": 4, "c3": 64}[args.config]
    eye, dirs = cpu_sample(cfg, stride)
    for _ in range(args.warmup):
        run_cpu(cfg, eye, dirs)
    times = []
    for _ in range(args.steps):
        dt, res = run_cpu(cfg, eye, dirs)
        times.append(dt)
    t = sum(times)
    value = len(dirs) * args.steps / t / 1e6
    cam = cfg.cameras[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded scene, ray-cast bake)",
        "config": config_record(cfg, args.config, 1, 1) | {
            "reference_sample": f"every {stride}-th pixel of one "
                                f"{cam.width}x{cam.height} view per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port",
                         "sample": f"{len(dirs)} rays per step (every "
                                   f"{stride}-th pixel of view 0)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "fetch_per_ray": float(res.fetch.mean()),
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3"])
    ap.add_argument("--views", type=int, default=0,
                    help="views per GPU per step (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--mode", default="filtered",
                    choices=["filtered", "exact", "check"],
                    help="trace_mode: fp32 decision filters + exact fallback "
                         "(default), exact fp64 only, or self-check")
    ap.add_argument("--lib", default=None,
                    help="alternative liblfprobe_b200 build (LFP_LIB_PATH)")
    args = ap.parse_args()
    if args.lib:
        os.environ["LFP_LIB_PATH"] = os.path.abspath(args.lib)
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as tdist

    from paper_2507_14624_b200 import device as dev
    from paper_2507_14624_b200 import dist as pdist
    from paper_2507_14624_b200 import render_frame
    from paper_2507_14624_b200.render import device_probe_set
    from paper_2507_14624_b200.trace import DEFAULT_CONFIG

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))

    views = args.views or config_views(args.config)
    cfg = build_config(args.config, views * world)
    cams = cfg.cameras
    W, H = cams[0].width, cams[0].height
    dps = device_probe_set(cfg.grid, local)
    g = dev.grid_params(cfg.grid.grid_origin, cfg.grid.cell_size, cfg.grid.dims,
                        DEFAULT_CONFIG, mode=args.mode)
    plan = pdist.ShardPlan(len(cams), W, H, world, rank)
    stream = torch.cuda.current_stream()
    dvc = torch.device("cuda", local)
    if world == 1:
        out = dev.RayOutputs(len(cams) * W * H, dvc)
        frame_st = frame_rgb = None
    else:
        out = dev.RayOutputs(plan.max_tiles * pdist.TILE_PIX, dvc)
        out.status.zero_()
        out.rgb.zero_()
        frame_st = torch.empty(len(cams) * W * H, dtype=torch.uint8,
                               device=dvc) if rank == 0 else None
        frame_rgb = torch.empty((len(cams) * W * H, 3), dtype=torch.float32,
                                device=dvc) if rank == 0 else None
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dvc)
    launches_per_step = 1 + (1 if (world > 1 and rank == 0) else 0)

    def step():
        if world == 1:
            dev.render_cameras(dps, g, cams, W, H, out, stream=stream)
        else:
            pdist.render_batch_sharded(dps, g, cams, W, H, plan, out,
                                       frame_st, frame_rgb, stream=stream)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()

    # per-launch algorithmic bytes: B_ray = 4 F + 12 H + 16
    out.stats.zero_()
    dev.render_cameras(dps, g, cams, W, H, out, tile_begin=plan.tile_begin,
                       tile_step=plan.tile_step, n_tiles=plan.n_tiles,
                       compact=world > 1, stream=stream)
    torch.cuda.synchronize()
    fetch_sum, n_miss, n_unk, n_hit = (int(v) for v in out.stats.cpu())
    n_local = n_miss + n_unk + n_hit
    alg_bytes = 4 * fetch_sum + 12 * n_hit + 16 * n_local

    ev = [(torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(gpu_smi_id(torch, local)) as clocks:
        for k in range(args.steps):
            flush.fill_(float(k))            # L2 flush, outside the events
            ev[k][0].record(stream)
            if world == 1:
                dev.render_cameras(dps, g, cams, W, H, out, stream=stream)
                ev[k][1].record(stream)
            else:
                dev.render_cameras(dps, g, cams, W, H, out,
                                   tile_begin=plan.tile_begin,
                                   tile_step=plan.tile_step,
                                   n_tiles=plan.n_tiles, compact=True,
                                   stream=stream)
                ev[k][1].record(stream)
                gat = pdist.gather_shards(plan, out.status, out.rgb)
                if gat is not None:
                    dev.untile(len(cams), W, H, world, gat[0], gat[1],
                               frame_st, frame_rgb,
                               shard_stride=plan.max_tiles, stream=stream)
            ev[k][2].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
    step_ms = sum(e[0].elapsed_time(e[2]) for e in ev)
    kern_ms = sum(e[0].elapsed_time(e[1]) for e in ev)
    t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dvc)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    step_ms, kern_ms_max = (float(v) for v in t.cpu())

    rays_total = len(cams) * W * H * args.steps
    value = rays_total / (step_ms * 1e-3) / 1e6
    frames_per_s = len(cams) * args.steps / (step_ms * 1e-3)
    kern_avg_ms = kern_ms / args.steps
    hbm, peak_kind = peaks()
    achieved = alg_bytes / (kern_avg_ms * 1e-3) / 1e9

    # e2e: the public API with host buffers, per rank one view per call
    e2e = None
    if not args.no_e2e:
        cam = cams[rank % len(cams)]
        for _ in range(2):
            render_frame(cfg.grid, cam, device=local)
        n_e2e = max(3, min(args.steps, 20))
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            fr = render_frame(cfg.grid, cam, device=local)
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dvc)
        if world > 1:
            tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        e2e_s = float(te.item())
        n_px = W * H
        e2e = {"value": world * n_e2e * n_px / e2e_s / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": 104,
               "d2h_bytes_per_step": n_px * 12 + n_px + 32,
               "api": "render_frame(ProbeGrid, Camera) -> Frame (host arrays)",
               "frame_ms": e2e_s / n_e2e * 1e3}
        del fr

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        stride = {"c1": 1, "c2": 1, "c3": 16}[args.config]
        cpu = cpu_baseline(cfg, args.cpu_budget, stride)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded analytic room, ray-cast probe bake, "
                    "seeded cameras)",
            "config": config_record(cfg, args.config, world, views),
            "frames_per_s": frames_per_s,
            "kernel_mrays_s": len(cams) * W * H / world / (kern_avg_ms * 1e-3)
                              / 1e6,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "peak_kind": peak_kind,
                         "kernel": "render_cameras_kernel",
                         "alg_bytes_per_launch": alg_bytes,
                         "rays_per_launch": n_local,
                         "fetch_per_ray": fetch_sum / max(n_local, 1),
                         "hit_fraction": n_hit / max(n_local, 1),
                         "avg_launch_ms": kern_avg_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "trace_mode": args.mode,
            "lib": os.path.basename(os.environ.get("LFP_LIB_PATH", "")) or
                   "liblfprobe_b200.so",
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
