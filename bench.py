"""Benchmark: probe-traced Mrays/s (and frames/s) of the B200 grid tracer.

    python bench.py [--gpus N --steps K --warmup W --config c3|c1|c2|c4|c5]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # CPU reference arm (oracle port)

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU); under torchrun the world
size must equal N.

Workloads (BASELINE.json configs, seeded synthetic inputs, configs.py):
  c3 (default; BASELINE configs[2], the largest single-GPU configuration)
     8x4x8 probes 256^2/64^2 (fp16 payloads), 64 poses at 1920x1080 per
     step, 8x16 tiles interleaved over the N ranks (strong scaling), rank 0
     gathers the framebuffer over NCCL and untiles it.
  c2 4x4x4 probes 128^2/32^2, one 512x512 view per GPU per step.
     Weak scaling: the global batch has N views; its 8x16 pixel tiles are
     interleaved over the ranks, each rank traces its tiles against its own
     probe-set replica, rank 0 gathers the framebuffer over NCCL (the only
     collective) and untiles it.
  c1 the same with the 2x2x2 / 32^2 room and a 128x128 view.
  c4 3-level 128^2/32^2 hierarchy (9,344 probes), one 3840x2160 view per
     GPU per step.
  c5 the c3 probe set, 2^26 incoherent f32 rays per step split into N
     contiguous batches (strong scaling); each rank bins its rays by
     (entry cube, direction octant), sorts and traces them in bin order,
     rank 0 gathers every per-ray output (status, probe, texel, fetch, rgb,
     hit distance).
Inputs (probe set, cameras / rays) are resident in HBM before the timed
region. L2 (126 MB) is flushed between steps by a 512 MiB write outside the
timed events (the c2 probe set, 28 MB, would otherwise stay L2-resident).
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
C5_RAYS = 1 << 26

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting",
            0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
            0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def ncu_traffic(config):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)[config]["dram_bytes_per_launch"]
    except Exception:
        return None


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
        time.sleep(0.15)
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
        sm, mx, pw, reasons = [], [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                pw.append(float(r[2]))
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
                "power_w_max": max(pw) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def gpu_smi_id(torch, dev_index):
    try:
        p = torch.cuda.get_device_properties(dev_index)
        return "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id,
                                      p.pci_device_id)
    except Exception:
        return dev_index


def build_config(name, views, device=0):
    """The seeded config; GPU bakes (C3/C5 probe set, C4 hierarchy) run on
    this rank's own `device` (every rank bakes an identical replica)."""
    from paper_2507_14624_b200 import configs
    if name == "c1":
        return configs.c1()
    if name == "c2":
        return configs.c2(n_views=views)
    if name in ("c3", "c5"):
        return configs.c3(n_views=max(views, 1), device=device)
    if name == "c4":
        return configs.c4(n_views=views, device=device)
    raise SystemExit(f"unknown config {name}")


def config_record(cfg, name, world, views):
    ps = cfg.grid.probe_set
    rec = {
        "workload": f"{name.upper()}: {cfg.description}",
        "probes": int(ps.dist_hi.shape[0]),
        "res_hi": int(ps.dist_hi.shape[1]), "res_lo": int(ps.dist_lo.shape[1]),
        "l2": "flushed between steps (512 MiB write, outside timed events)",
        "seeds": "configs.py (scene/bake/camera/ray seeds fixed)",
    }
    if getattr(cfg, "levels", None):
        rec["levels"] = [{"dims": list(g.dims), "cell": g.cell_size,
                          "probes": int(g.probe_set.n_probes)} for g in cfg.levels]
        rec["probes"] = sum(l["probes"] for l in rec["levels"])
    if name == "c5":
        rec.update({"workload": "C5: incoherent-ray stress, 2^26 f32 rays "
                                "(origins U(room), directions normalised "
                                "Gaussian) against the C3 probe set",
                    "rays_per_step": C5_RAYS,
                    "parallelism": f"ray-batch sharded x{world}, per-rank "
                                   "binning by (entry cube, octant)" +
                                   (", NCCL gather to rank 0" if world > 1 else "")})
        return rec
    cam = cfg.cameras[0]
    rec.update({
        "frame": [cam.width, cam.height],
        "views_per_step": views,
        "rays_per_step": views * cam.width * cam.height,
        "parallelism": f"tile-sharded x{world} (interleaved 8x16 tiles), "
                       "probe set replicated" + (", NCCL gather to rank 0"
                                                 if world > 1 else ""),
    })
    return rec


# --------------------------------------------------------------------------
# CPU reference arm / baseline (the oracle port -- test infrastructure)
# --------------------------------------------------------------------------

# Bounded CPU samples of one step's workload (fraction of its rays):
#   c1, c2  every ray of the view (same_config holds for the reference arm)
#   c3      a seeded 1/FRAC subsample of the pixels of all 64 poses
#   c4      a seeded 1/FRAC subsample of the 4K view
#   c5      the first 2^26/FRAC rays of the bench ray set
REF_FRAC = {"c1": 1, "c2": 1, "c3": 64, "c4": 64, "c5": 256}
CPU_FRAC = {"c1": 1, "c2": 1, "c3": 256, "c4": 256, "c5": 256}
NUMBA_NOTE = ("the C port runs ~2.2x faster than the numba reference "
              "itself on the same host (C2, 8 cores: 1.03 vs 0.476 Mrays/s, "
              "identical outputs), so this baseline is conservative")


def cpu_sample(cfg, name, frac, seed=12345):
    """(origins (N, 3) f64 or eye (3,), dirs (N, 3) f64, description) of a
    bounded sample of one step's workload; directions computed in the
    reference's op order (render.py:50-62) by the oracle."""
    from oracle import oracle
    if name == "c5":
        from paper_2507_14624_b200 import configs
        o, d = configs.c5_rays(cfg.scene, C5_RAYS // frac)
        return (o.astype(np.float64), d.astype(np.float64),
                f"the first {C5_RAYS // frac} rays of the C5 ray set")
    rng = np.random.default_rng(seed)
    os_, ds_ = [], []
    for cam in cfg.cameras:
        basis, tv, th = oracle.camera_params(cam)
        dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
        if frac > 1:
            idx = np.sort(rng.choice(len(dirs), len(dirs) // frac,
                                     replace=False))
            dirs = dirs[idx]
        ds_.append(dirs)
        os_.append(np.broadcast_to(np.asarray(cam.eye, np.float64),
                                   dirs.shape))
    what = (f"every ray of {len(cfg.cameras)} view(s)" if frac == 1 else
            f"a seeded 1/{frac} pixel subsample of all {len(cfg.cameras)} "
            "view(s)")
    if len(cfg.cameras) == 1:
        return np.asarray(cfg.cameras[0].eye, np.float64), ds_[0], what
    return (np.ascontiguousarray(np.concatenate(os_)),
            np.ascontiguousarray(np.concatenate(ds_)), what)


def run_cpu(cfg, eye, dirs):
    from oracle import oracle
    t0 = time.perf_counter()
    if getattr(cfg, "levels", None):
        res = oracle.trace_hierarchy(cfg.levels, eye, dirs)
    else:
        g = cfg.grid
        res = oracle.trace_rays(g.probe_set, g.grid_origin, g.cell_size,
                                g.dims, eye, dirs)
    return time.perf_counter() - t0, res


def cpu_baseline(cfg, name, budget_s=12.0):
    """Oracle port on all host threads over repeated passes of a bounded
    sample, ~budget_s of CPU time."""
    from oracle import oracle
    threads = os.cpu_count() or 1
    oracle.set_num_threads(threads)
    eye, dirs, what = cpu_sample(cfg, name, CPU_FRAC[name])
    run_cpu(cfg, eye if eye.ndim == 1 else eye[:4096], dirs[:4096])  # warm
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
            "sample": f"{reps} pass(es) over {what} ({len(dirs)} rays/pass), "
                      f"C oracle (oracle/lfp_oracle.c, OpenMP {threads} "
                      "threads)",
            "note": NUMBA_NOTE}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = build_config(args.config, 64 if args.config == "c3" else 1)
    from oracle import oracle
    threads = os.cpu_count() or 1
    oracle.set_num_threads(threads)
    frac = REF_FRAC[args.config]
    eye, dirs, what = cpu_sample(cfg, args.config, frac)
    for _ in range(args.warmup):
        run_cpu(cfg, eye, dirs)
    times = []
    res = None
    for _ in range(args.steps):
        dt, res = run_cpu(cfg, eye, dirs)
        times.append(dt)
    t = sum(times)
    value = len(dirs) * args.steps / t / 1e6
    views = len(cfg.cameras) if args.config != "c5" else 0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.config in ("c1", "c2", "c4") else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded scene, ray-cast bake)",
        "config": config_record(cfg, args.config, 1, views) | {
            "reference_sample": f"{what} per step ({len(dirs)} rays)",
            "same_config": frac == 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port",
                         "sample": f"{len(dirs)} rays per step ({what})",
                         "note": NUMBA_NOTE},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "fetch_per_ray": float(res.fetch.mean()),
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

class Workload:
    """One step of the hot path on this rank + its algorithmic bytes."""

    def __init__(self, args, world, rank, dvc):
        import torch

        from paper_2507_14624_b200 import dist as pdist
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        self.torch, self.dev, self.pdist = torch, dev, pdist
        self.name, self.world, self.rank, self.dvc = args.config, world, rank, dvc
        name = args.config
        if name in ("c1", "c2", "c4"):
            self.views = args.views or 1
            views_total = self.views * world          # weak scaling
        elif name == "c3":
            self.views = views_total = args.views or 64   # strong scaling
        else:
            self.views = views_total = 1
        self.cfg = build_config(name, views_total, device=dvc.index)
        self.dps = device_probe_set(self.cfg.grid, dvc.index)
        self.levels = None
        if name == "c4":
            self.levels = [(device_probe_set(gr, dvc.index),
                            dev.grid_params(gr.grid_origin, gr.cell_size,
                                            gr.dims, DEFAULT_CONFIG,
                                            mode=args.mode))
                           for gr in self.cfg.levels]
        self.g = dev.grid_params(self.cfg.grid.grid_origin,
                                 self.cfg.grid.cell_size, self.cfg.grid.dims,
                                 DEFAULT_CONFIG, mode=args.mode,
                                 schedule=args.schedule,
                                 min_active=args.min_active)
        self.stream = torch.cuda.current_stream(dvc)
        self.extra_in_bytes = 0
        self.launches = 1          # our kernels per trace() call
        self.binned = False
        if name == "c5":
            from paper_2507_14624_b200 import configs
            lo, hi = pdist.ray_share(C5_RAYS, world, rank)
            o, d = configs.c5_rays(self.cfg.scene, hi - lo, start=lo)
            self.o = torch.from_numpy(o).to(dvc)
            self.d = torch.from_numpy(d).to(dvc)
            self.n_local = hi - lo
            self.max_local = (C5_RAYS + world - 1) // world
            # every per-ray output of trace_grid_ray (K:653-657) + hit_t
            self.out = dev.RayOutputs(self.max_local, dvc, probe=True,
                                      texel=True, fetch=True, hit_t=True)
            self.out.status.zero_()
            self.out.rgb.zero_()
            self.extra_in_bytes = 24
            self.rays_per_step = C5_RAYS
            self.frames_per_step = 0
            # the wavefront schedule (default at this size) sorts its rays
            # itself; binning applies to the per-ray schedules
            self.binned = (not args.no_binning and
                           args.schedule in ("nested", "persistent"))
        else:
            cams = self.cfg.cameras
            self.cams = cams
            self.W, self.H = cams[0].width, cams[0].height
            self.plan = pdist.ShardPlan(len(cams), self.W, self.H, world, rank)
            n = len(cams) * self.W * self.H
            if world == 1:
                self.out = dev.RayOutputs(n, dvc)
            else:
                self.out = dev.RayOutputs(self.plan.max_tiles * pdist.TILE_PIX, dvc)
                self.out.status.zero_()
                self.out.rgb.zero_()
            self.frame_st = self.frame_rgb = None
            if world > 1 and rank == 0:
                self.frame_st = torch.empty(n, dtype=torch.uint8, device=dvc)
                self.frame_rgb = torch.empty((n, 3), dtype=torch.float32,
                                             device=dvc)
            self.rays_per_step = n
            self.frames_per_step = len(cams)

    # -- kernels -----------------------------------------------------------
    def trace(self):
        """The traced launch(es) of one step on this rank (no collective)."""
        dev = self.dev
        if self.name == "c5":
            out = self.out
            if self.binned:
                keys = dev.bin_rays(self.g, self.o, self.d, stream=self.stream)
                order = dev.ray_order(keys)
                dev.trace_rays_ordered(self.dps, self.g, self.o, self.d, order,
                                       out, stream=self.stream)
            else:
                dev.trace_rays(self.dps, self.g, self.o, self.d, out,
                               stream=self.stream)
            self.launches = dev.last_launches()
            return
        if self.levels is not None:
            if self.world == 1:
                dev.render_hierarchy(self.levels, self.cams, self.W, self.H,
                                     self.out, stream=self.stream)
            else:
                dev.render_hierarchy(self.levels, self.cams, self.W, self.H,
                                     self.out, tile_begin=self.plan.tile_begin,
                                     tile_step=self.plan.tile_step,
                                     n_tiles=self.plan.n_tiles, compact=True,
                                     stream=self.stream)
        elif self.world == 1:
            dev.render_cameras(self.dps, self.g, self.cams, self.W, self.H,
                               self.out, stream=self.stream)
        else:
            dev.render_cameras(self.dps, self.g, self.cams, self.W, self.H,
                               self.out, tile_begin=self.plan.tile_begin,
                               tile_step=self.plan.tile_step,
                               n_tiles=self.plan.n_tiles, compact=True,
                               stream=self.stream)

    def gather(self):
        """Framebuffer (or per-ray result) gather to rank 0 + untile."""
        if self.world == 1:
            return
        pdist = self.pdist
        o = self.out
        if self.name == "c5":
            pdist.gather_rows([o.status, o.probe, o.texel, o.fetch, o.rgb,
                               o.hit_t], self.max_local)
            return
        g = pdist.gather_shards(self.plan, pdist._comm(o.status),
                                pdist._comm(o.rgb))
        if g is None:
            return
        st_all, rgb_all = (t.to(self.dvc) for t in g)
        self.dev.untile(len(self.cams), self.W, self.H, self.world, st_all,
                        rgb_all, self.frame_st, self.frame_rgb,
                        shard_stride=self.plan.max_tiles, stream=self.stream)

    def launches_per_step(self):
        if self.name == "c5":
            # bin keys + sort (library) + ordered trace, or the wavefront's
            # iterations (CUB sorts not counted); only ours counted
            return (1 if self.binned else 0) + self.launches
        return 1 + (1 if (self.world > 1 and self.rank == 0) else 0)

    def algorithmic_bytes(self):
        """Sum of B_ray = 4 F + 12 H + 16 (+24 explicit ray input) over this
        rank's rays of one launch."""
        self.out.stats.zero_()
        self.trace()
        self.torch.cuda.synchronize()
        f, m, u, h = (int(v) for v in self.out.stats.cpu())
        n = m + u + h
        return (4 * f + 12 * h + (16 + self.extra_in_bytes) * n, n, f, h)


def e2e_measure(wl, steps, world, rank, local):
    """Same metric through the public API with host buffers, H2D of the
    step's inputs and D2H of its results inside the timed region:
      N = 1: render_frame(grid, cam) per camera (the reference's call,
             render.py:102) / trace_rays(grid, origins, dirs) for C5;
      N > 1: dist.render_frames(grid, cams) / dist.trace_rays_sharded --
             per-rank trace, the gather to rank 0, untile and D2H there.
    Timed with CUDA events on the current stream, max over ranks."""
    import torch
    import torch.distributed as tdist

    import paper_2507_14624_b200 as pkg
    from paper_2507_14624_b200 import dist as pdist
    if wl.name == "c5":
        from paper_2507_14624_b200 import configs
        if world == 1:
            # the step's inputs live in page-locked host memory (contract)
            o_pin = wl.o.cpu().pin_memory()
            d_pin = wl.d.cpu().pin_memory()
            o_h, d_h = o_pin.numpy(), d_pin.numpy()
            call = lambda: pkg.trace_rays(wl.cfg.grid, o_h, d_h, device=local)  # noqa: E731
            api = ("trace_rays(ProbeGrid, origins, dirs) page-locked host f32 "
                   "arrays -> host results")
        else:
            o_h, d_h = configs.c5_rays(wl.cfg.scene, C5_RAYS)
            call = lambda: pdist.trace_rays_sharded(  # noqa: E731
                wl.cfg.grid, o_h, d_h, device=local)
            api = ("dist.trace_rays_sharded(ProbeGrid, origins, dirs): host "
                   "f32 arrays, per-rank share, gather of every per-ray "
                   "output to rank 0, D2H there")
        rays = C5_RAYS
        h2d = o_h.nbytes + d_h.nbytes
        d2h = rays * (1 + 4 * 4 + 12 + 4) + 32
    else:
        src = getattr(wl.cfg, "hierarchy", None) or wl.cfg.grid
        if world == 1:
            cams = wl.cams

            def call():
                for cam in cams:
                    pkg.render_frame(src, cam, device=local)
            api = (f"render_frame(grid, Camera) -> Frame (host arrays), "
                   f"{len(cams)} call(s) per step")
        else:
            cams = wl.cams
            call = lambda: pdist.render_frames(src, cams, device=local)  # noqa: E731
            api = (f"dist.render_frames(grid, {len(cams)} cameras) -> Frames "
                   "on rank 0: tile-sharded trace, NCCL gather, untile, D2H")
        rays = sum(c.width * c.height for c in cams)
        h2d, d2h = 104 * len(cams), 13 * rays + 32 * len(cams)
    call()
    k = max(3, min(steps, 20))
    stream = torch.cuda.current_stream(wl.dvc)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(k):
        call()
    e1.record(stream)
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3
    te = torch.tensor([dt], dtype=torch.float64)
    if world > 1:
        te = pdist._comm(te.to(wl.dvc))
        tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
    dt = float(te.item())
    return {"value": k * rays / dt / 1e6, "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": api, "call_ms": dt / k * 1e3}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3",
                    choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--views", type=int, default=0,
                    help="views per step (per GPU for c1/c2/c4, total for c3)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-binning", action="store_true",
                    help="c5: trace rays in input order")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--mode", default="filtered",
                    choices=["filtered", "exact", "check"],
                    help="trace_mode: fp32 decision filters + exact fallback "
                         "(default), exact fp64 only, or self-check")
    ap.add_argument("--schedule", default="default",
                    choices=["default", "nested", "persistent", "wave"],
                    help="traversal schedule (default: nested for cameras, "
                         "wavefront for >= 2^20 explicit rays)")
    ap.add_argument("--min-active", type=int, default=0,
                    help="persistent schedule stepping threshold (0 = 16)")
    ap.add_argument("--lib", default=None,
                    help="alternative liblfprobe_b200 build (LFP_LIB_PATH)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-logic test of the N>1 path on one GPU "
                         "(gather through host memory)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.lib:
        os.environ["LFP_LIB_PATH"] = os.path.abspath(args.lib)

    if args.impl == "reference":
        return run_reference(args)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)

    import torch
    import torch.distributed as tdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dvc = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=dvc)
        else:
            tdist.init_process_group("gloo")

    wl = Workload(args, world, rank, dvc)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dvc)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        wl.trace()
        wl.gather()
    torch.cuda.synchronize()
    alg_bytes, n_local, fetch_sum, n_hit = wl.algorithmic_bytes()

    stream = wl.stream
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
            wl.trace()
            ev[k][1].record(stream)
            wl.gather()
            ev[k][2].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
    step_ms = sum(e[0].elapsed_time(e[2]) for e in ev)
    kern_ms = sum(e[0].elapsed_time(e[1]) for e in ev)
    t = torch.tensor([step_ms, kern_ms], dtype=torch.float64)
    if world > 1:
        if args.dist_backend == "nccl":
            t = t.to(dvc)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    step_ms, kern_ms_max = (float(v) for v in t.cpu())

    value = wl.rays_per_step * args.steps / (step_ms * 1e-3) / 1e6
    kern_avg_ms = kern_ms / args.steps
    hbm, peak_kind = peaks()
    achieved = alg_bytes / (kern_avg_ms * 1e-3) / 1e9

    e2e = None if args.no_e2e else e2e_measure(wl, args.steps, world, rank,
                                               local)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl.cfg, args.config, args.cpu_budget)

    if rank == 0:
        kernel = {"c5": ("wave_kernel: all wavefront iterations of the step"
                         if wl.launches > 1 else
                         "trace_rays_kernel / persistent_kernel" +
                         (" (binned)" if wl.binned else "")),
                  "c4": "render_hierarchy_kernel"}.get(args.config,
                                                       "render_cameras_kernel")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.config in ("c1", "c2", "c4") else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded analytic scene, ray-cast probe bake, "
                    "seeded cameras / rays)",
            "config": config_record(wl.cfg, args.config, world,
                                    wl.frames_per_step),
            "frames_per_s": (wl.frames_per_step * args.steps / (step_ms * 1e-3)
                             if wl.frames_per_step else None),
            "kernel_mrays_s_per_gpu": n_local / (kern_avg_ms * 1e-3) / 1e6,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": ncu_traffic(args.config),
                         "traffic_unit": "bytes per launch (ncu, cold cache)",
                         "peak_kind": peak_kind,
                         "kernel": kernel,
                         "alg_bytes_per_launch": alg_bytes,
                         "rays_per_launch": n_local,
                         "fetch_per_ray": fetch_sum / max(n_local, 1),
                         "hit_fraction": n_hit / max(n_local, 1),
                         "avg_launch_ms": kern_avg_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": wl.launches_per_step() * args.steps,
            "clocks": clocks.summary(),
            "trace_mode": args.mode,
            "schedule": args.schedule,
            "lib": os.path.basename(os.environ.get("LFP_LIB_PATH", "")) or
                   "liblfprobe_b200.so",
        }
        if args.dist_backend != "nccl" and world > 1:
            line["dist_backend"] = args.dist_backend
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
