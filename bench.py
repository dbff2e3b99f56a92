#!/usr/bin/env python
"""CSFD SLAM frame-derivatives/s at 640x480 (BASELINE.json metric).

Workload (N=1, default --workload config2): BASELINE config 2 — 100 VGA depth frames of the seeded
procedural room (synthetic stand-in for TUM-style sequences, rendered on the
device by the harness; not timed), hashed 8^3-block TSDF at 5 mm voxels with
2^20 buckets, 10 CSFD directions (6 first-frame twist + 4 intrinsics),
objective = accumulated trajectory error.  One step = one full CSFD run over
all frames (volume reset, frame 0 fused at exp(xi0*)T0, frames 1..99 tracked
with the lifted 3-level ICP and fused).  Units = frames x directions.

  value       device-resident inputs, CUDA events on the library stream
  e2e         the public API call Pipeline.run_host() from pinned host
              frames: H2D of the step's frames + D2H of the gradient inside
              the timed region
  roofline    dominant kernel category, algorithmic bytes per launch /
              average launch time (CUDA events on the launching stream)
  cpu_baseline the CPU oracle (oracle/, a restatement of the reference,
              which cannot be built here) on a bounded sample, rank 0 only

Multi-GPU (torchrun): the 10 directions are sharded in contiguous blocks
(paper_2405_02187_b200/shard.py); each rank recomputes the shared real
pipeline; the derivative columns are all-gathered over NCCL.  Total work is
fixed, so scaling is "strong".  --impl reference times the CPU oracle port
(the reference's own CPU path restated) on a bounded sample of the same
workload.

--workload config5: BASELINE config 5 — the config-2 scene fused into a
hashed TSDF (100 VGA frames at the ground-truth poses, untimed setup), then
256 candidate views (seeded, free space) each raycast at 320x240 with the
pose lifted on its 6 twist channels, scored by the builder-defined coverage
objective.  Units = views x 6 directions (1536 per step).

--workload config4: BASELINE config 4 — 500 VGA frames over a 60x60 m
procedural terrain with 200 boxes (seed 3), hashed 2 cm voxels; 64
directions = 6 first-frame twist + 4 intrinsics + 6 x 9 keyframe twists
(keyframes every 50 frames).  The job is 8 directions per GPU at 8 GPUs:
each rank runs its 8-direction share (rank r of the 8-way split), so the
per-GPU work is fixed ("weak"); units = frames x directions over all ranks.

--workload reloc: camera relocalization on the config-2
scene — 8 queries, eta-switched Newton; relocalizations/s (bench_reloc.py).

--workload surfel: the surfel (X-EF) front end — 100 VGA
frames fused at poses lifted on 6 twist directions (bench_surfel.py).

--workload config1: BASELINE config 1 — the toy room (3 spheres, seed 0), 10
frames at 160x120 (fx = fy = 120), dense 128^3 TSDF at 2 cm (mu 6 cm),
3-level ICP 10/5/4, h = 1e-20, gradient of the final translation error
w.r.t. the 6 first-frame twist parameters.  Units = frames x 6 directions.

--workload config3: BASELINE config 3 — the same VGA scene, 30 frames, the
full 10x10 Hessian as 55 second-order parameter pairs (one reference
Bicomplex per pair, packed as channel slots of one evaluation).  Units =
frames x pairs; the pairs are sharded across ranks like directions.

`value` is timed without per-kernel events; a second, profiled pass of the
same steps (CUDA events around every kernel category on the library stream)
gives the per-kernel split and the rooflines.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CSFD SLAM frame-derivatives/sec at 640×480 (frames×directions/s), 1/2/4/8 GPU"
UNIT = "frame-derivatives/s"
DIRS = list(range(10))  # 6 first-frame twist components (rho, phi) + fx, fy, cx, cy
PAIRS = [(i, j) for i in range(10) for j in range(i, 10)]  # 55 Hessian pairs (config 3)
DIRS1 = list(range(6))  # config 1: the 6 first-frame twist parameters
DIRS4 = list(range(64))  # config 4: 0-5 first-frame twist, 6-9 intrinsics, 10-63 keyframes 1-9 (every 50 frames)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=["config1", "config2", "config3", "config4", "config5", "reloc", "surfel"], default="config2")
    ap.add_argument("--frames", type=int, default=0, help="0 = the workload's frame count (100 / 30)")
    ap.add_argument("--cpu-frames", type=int, default=CPU_FRAMES, help="CPU-baseline sample: frames")
    ap.add_argument("--cpu-dirs", type=int, default=CPU_UNITS, help="CPU-baseline sample: directions (one pass each)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-json", default="")
    return ap.parse_args()


# The descriptors below are plain ctypes structs (make_pipeline_cfg is pure
# Python); `icp` defaults to the product's csf_default_icp_cfg, and the CPU
# legs pass the oracle's copy of the reference defaults instead, so
# --impl reference never loads the product library.
def pipeline_cfg1(csf, capi, k, dirs, n_frames, icp=None):
    """BASELINE config 1: dense 128^3 at 2 cm (origin keeps the 4x4x3 m room
    inside), mu = 6 cm, h = 1e-20, final-translation-error objective."""
    import ctypes as C
    dense = capi.VolumeParams((C.c_int * 3)(128, 128, 128), 0.02, (C.c_double * 3)(-2.1, -1.28, -0.1), 0.06, 128.0)
    return csf.make_pipeline_cfg(hashed=False, k=k, dirs=dirs, h=1e-20,
                                 objective=capi.OBJECTIVE_FINAL_TRANSLATION_ERROR, max_frames=n_frames, dense=dense,
                                 icp=icp)


def pipeline_cfg4(csf, capi, k, dirs, n_frames, keyframe_interval=50, icp=None):
    import ctypes as C
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 5 * 0.02, 128.0, 20, 1 << 21)
    return csf.make_pipeline_cfg(hashed=True, k=k, dirs=dirs, h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                 max_frames=n_frames, hash_params=hp, keyframe_interval=keyframe_interval, icp=icp)


def pipeline_cfg(csf, capi, k, dirs, n_frames, pairs=None, icp=None):
    import ctypes as C
    # block pool: config 2 allocates ~68k blocks over 100 frames; second-order
    # voxels carry 3 slots per pair, so the pool is sized to the 30-frame run
    max_blocks = (1 << 18) if pairs is None else (1 << 16)
    hp = capi.HashParams(0.005, (C.c_double * 3)(0.0, 0.0, 0.0), 5 * 0.005, 128.0, 20, max_blocks)
    return csf.make_pipeline_cfg(hashed=True, k=k, dirs=[] if pairs is not None else dirs, h=1e-8,
                                 objective=capi.OBJECTIVE_TRAJECTORY_ERROR, max_frames=n_frames, hash_params=hp,
                                 pairs=pairs, icp=icp)


def reference_icp():
    """The reference's tracker defaults (icp.hpp:33-53) from the oracle, with
    the lifted pipeline's linearized solver — no product library call."""
    from oracle import orc
    from paper_2405_02187_b200 import capi
    return orc.default_icp_cfg(solver=capi.SOLVER_LINEARIZED)


# The bounded CPU sample shared by the GPU arm's cpu_baseline and by
# --impl reference: the workload's first CPU_FRAMES frames x CPU_UNITS
# directions (pairs for config 3), one oracle pass per direction — the
# reference's own pattern (diff.hpp:46-72).
CPU_FRAMES, CPU_UNITS = 3, 2


class Clocks:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait(timeout=10)
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1].split()[0]))
                mx = float(r[2].split()[0])
                for n, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(n)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def synth_rgb(depth):
    """uint8 colour frames [n][h][w][3] for the RGB-D ingest (configs 2-3):
    a seeded albedo texture (seed 1, the scene's seed) shaded by the rendered
    depth; invalid pixels black."""
    rng = np.random.default_rng(1)
    albedo = rng.integers(64, 256, size=(1,) + depth.shape[1:] + (3,), dtype=np.int32)
    shade = np.clip(255.0 / (1.0 + depth), 0, 255).astype(np.int32)[..., None]
    return np.where(depth[..., None] > 0, (albedo * shade) >> 8, 0).astype(np.uint8)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_record(cat, workload):
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(workload, {}).get(cat)
    except Exception:
        return None


def traffic_for(cat, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the
    category's kernel from the committed ncu --set full capture
    (profiles/traffic.json, written by tools/ncu_traffic.py), or None."""
    r = _ncu_record(cat, workload)
    return r.get("dram_bytes") if isinstance(r, dict) else r


def fp64_peak():
    """The FP64 pipe peak measured on this pool (tools/fp64_peak.cu, committed
    under profiles/): (TFLOP/s with FMA, source)."""
    for p in sorted((ROOT / "profiles").glob("*fp64_peak.json"), reverse=True):
        try:
            return float(json.loads(p.read_text())["fp64_tflops_fma"]), f"measured ({p.name})"
        except Exception:
            continue
    return None, "not measured"


def fp64_roofline(cat, workload):
    """FP64 throughput of the category's captured launch (ncu thread-instruction
    counts / ncu duration) against the measured FP64 peak."""
    r = _ncu_record(cat, workload)
    if not isinstance(r, dict) or not r.get("duration_s"):
        return None
    peak, src = fp64_peak()
    ach = r["fp64_flops"] / r["duration_s"] / 1e12
    return {"achieved_tflops": ach, "peak_tflops": peak, "frac": ach / peak if peak else None,
            "pipe_active_pct": r.get("fp64_pipe_active_pct"), "peak_source": src,
            "source": "one level-0 launch under ncu (profiles/traffic.json): 2 dfma + dadd + dmul per duration"}


def cpu_sample(depth, gt, k, frames, units, workload, packed=False):
    """One run of the CPU sample: seconds for `units` one-pass-per-direction
    oracle runs over the first `frames` frames (packed=True: one Lifted<10>
    pass over all 10 directions instead, a labelled variant)."""
    from oracle import orc
    import paper_2405_02187_b200 as csf
    from paper_2405_02187_b200 import capi
    icp = reference_icp()
    secs = 0.0
    if packed:
        cfg = pipeline_cfg(csf, capi, k, DIRS, frames, icp=icp)
        return orc.pipeline_run(cfg, depth[:frames], gt[:frames])[-1]
    for d in range(units):
        if workload == "config3":
            cfg = pipeline_cfg(csf, capi, k, [], frames, pairs=[PAIRS[d]], icp=icp)
            secs += orc.pipeline_hessian(cfg, depth[:frames], gt[:frames])[-1]
        elif workload == "config4":
            cfg = pipeline_cfg4(csf, capi, k, [DIRS4[d]], frames, icp=icp)
            secs += orc.pipeline_run(cfg, depth[:frames], gt[:frames])[-1]
        elif workload == "config1":
            cfg = pipeline_cfg1(csf, capi, k, [DIRS1[d]], frames, icp=icp)
            secs += orc.pipeline_run(cfg, depth[:frames], gt[:frames])[-1]
        else:
            cfg = pipeline_cfg(csf, capi, k, [DIRS[d]], frames, icp=icp)
            secs += orc.pipeline_run(cfg, depth[:frames], gt[:frames])[-1]
    return secs


def cpu_baseline(depth, gt, k, frames, ndirs, workload="config2"):
    """Oracle port, one Complex-style pass per direction (the reference's
    pattern, diff.hpp:46-56) or one Bicomplex pass per pair (diff.hpp:58-72),
    all host threads (OpenMP); plus, labelled, the packed Lifted<10> CPU pass
    (config 2) and a single-core number."""
    secs = cpu_sample(depth, gt, k, frames, ndirs, workload)
    units = frames * ndirs
    cores = os.cpu_count() or 1
    omp = os.environ.get("OMP_NUM_THREADS")
    if omp:
        cores = int(omp)
    what = "pair" if workload == "config3" else "direction"
    out = {"value": units / secs, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{workload} first {frames} VGA frames x {ndirs} {what}s, one pass per {what} "
                     f"({units} units in {secs:.2f} s)", "host": host_info()}
    if workload == "config2":
        ps = cpu_sample(depth, gt, k, frames, ndirs, workload, packed=True)
        out["packed_cpu"] = {"value": frames * len(DIRS) / ps, "unit": UNIT, "cores": cores,
                             "sample": f"first {frames} frames x {len(DIRS)} directions in ONE Lifted<10> oracle pass "
                                       f"({ps:.2f} s; the builder's packed CPU variant, not the reference's pattern)"}
    # also a single-core number (the same oracle on one OpenMP thread, 2 frames x 1 unit)
    try:
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(1)
        f1 = min(2, frames)
        t1 = cpu_sample(depth, gt, k, f1, 1, workload)
        gomp.omp_set_num_threads(cores)
        out["single_core"] = {"value": f1 / t1, "unit": UNIT, "cores": 1,
                              "sample": f"first {f1} frames x 1 {what}, OMP 1 thread ({t1:.2f} s)"}
    except Exception as e:  # pragma: no cover
        out["single_core"] = {"value": None, "error": str(e)}
    return out


def host_info() -> dict:
    """nproc, OMP_NUM_THREADS and the CPU model string."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS"), "cpu_model": model}


def run_reference(args):
    """--impl reference: the CPU oracle port on the box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2405_02187_b200 as csf
    from oracle import orc
    from paper_2405_02187_b200 import capi
    if args.workload == "config5":
        # bounded sample: a volume fused from 10 VGA frames (untimed), 2 views x 6 directions per step
        nf = 10
        depth, gt, k = orc.workload(2, nf)
        hp = capi.HashParams(0.005, (__import__("ctypes").c_double * 3)(0, 0, 0), 0.025, 128.0, 20, 1 << 18)
        vo = orc.Volume(hp, 6, True)
        intr = np.zeros((4, 7))
        intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
        for f in range(nf):
            pose = np.zeros((12, 7))
            pose[:, 0] = gt[f]
            vo.surface_update(depth[f].astype(np.float64), pose, intr)
        views = csf.config5_views(256, seed=4)[:2]
        kv = csf.intrinsics(k.fx / 2, k.fy / 2, k.cx / 2, k.cy / 2, 320, 240)
        for _ in range(args.warmup):
            vo.view_scores(views, kv)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            vo.view_scores(views, kv)
        secs = time.perf_counter() - t0
        value = len(views) * 6 * args.steps / secs
        cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded procedural room, BASELINE config 5 shapes)",
            "config": {"workload": "config5 bounded CPU sample: 2 views x 6 directions per step (320x240)",
                       "views": 2, "directions": 6},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": "2 views x 6 directions per step, one Lifted<6> pass per view"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
        return
    frames, units = CPU_FRAMES, CPU_UNITS
    depth, gt, k = orc.workload({"config4": 4, "config1": 1}.get(args.workload, 2), frames)
    second = args.workload == "config3"
    for _ in range(args.warmup):
        cpu_sample(depth, gt, k, frames, units, args.workload)
    secs = 0.0
    for _ in range(args.steps):
        secs += cpu_sample(depth, gt, k, frames, units, args.workload)
    value = frames * units * args.steps / secs
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    what = "pair (Bicomplex pass)" if second else "direction"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded procedural room, BASELINE {args.workload} shapes)",
        "config": {"workload": f"{args.workload} {'160x120 dense' if args.workload == 'config1' else 'VGA hashed'}, "
                               f"bounded CPU sample: first {frames} frames x {units} {what}s per step",
                   "frames": frames, "directions": units},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"first {frames} VGA frames x {units} {what}s per step, one oracle pass per {what} "
                                   "(oracle/ restatement; the reference needs Eigen/libpng/doctest, absent); the same "
                                   "sample as the GPU arm's cpu_baseline", "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.workload == "config2":
        ps = cpu_sample(depth, gt, k, frames, units, args.workload, packed=True)
        line["packed_cpu"] = {"value": frames * len(DIRS) / ps, "unit": UNIT, "cores": cores,
                              "sample": f"first {frames} frames x {len(DIRS)} directions in one Lifted<10> pass "
                                        f"({ps:.2f} s; builder's packed CPU variant, labelled, not the value)"}
    print(json.dumps(line), flush=True)


def algorithmic_bytes_per_step(cat, stats, D, W, H, n_frames):
    """Algorithmic HBM bytes of one kernel category over one step.

    stats[f] = (iterations, correspondences, converged, blocks, visible blocks, new blocks, ...)."""
    P = W * H
    P_tot = P + P // 4 + P // 16            # three pyramid levels
    vis_vox = float(stats[:n_frames, 4].sum()) * 512
    tracked = max(n_frames - 1, 0)
    if cat == "integrate":
        fused = float(stats[:n_frames, 6].sum())
        return fused * 2 * (16 + 8 * D) + n_frames * 8 * P, \
            "sum over frames of fused voxels x 2 x (16 + 8D) B (read+write F.re,W and D channels) + depth"
    if cat == "raycast":
        # each visible voxel's (F.re, W) read once per level + real maps/hits written
        return 3 * vis_vox * 16 * tracked / max(n_frames, 1) + tracked * P_tot * (6 * 8 + 16), \
            "3 levels x visible voxels x 16 B (F.re, W) + real vertex/normal maps and hit alphas written"
    if cat == "raycast_lift":
        # per pixel: the lifted vertex/normal written (48 (1+D) B) and the hit
        # record read (32 B); per hit pixel one trilinear cell of channel data
        # (8 voxels x 8D B) — its other samples' cells are the neighbours'
        # (L2 reuse).  Hits ~ the frame's correspondences' share of pixels.
        hit_frac = float(stats[1:n_frames, 1].mean()) / (P / 4) if n_frames > 1 else 0.5
        hit_frac = min(max(hit_frac, 0.0), 1.0)
        return tracked * P_tot * (6 * 8 * (1 + D) + 32 + hit_frac * 8 * 8 * D), \
            "per pixel: lifted vertex/normal written 48(1+D) B + hit record 32 B; per hit pixel one " \
            "trilinear cell of channels 64D B (hit fraction from the level-0 correspondence count)"
    if cat == "icp":
        its = float(stats[1:n_frames, 0].sum())
        corr = float(stats[1:n_frames, 1].mean()) if n_frames > 1 else 0.0
        per_it = corr * 6 * 8 * (1 + D) + 148 * 27 * (1 + D) * 8 * 2
        per_level = (P // 4) * 3 * 8  # the level's measured depth (3 taps per slot), read once per level launch
        return its * per_it + 3 * tracked * per_level, \
            "per taken iteration: model vertex/normal (1+D channels) per correspondence + 148 tile partials " \
            "written and read; per level launch the measured depth once"
    if cat == "bilateral":
        return tracked * (4 + 8 + 8) * P, "float32 depth in, raw + filtered float64 out"
    return None, None


def run_config5(args):
    """BASELINE config 5: view scoring over a fused config-2 volume."""
    import torch
    import paper_2405_02187_b200 as csf
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    ctx = csf.Context(local)
    n_frames = 100
    depth, gt, k = csf.synth_workload(2, n_frames, ctx=ctx)
    vol = csf.HashedVolume(0.005, (0.0, 0.0, 0.0), 0.025, 128.0, 20, 1 << 18, channels=6, ctx=ctx)
    intr = np.zeros((4, 7))
    intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    for f in range(n_frames):
        pose = np.zeros((12, 7))
        pose[:, 0] = gt[f]
        vol.surface_update(depth[f].astype(np.float64), pose, intr)
    views_all = csf.config5_views(256, seed=4)
    from paper_2405_02187_b200.shard import shard_directions
    _, mine = shard_directions(list(range(len(views_all))), world, rank)
    views = views_all[mine]
    kv = csf.intrinsics(k.fx / 2, k.fy / 2, k.cx / 2, k.cy / 2, 320, 240)
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(max(args.warmup, 0)):
        vol.view_scores(views, kv)
    ctx.synchronize()
    clocks = Clocks(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        sc, g = vol.view_scores(views, kv)
    e1.record(stream)
    ctx.synchronize()
    t_e2e = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count - l0
    clk = clocks.stop()
    ctx.profile(True)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        vol.view_scores(views, kv)
    p1.record(stream)
    ctx.synchronize()
    prof_ms = p0.elapsed_time(p1)
    prof = ctx.profile_read()
    ctx.profile(False)
    if dist is not None:
        t = torch.tensor([ms, t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, t_e2e = float(t[0].item()), float(t[1].item())
    units = len(views_all) * 6
    value = units * args.steps / (ms / 1000.0)
    peak, peak_src = measured_peak()
    P = 320 * 240
    rooflines = {}
    for cat, (cat_ms, cat_n) in prof.items():
        if cat_n == 0 or cat_ms <= 0:
            continue
        if cat == "raycast":
            b, bd = P * (16 + 6 * 8 + 3 * 8), "per ray: hit alphas + real vertex/normal maps written (samples are L2 gathers)"
        elif cat == "raycast_lift":
            b, bd = P * 6 * 8 * 7, "per pixel: lifted vertex/normal maps written (7 channels)"
        elif cat == "misc":
            b, bd = P * (6 * 8 * 7 + 7 * 8), "per pixel: lifted vertex + normal read, 7 term slots written"
        else:
            continue
        avg = cat_ms / cat_n
        ach = b / (avg / 1000.0) / 1e9
        rooflines[cat] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                          "traffic": traffic_for(cat, "config5"), "kernel": cat, "avg_launch_ms": avg,
                          "launches": cat_n, "share_of_step": cat_ms / prof_ms, "algorithmic_bytes_per_launch": b,
                          "bytes_model": bd, "peak_source": peak_src}
    roofline = max(rooflines.values(), key=lambda r: r["share_of_step"]) if rooflines else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded procedural room; BASELINE config 5 shapes)",
        "config": {"workload": "config5: 256 candidate views x 6 twist directions, 320x240 lifted raycast each, "
                               "over the config-2 scene fused at 5 mm (hashed)", "views": len(views_all),
                   "views_per_rank": len(views), "directions": 6, "order": 1,
                   "parallelism": f"views sharded x{world}", "l2": "hashed volume (GBs) >> L2"},
        "e2e": {"value": units * args.steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(views.nbytes),
                "d2h_bytes_per_step": int(len(views) * 7 * 8)},
        "gpu_launches": int(launches), "roofline": roofline, "roofline_by_kernel": rooflines, "clocks": clk,
        "kernel_ms_per_step": {c: v[0] / args.steps for c, v in prof.items()},
        "profiled_ms_per_step": prof_ms / args.steps,
        "scores_head": [float(x) for x in sc[:4]], "grad_head": [float(x) for x in g[0]],
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import orc
            hp = __import__("paper_2405_02187_b200").capi.HashParams(0.005, (__import__("ctypes").c_double * 3)(0, 0, 0),
                                                                     0.025, 128.0, 20, 1 << 18)
            vo = orc.Volume(hp, 6, True)
            for f in range(n_frames):
                pose = np.zeros((12, 7))
                pose[:, 0] = gt[f]
                vo.surface_update(depth[f].astype(np.float64), pose, intr)
            t1 = time.perf_counter()
            nv = 4
            vo.view_scores(views_all[:nv], kv)
            secs = time.perf_counter() - t1
            cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
            line["cpu_baseline"] = {"value": nv * 6 / secs, "unit": UNIT, "cores": cores, "kind": "port",
                                    "sample": f"{nv} views x 6 directions, one Lifted<6> pass per view "
                                              f"({nv * 6} units in {secs:.2f} s; volume fusion not timed)"}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.workload == "surfel":
        import bench_surfel
        if args.impl == "reference":
            bench_surfel.run_reference(args)
        else:
            bench_surfel.run(args, measured_peak, Clocks)
        return
    if args.workload == "reloc":
        import bench_reloc
        if args.impl == "reference":
            bench_reloc.run_reference(args)
        else:
            bench_reloc.run(args, measured_peak, Clocks)
        return
    if args.workload == "config5" and args.impl != "reference":
        run_config5(args)
        return
    second = args.workload == "config3"
    four = args.workload == "config4"
    one = args.workload == "config1"
    if args.frames <= 0:
        args.frames = 30 if second else (500 if four else (10 if one else 100))
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import paper_2405_02187_b200 as csf
    from paper_2405_02187_b200.shard import attach_native_comm, gather_columns_native, shard_directions

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_2405_02187_b200 import capi
    ctx = csf.Context(local)
    n = args.frames
    depth, gt, k = csf.synth_workload(4 if four else (1 if one else 2), n, ctx=ctx)
    if one:
        units_all = DIRS1
        off, mine = shard_directions(units_all, world, rank)
        cfg = pipeline_cfg1(csf, capi, k, mine, n)
    elif four:
        # weak scaling: every rank runs one 8-direction share of the 8-GPU job
        off, mine = shard_directions(DIRS4, 8, rank % 8)
        units_all = [d for r in range(world) for d in shard_directions(DIRS4, 8, r % 8)[1]]
        cfg = pipeline_cfg4(csf, capi, k, mine, n)
    else:
        units_all = PAIRS if second else DIRS          # the sharded work items
        off, mine = shard_directions(units_all, world, rank)
        cfg = pipeline_cfg(csf, capi, k, mine, n, pairs=mine if second else None)
    pipe = csf.Pipeline(cfg, ctx=ctx)
    pipe.upload(depth, gt)
    stream = torch.cuda.ExternalStream(ctx.stream)

    for _ in range(max(args.warmup, 0)):
        pipe.run()
    ctx.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---------------- timed region: device-resident inputs, no per-kernel events.
    # Both launch modes of the same run are timed: the stream of PDL-chained
    # launches, and the run replayed as one CUDA graph (csf_pipeline_set_graph;
    # bit-identical, tests/test_graph.py); `value` is the faster of the two.
    def timed(graph: bool):
        pipe.set_graph(graph)
        if graph:
            for _ in range(2):  # capture, then one replay
                pipe.run()
        ctx.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = ctx.launch_count
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            pipe.run()
        e1.record(stream)
        ctx.synchronize()
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1), ctx.launch_count - l0

    clocks = Clocks(local)
    ms_stream, launches_stream = timed(False)
    ms_graph, launches_graph = timed(True)
    pipe.set_graph(False)
    clk = clocks.stop()
    if dist is not None:  # max over ranks of each mode, then one choice for all ranks
        t = torch.tensor([ms_stream, ms_graph], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_stream, ms_graph = float(t[0].item()), float(t[1].item())
    use_graph = ms_graph < ms_stream
    ms, launches = (ms_graph, launches_graph) if use_graph else (ms_stream, launches_stream)
    if second:
        hr = pipe.hessian(stats=True)
        local_cols, stats = hr.hessian, hr.stats
    else:
        res = pipe.result()
        local_cols, stats = res.gradient, res.stats
    if dist is not None:
        # collective C2 in the C-ABI: csf_gather_columns over the context's NCCL communicator
        attach_native_comm(ctx, world, rank)
        cols = gather_columns_native(ctx, np.asarray(local_cols), len(units_all), world)
    if dist is None:
        cols = local_cols

    units_per_step = n * len(units_all)
    value = units_per_step * args.steps / (ms / 1000.0)

    # ---------------- profiled pass (same steps): per-kernel-category CUDA events
    ctx.synchronize()
    ctx.profile(True)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        pipe.run()
    p1.record(stream)
    ctx.synchronize()
    prof_ms = p0.elapsed_time(p1)
    prof = ctx.profile_read()
    ctx.profile(False)

    # ---------------- e2e through the public API from pinned host memory, in
    # the launch mode `value` chose (graph: the per-frame upload waits are
    # external event-wait nodes of the replayed run); two untimed calls set
    # up the capture
    pinned = torch.empty(depth.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = depth
    host_frames = pinned.numpy()
    # configs 2 and 3 ingest uint8 RGB beside the depth (BASELINE configs[1]);
    # the path never reads colour (the reference has none), it is uploaded only
    host_rgb = None
    if not one and not four:
        rgb_pinned = torch.empty(depth.shape + (3,), dtype=torch.uint8, pin_memory=True)
        rgb_pinned.numpy()[:] = synth_rgb(depth)
        host_rgb = rgb_pinned.numpy()
    pipe.set_graph(use_graph)
    for _ in range(2):
        pipe.run_host(host_frames, gt, rgb=host_rgb)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = pipe.run_host(host_frames, gt, rgb=host_rgb)
    t_e2e = time.perf_counter() - t0
    pipe.set_graph(False)
    if dist is not None:
        t = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e_value = units_per_step * args.steps / t_e2e
    h2d = int(depth.nbytes + gt.nbytes + (host_rgb.nbytes if host_rgb is not None else 0))
    d2h = int(8 * (len(mine) + 1))

    # ---------------- roofline: every category with a bytes model; the dominant one is `roofline`
    peak, peak_src = measured_peak()
    slots = 3 * len(mine) if second else len(mine)
    rooflines = {}
    for cat, (cat_ms, cat_n) in prof.items():
        bytes_step, bytes_def = algorithmic_bytes_per_step(cat, stats, slots, k.width, k.height, n)
        if bytes_step is None or cat_n == 0 or cat_ms <= 0:
            continue
        bytes_per_launch = bytes_step * args.steps / cat_n
        avg_ms = cat_ms / cat_n
        achieved = bytes_per_launch / (avg_ms / 1000.0) / 1e9
        rooflines[cat] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                          "frac": achieved / peak, "traffic": traffic_for(cat, args.workload), "kernel": cat,
                          "avg_launch_ms": avg_ms, "launches": cat_n, "share_of_step": cat_ms / prof_ms,
                          "algorithmic_bytes_per_launch": bytes_per_launch, "bytes_model": bytes_def,
                          "peak_source": peak_src, "fp64": fp64_roofline(cat, args.workload)}
    roofline = max(rooflines.values(), key=lambda r: r["share_of_step"]) if rooflines else None

    if one:
        workload = (f"config1: {n} frames 160x120, dense 128^3 TSDF at 2 cm (mu 6 cm), h = 1e-20, "
                    f"{len(units_all)} first-frame twist directions")
    elif four:
        workload = (f"config4: {n} VGA frames, 60x60 m terrain + 200 boxes, hashed 8^3 blocks 2 cm, 64 directions "
                    f"(6 first-frame + 4 intrinsics + 54 keyframe twists), 8 directions per GPU")
    elif second:
        workload = (f"config3: {n} VGA frames, hashed 8^3 blocks 5 mm, 2^20 buckets, 10x10 Hessian = "
                    f"{len(PAIRS)} bicomplex pairs")
    else:
        workload = f"config2: {n} VGA frames, hashed 8^3 blocks 5 mm, 2^20 buckets, {len(DIRS)} CSFD directions"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak" if four else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (seeded procedural terrain rendered on device; BASELINE config 4 shapes)" if four else
                 "synthetic (seeded toy room rendered on device; BASELINE config 1 shapes)" if one else
                 "synthetic (seeded procedural room rendered on device; BASELINE config 2 shapes)"),
        "config": {"workload": workload, "frames": n, "directions": len(units_all),
                   "directions_per_rank": len(mine), "order": 2 if second else 1,
                   "parallelism": f"{'pairs' if second else 'directions'} sharded x{world}",
                   "l2": ("working set: dense 128^3 x (16 + 6x8) B = 134 MB volume + maps > L2 (126 MB), "
                          "no flush" if one else
                          "working set (hashed volume, ~GBs) >> L2")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ingest": "float32 depth + uint8 RGB (colour unused by the path)" if host_rgb is not None
                else "float32 depth"},
        "gpu_launches": int(launches),
        "launch_mode": {"used": "cuda_graph" if use_graph else "stream", "stream_ms_per_step": ms_stream / args.steps,
                        "graph_ms_per_step": ms_graph / args.steps},
        "roofline": roofline,
        "roofline_by_kernel": rooflines,
        "clocks": clk,
        "kernel_ms_per_step": {c: v[0] / args.steps for c, v in prof.items()},
        "profiled_ms_per_step": prof_ms / args.steps,
        ("hessian_pairs" if second else "gradient"): [float(x) for x in cols],
        "blocks_allocated": int(stats[-1, 3]),
        "per_frame": {"visible_blocks": float(stats[:n, 4].mean()), "fused_voxels": float(stats[:n, 6].mean()),
                      "icp_iterations": float(stats[1:n, 0].mean()) if n > 1 else 0.0,
                      "correspondences": float(stats[1:n, 1].mean()) if n > 1 else 0.0},
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(depth, gt, k, args.cpu_frames, args.cpu_dirs, args.workload)
        except Exception as e:  # the oracle must have been built by build()
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if args.profile_json:
        Path(args.profile_json).write_text(json.dumps(prof, indent=1))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
