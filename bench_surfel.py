"""bench.py --workload surfel: the surfel (X-EF) front end (SURVEY §8(f)
row 4) on the config-2 scene.

Setup (untimed): 100 VGA depth frames of the seeded procedural room.  Step:
a fresh SurfelMap with 6 derivative channels; every frame fused by
update_surfels at its ground-truth pose lifted on the 6 twist directions
(exp(xi) T, xi seeded h = 1e-8 per channel; left increment, se3.hpp:116-119):
index map (two stable radix sorts), one-to-many association, scan-order
accumulation / commit-once update, append.  Units = frames x 6 directions
(frame-derivatives/s, the headline's unit).  value: CUDA-event time of the
public call, which takes host frames (each frame's lifted depth H2D is inside
the timed region); e2e: wall clock of the same loop.  Roofline: per frame, algorithmic bytes = the map read by
the index-map projection (24 B real position per surfel) + sort traffic
(2 sorts x ~4 passes x 2 x 12 B per surfel) + association reads (16 cells of
candidates x 48 B) + the committed surfels' lifted state (2 x 404 B) + the
frame's lifted maps (2 x 48 x 7 B per pixel) — HBM-bound; measured against
MEASURED_PEAKS.json.  cpu_baseline: the oracle on the first 3 frames.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

D = 6


def lifted_poses(gt, h=1e-8):
    """exp(xi) T with xi_d = h on channel d: first-order lift of the left
    increment, R' = R + h [e_phi]x R, t' = t + h (rho + [e_phi]x t)."""
    out = []
    for p in gt:
        R, t = p[:9].reshape(3, 3), p[9:]
        L = np.zeros((12, 1 + D))
        L[:9, 0] = R.reshape(9)
        L[9:, 0] = t
        for c in range(3):  # rho
            L[9 + c, 1 + c] = h
        for a in range(3):  # phi
            e = np.zeros(3)
            e[a] = 1.0
            S = np.array([[0, -e[2], e[1]], [e[2], 0, -e[0]], [-e[1], e[0], 0]])
            L[:9, 4 + a] = (h * (S @ R)).reshape(9)
            L[9:, 4 + a] = h * (S @ t)
        out.append(L)
    return out


def run(args, measured_peak, Clocks):
    import torch
    import paper_2405_02187_b200 as csf
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    torch.cuda.set_device(local)
    ctx = csf.Context(local)
    n_frames = 100
    depth, gt, k = csf.synth_workload(2, n_frames, ctx=ctx)
    poses = lifted_poses(gt)
    frames = []
    for f in range(n_frames):  # unperturbed host frames in pinned memory (lifted on the device)
        t = torch.zeros(depth[f].shape, dtype=torch.float64, pin_memory=True)
        d = t.numpy()
        d[...] = depth[f]
        frames.append(d)
    cfg = csf.default_surfel_cfg()
    stream = torch.cuda.ExternalStream(ctx.stream)

    m = csf.SurfelMap(D, ctx=ctx)

    def step():
        m.clear()  # a fresh map each step; device capacity kept from the warm-up
        st = [csf.update_surfels(m, frames[f], poses[f], k, f, cfg) for f in range(n_frames)]
        return m, st

    for _ in range(max(args.warmup, 0)):
        step()
    ctx.synchronize()
    clocks = Clocks(local)
    torch.cuda.synchronize()
    l0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        _, st = step()
        n_map = m.size()
    e1.record(stream)
    ctx.synchronize()
    t_e2e = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count - l0
    clk = clocks.stop()
    units = n_frames * D
    value = units * args.steps / (ms / 1000.0)
    merged = float(np.mean([s.merged_pixels for s in st]))
    created = [s.created for s in st]
    mean_map = float(np.mean(np.cumsum(created)))
    P = k.width * k.height
    C = 1 + D
    surfel_b = 2 * 3 * C * 8 + C * 8 + 12
    b_frame = mean_map * (24 + 2 * 4 * 2 * 12) + merged * 16 * 48 + 2 * merged * surfel_b + 2 * P * 48 * C
    ach = b_frame * n_frames * args.steps / (ms / 1000.0) / 1e9
    peak, src = measured_peak()
    unit = "frame-derivatives/s"
    line = {
        "metric": "surfel (X-EF) fusion frame-derivatives/s at 640x480 (frames x 6 pose directions)",
        "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded procedural room; BASELINE config 2 frames)",
        "config": {"workload": "surfel: 100 VGA frames fused into a surfel map at ground-truth poses lifted on "
                               "6 twist directions", "frames": n_frames, "directions": D,
                   "final_surfels": int(n_map), "mean_merged_pixels": merged, "parallelism": "replicas only",
                   "l2": "surfel map (GBs) >> L2"},
        "e2e": {"value": units * args.steps / t_e2e, "unit": unit,
                "h2d_bytes_per_step": int(sum(f.nbytes for f in frames) + n_frames * 12 * C * 8),
                "d2h_bytes_per_step": int(n_frames * 8)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "kernel": "update_surfels (whole frame)",
                     "algorithmic_bytes_per_launch": b_frame, "peak_source": src,
                     "bytes_model": "per frame: map projection 24 B/surfel + 2 radix sorts (~4 passes x 2 x 12 B) "
                                    "+ 16-cell candidate reads 48 B + merged surfels' lifted state r+w + lifted "
                                    "frame maps"},
        "clocks": clk,
    }
    # e2e above includes the host->device copies of the lifted frames inside update_surfels (public API)
    if not args.no_cpu:
        try:
            from oracle import orc
            mo = orc.Surfels(D)
            nf = 3
            t1 = time.perf_counter()
            for f in range(nf):
                dl = np.zeros(frames[f].shape + (1 + D,))
                dl[..., 0] = frames[f]
                mo.update(dl, poses[f], k, f, capi_cfg(cfg))
            secs = time.perf_counter() - t1
            cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
            line["cpu_baseline"] = {"value": nf * D / secs, "unit": unit, "cores": cores, "kind": "port",
                                    "sample": f"oracle update_surfels on the first {nf} frames x {D} directions "
                                              f"(Lifted<6> scalar, association OpenMP over rows; {secs:.2f} s)"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)


def capi_cfg(cfg):
    return cfg


def run_reference(args):
    import paper_2405_02187_b200 as csf
    from oracle import orc
    if int(os.environ.get("RANK", "0")) != 0:
        return
    depth, gt, k = orc.workload(2, 3)  # the oracle renderer: no GPU work on the reference arm
    poses = lifted_poses(gt)
    from paper_2405_02187_b200 import capi
    cfg = capi.SurfelCfg(0.05, 30.0, 0.05, 0.025, 1)  # surfel.hpp defaults
    vals = []
    t0 = time.perf_counter()
    for _ in range(max(args.steps, 1)):
        mo = orc.Surfels(D)
        t1 = time.perf_counter()
        for f in range(3):
            d = np.zeros(depth[f].shape + (1 + D,))
            d[..., 0] = depth[f]
            mo.update(d, poses[f], k, f, cfg)
        vals.append(3 * D / (time.perf_counter() - t1))
    v = float(np.median(vals))
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    print(json.dumps({"impl": "reference", "metric": "surfel (X-EF) fusion frame-derivatives/s at 640x480 "
                      "(frames x 6 pose directions)", "value": v, "unit": "frame-derivatives/s", "n_gpus": 1,
                      "steps": args.steps, "warmup": 0,
                      "ms_per_step": 1000.0 * (time.perf_counter() - t0) / max(args.steps, 1),
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": "surfel"},
                      "cpu_baseline": {"value": v, "unit": "frame-derivatives/s", "cores": cores, "kind": "port",
                                       "sample": "oracle update_surfels, first 3 frames x 6 directions"},
                      "e2e": {"value": v, "unit": "frame-derivatives/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}), flush=True)
