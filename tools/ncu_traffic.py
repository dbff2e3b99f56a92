"""Summarise ncu --set full captures (gpurun_out/prof_<kernel>.ncu-rep) into
profiles/traffic.json (DRAM bytes per launch per bench kernel category, read
by bench.py's roofline `traffic`) and profiles/<round>_ncu_<kernel>.csv."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CATS = {"k_icp_level": "icp", "k_raycast_march": "raycast", "k_raycast_march_seg": "raycast_seg",
        "k_raycast_lift_coop": "raycast_lift", "k_integrate_hashed": "integrate", "k_bilateral": "bilateral"}
KEEP = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "dram__throughput",
        "sm__throughput", "launch__registers_per_thread", "sm__warps_active", "launch__occupancy_limit",
        "smsp__inst_executed", "sm__inst_executed_pipe_fp64", "l1tex__t_bytes", "lts__t_bytes", "launch__grid_size",
        "launch__block_size", "sm__pipe_fp64_cycles_active", "smsp__average_warp", "achieved_occupancy",
        "smsp__sass_thread_inst_executed_op_d", "smsp__pcsamp")


def to_bytes(v, unit):
    f = float(str(v).replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


CATS_C3 = {"c3_integrate": "integrate", "c3_lift2": "raycast_lift"}  # tools/ncu_c3_o2.sh


def main(workload="config2", rnd="r01"):
    out = {}
    for kern, cat in (CATS_C3 if workload == "config3" else CATS).items():
        rep = ROOT / "gpurun_out" / f"prof_{kern}.ncu-rep"
        if not rep.exists():
            continue
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        head, units, vals = rows[0], rows[1], rows[2]
        rec = {h: (v, u) for h, u, v in zip(head, units, vals)}
        rd = to_bytes(*rec["dram__bytes_read.sum"])
        wr = to_bytes(*rec["dram__bytes_write.sum"])

        def num(name):
            v = rec.get(name)
            return float(str(v[0]).replace(",", "")) if v and v[0] not in ("", "n/a") else 0.0
        dur_us = num("gpu__time_duration.sum")  # unit us in --set full captures
        unit = rec.get("gpu__time_duration.sum", ("", "us"))[1]
        dur_s = dur_us * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-6)
        flops = (2.0 * num("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum") +
                 num("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum") +
                 num("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"))
        out[cat] = {"dram_bytes": rd + wr, "duration_s": dur_s, "fp64_flops": flops,
                    "fp64_pipe_active_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "dram_gbs": (rd + wr) / dur_s / 1e9 if dur_s > 0 else None,
                    "fp64_tflops": flops / dur_s / 1e12 if dur_s > 0 else None}
        keep = [(h, u, v) for h, u, v in zip(head, units, vals) if h.startswith(KEEP) or h in ("Kernel Name",)]
        with open(ROOT / "profiles" / f"{rnd}_ncu_{kern}.csv", "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["metric", "unit", "value"])
            w.writerows(keep)
        print(f"{cat:14s} {kern:24s} dram {out[cat]['dram_bytes'] / 1e6:10.2f} MB  time {dur_s * 1e6:9.1f} us  "
              f"fp64 {flops / 1e9:8.3f} GFLOP ({out[cat]['fp64_pipe_active_pct']:.1f}% pipe)")
    p = ROOT / "profiles" / "traffic.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    d["_note"] = ("per category, ONE launch (frame 5, level 0 for per-level kernels) under ncu --set full "
                  "--clock-control none (cold caches, serialised): DRAM bytes read+write, duration, FP64 flops "
                  "(2 dfma + dadd + dmul thread instructions), FP64 pipe active %; tools/ncu_capture.sh + "
                  "tools/ncu_traffic.py")
    d[workload] = out
    p.write_text(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
