"""Summarise ncu captures into profiles/ (runs here, on the CPU box).

  python scripts/ncu_summary.py <report.ncu-rep> <n_points> [--counts]

Prints time, registers, occupancy, issue/FP64 utilisation, DRAM traffic per
point and the top stall reasons; with --counts also writes the flux kernel's
dynamic FP64 flop count and DRAM bytes per point to profiles/flux_ncu_counts.json
(consumed by bench.py's roofline block).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {k: (u, v) for k, u, v in zip(rows[0], rows[1], rows[2])}


def num(d, k):
    """Value in ms for times, MB for byte counts, as-is otherwise."""
    try:
        u, v = d[k]
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)
    except (KeyError, ValueError):
        return None


def main():
    report, n = sys.argv[1], int(sys.argv[2])
    d = raw(report)
    cyc = num(d, "sm__cycles_elapsed.avg")
    per_cycle = {op: num(d, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
                 for op in ("dfma", "dadd", "dmul")}
    fp = {op: v * cyc / n for op, v in per_cycle.items() if v is not None}
    flops = 2 * fp.get("dfma", 0) + fp.get("dadd", 0) + fp.get("dmul", 0)
    dram = (num(d, "dram__bytes_read.sum") or 0) * 1e6 + (num(d, "dram__bytes_write.sum") or 0) * 1e6
    stalls = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      num(d, k)) for k in d if "average_warps_issue_stalled" in k and "not_issued" not in k),
                    key=lambda t: -(t[1] or 0))[:6]
    summary = {
        "report": os.path.basename(report),
        "duration_ms": num(d, "gpu__time_duration.sum"),
        "registers": num(d, "launch__registers_per_thread"),
        "achieved_occupancy_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "dram_throughput_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warp_inst_per_point": (num(d, "smsp__inst_executed.sum") or 0) / n,
        "fp64_thread_inst_per_point": {k: round(v, 1) for k, v in fp.items()},
        "fp64_flops_per_point": flops,
        "dram_bytes_per_point": dram / n,
        "top_stalls": stalls,
    }
    print(json.dumps(summary, indent=1))
    if "--counts" in sys.argv:
        path = os.path.join(ROOT, "profiles", "flux_ncu_counts.json")
        json.dump({"source": os.path.basename(report), "n_points": n,
                   "flux_fp64_flops_per_point": flops, "flux_dram_bytes_per_point": dram / n,
                   "flux_fp64_thread_inst_per_point": fp,
                   "note": "dynamic counts of the flux kernel from one ncu --set full capture "
                           "(NACA 0012 O-cloud, order 2; n_points above); flops = 2*DFMA + DADD + DMUL"},
                  open(path, "w"), indent=1)
        print("wrote", path)


if __name__ == "__main__":
    main()
