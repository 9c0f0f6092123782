"""Summarise an ncu --set full report (one kernel) into a small text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<name>.txt "<command line>"
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "SM Busy", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "Waves Per SM",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, dst, cmd=""):
    lines = [f"ncu --set full --clock-control none --import-source on  ({cmd})", ""]
    r = ncu_csv(rep, "details")
    h = r[0]
    kname = None
    for row in r[1:]:
        d = dict(zip(h, row))
        kname = kname or d.get("Kernel Name")
        if d.get("Metric Name") in KEYS:
            lines.append(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    lines.insert(1, f"kernel: {kname}")
    rr = ncu_csv(rep, "raw")
    h, u, v = rr[0], rr[1], rr[2]
    lines.append("")
    for i, name in enumerate(h):
        if name in RAW:
            lines.append(f"{name:70s} {v[i]} {u[i]}")
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), name.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    lines.append("")
    lines.append("warp stall reasons (warps per issue-active cycle):")
    for val, name in sorted(stalls, reverse=True)[:10]:
        lines.append(f"  {name:28s} {val:.3f}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
