"""Summaries of ncu reports (run here, no GPU): SOL/occupancy/memory metrics and top source lines."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Avg. Active Threads Per Warp", "Issued Ipc Active", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Dynamic Shared Memory Per Block", "Grid Size", "Theoretical Occupancy"]


def _k(kernel):
    return ["-k", f"regex:{kernel}"] if kernel else []


def details(rep, kernel=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"] + _k(kernel), capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    res = {}
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in WANT and d["Metric Name"] not in res:
            res[d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
    return res


def raw(rep, names, kernel=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + _k(kernel), capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    res = {}
    for row in r[2:]:
        for n in names:
            if n in h:
                i = h.index(n)
                res[n] = row[i] + " " + u[i]
    return res


def hot_lines(rep, top=20, kernel=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + _k(kernel),
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    cur = None
    lines = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 5 and r[0] not in ("", "Line No"):
            lines.append((cur, r[0], r[1], f(r[4])))
    tot = sum(x[3] for x in lines) or 1
    return [(100 * s / tot, fl, ln, src.strip()[:90]) for fl, ln, src, s in sorted(lines, key=lambda x: -x[3])[:top]]


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, v in details(rep).items():
        print(f"{k:40s} {v}")
    for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_atom.sum",
                          "lts__t_sectors_op_red.sum", "smsp__inst_executed.sum"]).items():
        print(f"{k:40s} {v}")
    print("--- hottest source lines (warp stall samples) ---")
    for pct, fl, ln, src in hot_lines(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 20):
        print(f"{pct:5.1f}% {fl}:{ln} {src}")
