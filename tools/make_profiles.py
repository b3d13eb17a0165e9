"""Write round profile summaries into profiles/ from ncu reports in gpurun_out/ (run here)."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(__file__))
from ncu_summary import details, hot_lines, raw  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def mb(s):
    v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def summarize(rep, kernel, out, title):
    d = details(rep, kernel)
    r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                  "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "gpu__time_duration.sum",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"],
            kernel)
    lines = [f"# {title}", f"source report: {os.path.basename(rep)} (ncu --set full --clock-control none), kernel {kernel}",
             ""]
    lines += [f"{k:40s} {v}" for k, v in d.items()]
    lines += [f"{k:40s} {v}" for k, v in r.items()]
    lines += ["", "hottest source lines (warp stall samples):"]
    lines += [f"{p:5.1f}% {fl}:{ln} {src}" for p, fl, ln, src in hot_lines(rep, 25, kernel)]
    open(out, "w").write("\n".join(lines) + "\n")
    return mb(r["dram__bytes_read.sum"]) + mb(r["dram__bytes_write.sum"])


if __name__ == "__main__":
    # usage: make_profiles.py <report> <round tag> <frames per launch> kernel [kernel ...]
    # K1 = k_masks + k_walk + k_dedup: their summed DRAM bytes per frame feed bench.py's roofline.traffic
    rep, tag, fpl, kernels = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4:]
    per = {}
    for k in kernels:
        per[k] = summarize(rep, k, os.path.join(ROOT, "profiles", f"{tag}_{k}_ncu_summary.txt"), f"{tag} {k}") / fpl
        print(k, "dram bytes per frame", per[k])
    if "k_masks" in per and "k_walk" in per:
        k1 = [k for k in ("k_masks", "k_walk", "k_dedup") if k in per]
        json.dump({"dram_bytes_per_frame": sum(per[k] for k in k1), "source": os.path.basename(rep),
                   "per_kernel": per,
                   "note": "dram__bytes_read.sum + dram__bytes_write.sum of the K1 pass (%s) per frame" % " + ".join(k1)},
                  open(os.path.join(ROOT, "profiles", "k1_dram_bytes_per_frame.json"), "w"), indent=1)
