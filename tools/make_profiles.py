"""Write round profile summaries into profiles/ from ncu reports in gpurun_out/ (run here)."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(__file__))
from ncu_summary import details, hot_lines, raw  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def summarize(rep, out, frames_per_launch, title):
    d = details(rep)
    r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                  "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "gpu__time_duration.sum"])
    lines = [f"# {title}", f"source report: {os.path.basename(rep)} (ncu --set full --clock-control none)", ""]
    lines += [f"{k:40s} {v}" for k, v in d.items()]
    lines += [f"{k:40s} {v}" for k, v in r.items()]
    lines += ["", "hottest source lines (warp stall samples):"]
    lines += [f"{p:5.1f}% {fl}:{ln} {src}" for p, fl, ln, src in hot_lines(rep, 25)]
    open(out, "w").write("\n".join(lines) + "\n")

    def mb(s):
        v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    tot = mb(r["dram__bytes_read.sum"]) + mb(r["dram__bytes_write.sum"])
    return tot / frames_per_launch


if __name__ == "__main__":
    rep, tag, fpl = sys.argv[1], sys.argv[2], int(sys.argv[3])
    per_frame = summarize(rep, os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt"), fpl, tag)
    if len(sys.argv) > 4 and sys.argv[4] == "k1":
        json.dump({"dram_bytes_per_frame": per_frame, "source": os.path.basename(rep),
                   "note": "dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch / frames per launch"},
                  open(os.path.join(ROOT, "profiles", "k1_dram_bytes_per_frame.json"), "w"), indent=1)
    print(tag, "dram bytes per frame", per_frame)
