"""ncu CSV (--metrics dram__bytes_read.sum,dram__bytes_write.sum,... --csv, NVTX-filtered M1 / M2 runs of
tools/traffic_run.py) -> profiles/traffic_<config>.json: dram bytes per frame of the K1 pass
(k_masks + k_walk + k_dedup), of k_stage2 and of the other stage-1 kernels, per mode."""
import csv
import json
import sys
from collections import defaultdict

cfg = sys.argv[1]
out = {}
for mode, path in zip(["M1", "M2"], sys.argv[2:4]):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ix = {k: hdr.index(k) for k in ["Kernel Name", "Metric Name", "Metric Value"]}
    per = defaultdict(lambda: defaultdict(float))
    for r in rows[h + 1:]:
        if len(r) < len(hdr):
            continue
        k = r[ix["Kernel Name"]].split("(")[0].split("<")[0].replace("disc::", "").replace("void ", "").strip()
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            per[k][r[ix["Metric Name"]]] += float(v)
        except ValueError:
            pass
    frames = 64.0
    def b(ks):
        return sum(per[k]["dram__bytes_read.sum"] + per[k]["dram__bytes_write.sum"] for k in ks) / frames
    out[mode] = {"K1": b(["k_masks", "k_walk", "k_dedup"]), "stage2": b(["k_stage2"]),
                 "per_kernel_bytes_per_frame": {k: (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / frames
                                                for k, v in per.items()},
                 "per_kernel_us_per_frame": {k: v.get("gpu__time_duration.sum", 0.0) / frames / 1e3 for k, v in per.items()},
                 "atomics_sectors_per_frame": {k: (v.get("lts__t_sectors_op_atom.sum", 0.0) + v.get("lts__t_sectors_op_red.sum", 0.0)) / frames
                                               for k, v in per.items()},
                 "frames": 64, "source": path}
json.dump(out, open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
print(json.dumps(out, indent=1))
