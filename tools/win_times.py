"""Per-window stage-1 / K1 / stage-2 device times over a longer stream (DISC_TIMELINE marks)."""
import collections
import sys

recs = [l.split() for l in open(sys.argv[1]) if l.startswith("TL ")]
t = collections.defaultdict(list)
last = {}
for _, st, name, fr, ms in recs:
    ms = float(ms)
    if name in ("s1_begin", "s2_begin"):
        last[st] = ms
    if name in ("k_walk", "k_finalize", "k_stage2"):
        t[name].append(ms - last[st])
print("K1 (s1_begin -> k_walk):", " ".join(f"{x:.2f}" for x in t["k_walk"]))
print("S1 (s1_begin -> k_finalize):", " ".join(f"{x:.2f}" for x in t["k_finalize"]))
print("S2:", " ".join(f"{x:.2f}" for x in t["k_stage2"]))
