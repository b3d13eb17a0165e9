"""Summarise DISC_TIMELINE=1 output (lines 'TL <stream> <mark> <frame> <ms>'): per-kernel mean
duration (mark minus the previous mark on the same stream, so queueing behind the other stream's
work is included), and per-window stage spans.  usage: timeline_summary.py log [skip_windows]"""
import collections
import sys

recs = []
for line in open(sys.argv[1]):
    if line.startswith("TL "):
        _, st, name, fr, ms = line.split()
        recs.append((st, name, int(fr), float(ms)))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 1
# windows: split at s1_begin marks
wins, cur = [], []
for r in recs:
    if r[1] == "s1_begin" and cur:
        wins.append(cur)
        cur = []
    cur.append(r)
wins.append(cur)
recs = [r for w in wins[skip:] for r in w]
nwin = len(wins) - skip
dur = collections.defaultdict(float)
cnt = collections.Counter()
last = {}
for st, name, fr, ms in sorted(recs, key=lambda r: r[3]):
    if st in last and name not in ("s1_begin", "s2_begin"):
        dur[name] += ms - last[st]
        cnt[name] += 1
    last[st] = ms
print(f"windows {nwin}")
print(f"{'kernel':14s} {'ms/window':>10s} {'us/launch':>10s} launches/window")
for k, v in sorted(dur.items(), key=lambda kv: -kv[1]):
    print(f"{k:14s} {v / nwin:10.3f} {1000 * v / cnt[k]:10.1f} {cnt[k] / nwin:6.1f}")
t0 = recs[0][3]
t1 = recs[-1][3]
print(f"span {(t1 - t0) / max(nwin - 1, 1):.3f} ms/window (first mark to last mark / (windows-1))")

# per-stream busy/idle: gaps between a stream's consecutive marks that follow a stage-begin mark
streams = collections.defaultdict(list)
for st, name, fr, ms in recs:
    streams[st].append((ms, name))
for st, ev in streams.items():
    ev.sort()
    names = [n for _, n in ev]
    kind = "s2" if "k_stage2" in names else "s1"
    gaps = [(ev[i][0] - ev[i - 1][0], ev[i - 1][1], ev[i][1]) for i in range(1, len(ev)) if ev[i][1] in ("s1_begin", "s2_begin")]
    tot_gap = sum(g for g, _, _ in gaps)
    print(f"{kind}: {len(ev)} marks, waits before stage begins: {tot_gap / max(nwin, 1):.3f} ms/window")
