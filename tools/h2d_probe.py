"""Pinned host -> device copy bandwidth (one stream vs two), 150 MB in 4.7 MB pieces (an H window)."""
import torch
n, piece = 32, 4_700_000
src = [torch.empty(piece, dtype=torch.uint8).pin_memory() for _ in range(n)]
dst = [torch.empty(piece, dtype=torch.uint8, device="cuda") for _ in range(n)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for streams in (1, 2):
    best = 0
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            st = s1 if (streams == 1 or i % 2 == 0) else s2
            st.wait_event(e0)
            with torch.cuda.stream(st):
                dst[i].copy_(src[i], non_blocking=True)
        s1.synchronize(); s2.synchronize()
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1.record(); torch.cuda.synchronize()
        best = max(best, n * piece / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print(f"{streams} stream(s): {best:.1f} GB/s")
# the per-frame copies of an H M1 window (depth, mask bits, mask conf, tracking tokens) as the host
# path issues them: 4 copies per frame
sizes = [1_228_800, 2_304_000, 240, 1_175_040]
srcs = [[torch.empty(z, dtype=torch.uint8).pin_memory() for z in sizes] for _ in range(n)]
dsts = [[torch.empty(z, dtype=torch.uint8, device="cuda") for z in sizes] for _ in range(n)]
best = 0
for _ in range(5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        for a, b in zip(srcs[i], dsts[i]):
            b.copy_(a, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    best = max(best, n * sum(sizes) / (e0.elapsed_time(e1) / 1e3) / 1e9)
print(f"H window as 4 copies per frame: {best:.1f} GB/s")
