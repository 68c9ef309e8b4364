"""Pinned host -> device copy bandwidth on this box (the e2e path's ceiling)."""
import torch, time
n = 3323888640 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for chunks in (1, 7, 28):
    c = n // chunks
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for i in range(chunks):
                d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
            e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"chunks={chunks:3d} rep={rep} {4 * c * chunks / ms / 1e6:.1f} GB/s ({ms:.2f} ms)", flush=True)
# D2H for reference
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); h.copy_(d, non_blocking=True); e1.record(); e1.synchronize()
print(f"D2H {4 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
