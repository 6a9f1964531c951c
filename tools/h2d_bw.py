"""Pinned host -> device copy bandwidth on the box: one copy stream vs two (e2e path sizing)."""
import torch
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for label, parts in (("1 stream, 1 x 4 GiB", 1), ("1 stream, 4 x 1 GiB", 4), ("2 streams, 2 x 2 GiB", 2),
                     ("2 streams, 8 x 512 MiB", 8)):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step = n // parts
    for i in range(parts):
        st = s1 if (label.startswith("1") or i % 2 == 0) else s2
        with torch.cuda.stream(st):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
