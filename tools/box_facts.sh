#!/bin/bash
# One-shot box facts + FP64 microbenchmarks (run under gpurun).
mkdir -p gpurun_out
{
nvidia-smi; nproc; lscpu | head -20; free -g; df -h /tmp | tail -1
./tools/mb
python - <<'PY'
import torch, time
for dt, n in ((torch.float64, 8192), (torch.complex128, 4096), (torch.complex128, 8192)):
    a = torch.randn(n, n, dtype=dt, device='cuda'); b = torch.randn(n, n, dtype=dt, device='cuda')
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = (2 if dt == torch.float64 else 8) * n**3
    print(f"torch matmul {dt} {n}^3: {ms:.2f} ms  {fl/ms/1e9:.2f} TFLOP/s")
print(torch.cuda.mem_get_info())
PY
} > gpurun_out/box_facts.txt 2>&1
