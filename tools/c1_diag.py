import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1205_3830_b200 as rid
A = rid.generate(1, 1024, 512, 16, 0.0)
J = torch.empty(16, dtype=torch.int64, device="cuda")
P = rid.colmajor_empty(16, 512, device="cuda")
for _ in range(5): rid.decompose(A, 16, 24, 1, J=J, P=P)
ds = []
for _ in range(50):
    r = rid.decompose(A, 16, 24, 1, J=J, P=P); ds.append(r.diag)
keys = [k for k in ds[0] if k.startswith("t_")]
print({k: round(float(np.median([d[k] for d in ds]))*1e6, 1) for k in keys})
