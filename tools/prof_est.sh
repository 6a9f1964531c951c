#!/bin/bash
# ncu of the estimator's two streaming kernels (k_ax, k_z) at a config
CFG=${1:-C4}
PYC="import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
r = rid.decompose(A, c.k, c.l, 1)
print(rid.error_estimate(A, r.J, r.P, 2, 1))
torch.cuda.synchronize()"
python -c "$PYC" > gpurun_out/est_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"^k_(ax|z)$" -s 0 -c 2 -o gpurun_out/prof_est_$CFG -f python -c "$PYC" > gpurun_out/ncu_est.log 2>&1
echo "exit $?"
