#!/bin/bash
# ncu full set of the small-sketch QR (k_qrcp_smem) at a config (C2 by default)
CFG=${1:-C2}
mkdir -p gpurun_out
PY="import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
os.environ['RID_GRAPH'] = '0'
for _ in range(2): rid.decompose(A, c.k, c.l, 1)
torch.cuda.synchronize()"
python -c "$PY" > gpurun_out/prof_qs_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_qrcp_smem -s 1 -c 1 \
  -o gpurun_out/prof_qsmall_$CFG -f python -c "$PY" > gpurun_out/ncu_qs.log 2>&1
echo "ncu exit $?"
