#!/bin/bash
# ncu full set of the generation GEMM (k_zgemm_dmma mode 1: A = X·Y0 + ε·E) at a config
CFG=${1:-C4}
mkdir -p gpurun_out
PY="import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
torch.cuda.synchronize()"
python -c "$PY" > gpurun_out/prof_gen_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_zgemm_dmma -c 1 \
  -o gpurun_out/prof_gen_$CFG -f python -c "$PY" > gpurun_out/ncu_gen.log 2>&1
echo "ncu exit $?"
