#!/bin/bash
# ncu capture of one 3M sketch launch (k_zgemm3m) at a config
CFG=${1:-C4}
mkdir -p gpurun_out
python -c "
import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
for _ in range(2): rid.sketch(A, 1, c.l)
torch.cuda.synchronize()
" > gpurun_out/prof3m_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm3m -s 1 -c 1 \
  -o gpurun_out/prof_3m_$CFG -f python -c "
import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
for _ in range(2): rid.sketch(A, 1, c.l)
torch.cuda.synchronize()
" > gpurun_out/ncu_3m_$CFG.log 2>&1
echo "ncu exit $?"
