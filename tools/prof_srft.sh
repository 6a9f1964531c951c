#!/bin/bash
# launch list of one SRFT sketch at a config (k_srft_* and the residue GEMMs)
CFG=${1:-C4}
PYC="import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
for _ in range(2): rid.sketch_srft(A, 1, c.l)
torch.cuda.synchronize()"
python -c "$PYC" > gpurun_out/srft_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/srft_launches_$CFG.csv python -c "$PYC" > /dev/null 2>&1
echo done
