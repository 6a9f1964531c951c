#!/bin/bash
# ncu evidence for the error estimator at a config: launch list of one q = 2 estimate and full
# sets of the TMA-fed passes (k_ax_tma, k_z_tma)
CFG=${1:-C4}
mkdir -p gpurun_out
PY="import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS['$CFG']
A = rid.generate(1, c.m, c.n, c.k, c.noise)
r = rid.decompose(A, c.k, c.l, 1)
print(rid.error_estimate(A, r.J, r.P, 2, 1))"
python -c "$PY" > gpurun_out/prof_est_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_est_$CFG.csv python -c "$PY" > gpurun_out/ncu_est_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_ax_tma|k_z_tma" -s 2 -c 2 \
  -o gpurun_out/prof_est_$CFG -f python -c "$PY" > gpurun_out/ncu_est.log 2>&1
echo "ncu exit $?"
