#!/bin/bash
# ncu capture of one lazy-QR panel launch (k_qrcp_lazy; launch index $2, default 1 = panel 2)
CFG=${1:-C4}
SKIP=${2:-1}
mkdir -p gpurun_out
cat > /tmp/lazy_once.py << 'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS[sys.argv[1]]
A = rid.generate(1, c.m, c.n, c.k, c.noise)
r = rid.decompose(A, c.k, c.l, 1)
print("t_qrcp ms", r.diag["t_qrcp"] * 1e3)
PY
python /tmp/lazy_once.py $CFG > gpurun_out/prof_lazy_plain_$CFG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_qrcp_lazy -s $SKIP -c 1 \
  -o gpurun_out/prof_lazy_$CFG -f python /tmp/lazy_once.py $CFG > gpurun_out/ncu_lazy_$CFG.log 2>&1
echo "ncu exit $?"
