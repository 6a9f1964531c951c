#!/bin/bash
# ncu capture of one blocked-QRCP panel (k_qrcp_ring) on a config (panel index $2)
CFG=${1:-C5}
SKIP=${2:-8}
mkdir -p gpurun_out
python tools/dbg_qrcp_cfg.py $CFG > gpurun_out/prof_qrcp_plain_$CFG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_qrcp_ring -s $SKIP -c 1 \
  -o gpurun_out/prof_ring_$CFG -f python tools/dbg_qrcp_cfg.py $CFG > gpurun_out/ncu_ring_$CFG.log 2>&1
echo "ncu exit $?"
