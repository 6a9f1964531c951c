#!/bin/bash
# ncu evidence for a bench config: launch list of one bench step + full sets of the sketch
# (C4/C5: the four k_strassen3m launches of the timed step — 48-row products with two / one A
# blocks, remainder rows the same; other configs k_zgemm3m_tma), one blocked-QRCP panel
# (k_qrcp_ring) and one QRCP trailing update (k_zgemm_dmma mode 2). Run each ncu pass only after
# the plain command exits 0.
CFG=${CFG:-C4}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --q 1 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
SK=${SK:-k_strassen3m}
ncu --set full --clock-control none --import-source on -k regex:$SK -s 4 -c 4 -o gpurun_out/prof_sketch_$CFG -f $CMD > gpurun_out/ncu_sketch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_qrcp_ring -s 8 -c 1 -o gpurun_out/prof_qrcp_$CFG -f $CMD > gpurun_out/ncu_qrcp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm_dmma -s 12 -c 1 -o gpurun_out/prof_update_$CFG -f $CMD > gpurun_out/ncu_update.log 2>&1
echo "exit $?"
