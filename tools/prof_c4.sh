#!/bin/bash
# ncu evidence for a bench config: launch list of one bench step + full sets of the sketch
# (C4/C5: the four k_strassen3m launches of the timed step, one ncu session each — 48-row products with two / one A
# blocks, remainder rows the same; other configs k_zgemm3m_tma), one blocked-QRCP panel
# (k_qrcp_ring) and one QRCP trailing update (k_zgemm_dmma mode 2). Run each ncu pass only after
# the plain command exits 0.
CFG=${CFG:-C4}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --q 1 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
SK=${SK:-k_strassen3m}
# one ncu session per sketch launch: captured together, the launch that overlaps the aux-stream
# remainder reads back nan counters (profiles/r02s9); alone each one has clean counters
NSK=${NSK:-4}
for i in $(seq 0 $((NSK - 1))); do
  ncu --set full --metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum --clock-control none --import-source on -k regex:$SK -s $((NSK + i)) -c 1 -o gpurun_out/prof_sketch${i}_$CFG -f $CMD > gpurun_out/ncu_sketch$i.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_qrcp_ring -s 8 -c 1 -o gpurun_out/prof_qrcp_$CFG -f $CMD > gpurun_out/ncu_qrcp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm_dmma -s 12 -c 1 -o gpurun_out/prof_update_$CFG -f $CMD > gpurun_out/ncu_update.log 2>&1
echo "exit $?"
