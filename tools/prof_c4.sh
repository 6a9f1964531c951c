#!/bin/bash
# ncu evidence for bench C4: launch list + full sets of the sketch GEMM and the QRCP kernel.
CMD="python bench.py --config ${CFG:-C4} --steps 1 --warmup 1 --q 1 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG:-C4}.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_zgemm_dmma -s 1 -c 1 -o gpurun_out/prof_sketch_${CFG:-C4} -f $CMD > gpurun_out/ncu_sketch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_qrcp -c 1 -o gpurun_out/prof_qrcp_${CFG:-C4} -f $CMD > gpurun_out/ncu_qrcp.log 2>&1
echo "exit $?"
