#!/bin/bash
# Round evidence: GPU tests, default bench line, ncu launch list + full set of the sketch GEMM.
CFG=${CFG:-C4}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py --config $CFG > gpurun_out/bench_round_$CFG.log 2>&1; tail -1 gpurun_out/bench_round_$CFG.log | cut -c1-400
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --q 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_zgemm_dmma -s 1 -c 1 -o gpurun_out/prof_sketch_$CFG -f $CMD > gpurun_out/ncu_sketch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_qrcp -c 1 -o gpurun_out/prof_qrcp_$CFG -f $CMD > gpurun_out/ncu_qrcp.log 2>&1
echo "prof exit $?"
