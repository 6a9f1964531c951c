#!/bin/bash
# Round evidence in one call on one B200: GPU tests, smoke, the default bench line (C4), every
# config's bench line (tools/bench_all.sh), the reference arm, and the C4 ncu evidence
# (tools/prof_c4.sh: launch list + full sets of the sketch, one QR panel, one panel update).
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log | cut -c1-400
bash tools/bench_all.sh
python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "reference rc=$?"
tail -1 gpurun_out/bench_reference.log | cut -c1-300
bash tools/prof_c4.sh
