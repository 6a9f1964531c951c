CFG=C4
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --q 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm3m -s 3 -c 1 -o gpurun_out/prof_sketch_$CFG -f $CMD > gpurun_out/ncu_sketch.log 2>&1
echo "exit $?"
