# ncu of the Strassen sketch at C4 (tools/strassen_check.py): launch list + full set of the second
# call's kernels (rcomb, 48-row products, 24-row products, combine)
CFG=${1:-C4}
python tools/strassen_check.py $CFG > gpurun_out/strassen_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:strassen \
  --log-file gpurun_out/strassen_launches_$CFG.csv python tools/strassen_check.py $CFG > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:strassen -s 6 -c 6 \
  -o gpurun_out/prof_strassen_$CFG -f python tools/strassen_check.py $CFG > gpurun_out/ncu_strassen.log 2>&1
echo "exit $?"
