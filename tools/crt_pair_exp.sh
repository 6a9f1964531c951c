set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_crt.py -q -x 2>&1 | tail -5
for cfg in C4 C5 C3; do
 for rep in 1 2; do
  for v in 0 1; do
   RID_CRT_2SM=$v timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --q 0 --no-e2e --no-cpu-baseline > gpurun_out/pair_${cfg}_${v}_${rep}.json 2> gpurun_out/pair_${cfg}_${v}_${rep}.err
   echo "$cfg 2SM=$v rep=$rep rc=$?"; python - <<PY
import json
d=json.loads(open("gpurun_out/pair_${cfg}_${v}_${rep}.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], {k:v for k,v in d.items() if k in ("phases","clocks")})
PY
  done
 done
done
