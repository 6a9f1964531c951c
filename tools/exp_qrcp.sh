bash tools/dbg_qrcp_shapes.sh 2>&1 | grep -v "J equal True" ; echo shapes-done
timeout 120 python tools/dbg_qrcp_cfg.py C4
for c in C4 C5 C2; do
for env in "" "RID_QRCP_L2KEEP_MB=0"; do
  echo "== $c $env"; env $env timeout 120 python tools/trace_qrcp.py $c 1 > gpurun_out/exp.txt 2>&1; grep -E "variant|steps" gpurun_out/exp.txt
done; done
