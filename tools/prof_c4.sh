#!/bin/bash
# ncu evidence for a bench config: launch list of one bench step + full sets of the sketch's
# kernels and of the QR. INT8_CRT engine (C3-C5 default): one k_imma launch (the tcgen05 int8 GEMM,
# one of the sketch's column blocks), one k_crt_prepA and one k_crt_rec; DMMA engine (ENGINE=dmma
# or C1/C2): the sketch launches (SK, NSK). Then one blocked-QRCP panel (QRK: k_qrcp_lazy at C4, k_qrcp_ring at C5) and one QRCP
# trailing update (k_zgemm_dmma mode 2). Each ncu pass runs only after the plain command exits 0.
CFG=${CFG:-C4}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --q 1 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
if [ "${ENGINE:-crt}" = "crt" ]; then
  NB=${NB:-2}  # GEMM launches (column blocks) per sketch at C4 (148 + 108 tiles): skip the warm-up step's
  ncu --set full --clock-control none --import-source on -k regex:k_imma -s $NB -c 1 -o gpurun_out/prof_crt_gemm_$CFG -f $CMD > gpurun_out/ncu_gemm.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_crt_prepA -s $NB -c 1 -o gpurun_out/prof_crt_prep_$CFG -f $CMD > gpurun_out/ncu_prep.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_crt_rec -s $NB -c 1 -o gpurun_out/prof_crt_rec_$CFG -f $CMD > gpurun_out/ncu_rec.log 2>&1
else
  SK=${SK:-k_strassen3m}
  NSK=${NSK:-4}
  for i in $(seq 0 $((NSK - 1))); do
    ncu --set full --metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum --clock-control none --import-source on -k regex:$SK -s $((NSK + i)) -c 1 -o gpurun_out/prof_sketch${i}_$CFG -f $CMD > gpurun_out/ncu_sketch$i.log 2>&1
  done
fi
ncu --set full --clock-control none --import-source on -k regex:${QRK:-k_qrcp_lazy} -s ${QRS:-1} -c 1 -o gpurun_out/prof_qrcp_$CFG -f $CMD > gpurun_out/ncu_qrcp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm_dmma -s 12 -c 1 -o gpurun_out/prof_update_$CFG -f $CMD > gpurun_out/ncu_update.log 2>&1
echo "exit $?"
