# ncu of the single-pass SRFT (k_srft_fused) at C4: one full set of the second call's kernel
python tools/srft_fused_check.py C4 > gpurun_out/srft_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_srft_fused -s 1 -c 1 \
  -o gpurun_out/prof_srft_fused_C4 -f python tools/srft_fused_check.py C4 > gpurun_out/ncu_srft.log 2>&1
echo "exit $?"
