# ncu --set full captures at the bench batch, summarised on the box (the reports are ~28 MB each)
set -x
cap() {  # name, kernel regex, skip, stage
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/m3_$1_full -f \
    python tools/profile_stage.py --stage $4 --batch 65536 --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py full gpurun_out/m3_$1_full.ncu-rep > gpurun_out/m3_$1_full.md 2>&1
  echo >> gpurun_out/m3_$1_full.md; echo "#### barrier waits and stalls" >> gpurun_out/m3_$1_full.md; echo >> gpurun_out/m3_$1_full.md
  python tools/ncu_summary.py stalls gpurun_out/m3_$1_full.ncu-rep 20 >> gpurun_out/m3_$1_full.md 2>&1
  rm -f gpurun_out/m3_$1_full.ncu-rep
}
cap conv1 k_byteconv 1 0
cap conv2 k_padrow 3 1
cap conv3 k_padrow 3 2
cap conv4 k_tc_gemm 6 3
cap conv6 k_tc_gemm 6 5
ls -la gpurun_out
