set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 6 -c 1 -o gpurun_out/m3_conv4_full -f python tools/profile_stage.py --stage 3 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 6 -c 1 -o gpurun_out/m3_conv6_full -f python tools/profile_stage.py --stage 5 --batch 65536 --reps 1 > /dev/null 2>&1
