set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_byteconv -s 1 -c 1 -o gpurun_out/m3_conv1_full -f python tools/profile_stage.py --stage 0 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_padrow -s 2 -c 1 -o gpurun_out/m3_conv2_full -f python tools/profile_stage.py --stage 1 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_padrow -s 2 -c 1 -o gpurun_out/m3_conv3_full -f python tools/profile_stage.py --stage 2 --batch 65536 --reps 1 > /dev/null 2>&1
