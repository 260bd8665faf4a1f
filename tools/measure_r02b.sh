# Round-2 (second session) measurement set, run on the GPU box from the repo root; outputs gpurun_out/m3_*
set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/m3_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m3_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/m3_bench_bcnn.json 2> gpurun_out/m3_bench_bcnn.err
timeout 600 python bench.py --workload bmlp --no-extra > gpurun_out/m3_bench_bmlp.json 2> gpurun_out/m3_bench_bmlp.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/m3_ref_bcnn.json 2>&1
timeout 600 python bench.py --impl reference --workload bmlp --steps 5 --warmup 2 > gpurun_out/m3_ref_bmlp.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m3_launches_bcnn.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 python tools/profile_stage.py --workload bcnn --batch 65536 --map gpurun_out/m3_stage_map_bcnn.json > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m3_traffic_bcnn.csv python tools/profile_stage.py --workload bcnn --batch 65536 --map gpurun_out/m3_stage_map_bcnn.json > /dev/null 2>&1
timeout 600 python tools/profile_stage.py --workload bmlp --batch 16384 --map gpurun_out/m3_stage_map_bmlp.json > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m3_traffic_bmlp.csv python tools/profile_stage.py --workload bmlp --batch 16384 --map gpurun_out/m3_stage_map_bmlp.json > /dev/null 2>&1
# one --set full capture per kernel family at the bench batch: the stage's own launch follows one
# warm-up pass of the whole network (skip counts = that kernel's launches per network)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_byteconv -s 1 -c 1 -o gpurun_out/m3_conv1_full -f python tools/profile_stage.py --stage 0 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_padrow -s 2 -c 1 -o gpurun_out/m3_conv2_full -f python tools/profile_stage.py --stage 1 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_padrow -s 2 -c 1 -o gpurun_out/m3_conv3_full -f python tools/profile_stage.py --stage 2 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 6 -c 1 -o gpurun_out/m3_conv4_full -f python tools/profile_stage.py --stage 3 --batch 65536 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 6 -c 1 -o gpurun_out/m3_conv6_full -f python tools/profile_stage.py --stage 5 --batch 65536 --reps 1 > /dev/null 2>&1
ls -la gpurun_out | tail -30
