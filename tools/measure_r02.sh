# Round-2 measurement set (run on the GPU box from the repo root); outputs in gpurun_out/m2_*
set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/m2_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m2_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/m2_bench_bcnn.json 2> gpurun_out/m2_bench_bcnn.err
timeout 600 python bench.py --workload bmlp --no-extra > gpurun_out/m2_bench_bmlp.json 2> gpurun_out/m2_bench_bmlp.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/m2_ref_bcnn.json 2>&1
timeout 600 python bench.py --impl reference --workload bmlp --steps 5 --warmup 2 > gpurun_out/m2_ref_bmlp.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m2_launches_bcnn.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 python tools/profile_stage.py --workload bcnn --batch 65536 --map gpurun_out/m2_stage_map_bcnn.json > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m2_traffic_bcnn.csv python tools/profile_stage.py --workload bcnn --batch 65536 --map gpurun_out/m2_stage_map_bcnn.json > /dev/null 2>&1
timeout 600 python tools/profile_stage.py --workload bmlp --batch 16384 --map gpurun_out/m2_stage_map_bmlp.json > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m2_traffic_bmlp.csv python tools/profile_stage.py --workload bmlp --batch 16384 --map gpurun_out/m2_stage_map_bmlp.json > /dev/null 2>&1
for st in 0 1 3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_byteconv|k_padrow|k_tc_gemm" -c 1 -o gpurun_out/m2_stage${st}_full -f python tools/profile_stage.py --stage $st --batch 8192 --reps 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:k_pack -c 2 -o gpurun_out/m2_pack_full -f python tools/profile_pack.py > /dev/null 2>&1
ls -la gpurun_out | tail -30
