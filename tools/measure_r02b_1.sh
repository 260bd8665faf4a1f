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
