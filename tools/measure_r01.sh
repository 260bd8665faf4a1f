# Round-1 measurement set (run on the GPU box from the repo root); outputs in gpurun_out/m_*
# (fp4 tensor-core path default; the i8 path is benched alongside with B2_TC_FORMAT=i8)
set -x
timeout 300 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/m_pytest.txt 2>&1
python bench.py > gpurun_out/m_bench_bcnn.json 2> gpurun_out/m_bench_bcnn.err
python bench.py --workload bmlp > gpurun_out/m_bench_bmlp.json 2> gpurun_out/m_bench_bmlp.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m_ref_bcnn.json 2>&1
B2_ENGINE=popc python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/m_bench_bcnn_popc.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_bcnn.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_bmlp.csv python bench.py --workload bmlp --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
for w in bcnn bmlp; do
  b=8192; [ $w = bmlp ] && b=16384
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_traffic_$w.csv python tools/profile_stage.py --workload $w --batch $b --map gpurun_out/m_stage_map_$w.json > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_padrow_conv -s 2 -c 1 -o gpurun_out/m_conv2_full -f python tools/profile_stage.py --stage 1 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 8 -c 1 -o gpurun_out/m_conv4_full -f python tools/profile_stage.py --stage 3 --reps 1 > /dev/null 2>&1
timeout 900 python tools/sweep.py > gpurun_out/m_sweeps.jsonl 2> gpurun_out/m_sweeps.err
(cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mxf4_rate mxf4_rate.cu) && timeout 120 ./tools/microbench/mxf4_rate > gpurun_out/m_mxf4_rate.jsonl 2>&1
python tools/_fp4_peak.py > gpurun_out/m_lib_peaks.txt 2>&1
python tools/_b1_breakdown.py > gpurun_out/m_batch1.txt 2>&1
python tools/_pipe_probe.py > gpurun_out/m_pipe.txt 2>&1
B2_TC_FORMAT=i8 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu > gpurun_out/m_bench_bcnn_i8.json 2>&1
B2_TC_FORMAT=i8 python bench.py --workload bmlp --steps 20 --warmup 5 --no-extra --no-cpu > gpurun_out/m_bench_bmlp_i8.json 2>&1
ls gpurun_out
