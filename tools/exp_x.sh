for lib in libbitnn_b200.so libbitnn_b200_wi1.so; do
B2_LIB=paper_1705_07175_b200/lib/$lib timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph > gpurun_out/o_$lib.txt 2>&1
grep "stage [3-5]" gpurun_out/o_$lib.txt | cut -c1-40 | tr '\n' ' '; echo
done
B2_LIB=paper_1705_07175_b200/lib/libbitnn_b200_wi1.so timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
