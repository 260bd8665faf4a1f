timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_network.py -q -x 2>&1 | tail -1
for lib in libbitnn_b200.so libbitnn_b200_wf0.so; do for at in 1 0; do
B2_F4_ATMEM=$at B2_LIB=paper_1705_07175_b200/lib/$lib timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph > gpurun_out/o.txt 2>&1
echo "$lib AT=$at"; grep "stage [3-8]" gpurun_out/o.txt | cut -c1-40 | tr '\n' ' '; echo
done; done
