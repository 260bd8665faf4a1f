timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -1
for lib in libbitnn_b200.so libbitnn_b200_vb0.so libbitnn_b200_wia.so libbitnn_b200_wia0.so; do
echo $lib; B2_LIB=paper_1705_07175_b200/lib/$lib timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph 2>&1 | grep -a "stage [2]" | cut -c1-40 | tr '\n' ' '; echo
done
