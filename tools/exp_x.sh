timeout 600 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -2
for mc in 1 0; do
B2_MCAST=$mc timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph 2>&1 | grep -a "stage [3-5]" | cut -c1-40 | tr '\n' ' '; echo
done
