timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
B2_KBIAS=0 timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
for kb in 1 0; do
B2_KBIAS=$kb timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph 2>&1 | grep -a "stage [0-8]" | cut -c1-40 | tr '\n' ' '; echo
done
