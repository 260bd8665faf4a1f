timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "conv_bn_pack or align or padrow" 2>&1 | tail -3
for tw in 0 1; do
echo "== TW=$tw"
B2_PADROW_TW=$tw timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph 2>&1 | grep -a "stage [0-2]" | cut -c1-40 | tr '\n' ' '; echo
done
