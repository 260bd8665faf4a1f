timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
timeout 60 python tools/profile_stage.py --stage -1 --batch 65536 --reps 5 --graph > gpurun_out/o.txt 2>&1; grep "stage [0-8]" gpurun_out/o.txt | cut -c1-40 | tr '\n' ' '
