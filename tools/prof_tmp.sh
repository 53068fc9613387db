mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1.csv \
    python tools/profile_step.py --batch 1 --steps 3 > /dev/null 2>&1
python tools/tune_step.py --batch 1 4 --sparsity 10 5 --topk-ctas 148 64 32 16 --decode-target 256 128 64 > gpurun_out/tune_b1.txt 2>&1
python tools/trace_topk.py --batch 1 4 > gpurun_out/trace_topk_b1.txt 2>&1
python tools/trace_prologue.py --batch 1 > gpurun_out/trace_pro_b1.txt 2>&1
