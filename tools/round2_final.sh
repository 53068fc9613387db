#!/bin/bash
# usage (under gpurun): bash tools/round2_final.sh
# round-2 measurement set at HEAD: GPU tests, bench lines of the three layouts,
# the step's ncu launch list (time + DRAM bytes), ncu --set full of the step
# kernels, the one-launch row-spread kernel (B = 1) and the tcgen05 prefill, and
# the C5 sweep.
out=gpurun_out/r2f
mkdir -p $out
python -m paper_2602_06283_b200.build > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $out/gpu_tests.log 2>&1; tail -2 $out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
timeout 900 python bench.py --layout seq --steps 20 --warmup 5 > $out/bench_seq.json 2> $out/bench_seq.err
timeout 900 python bench.py --ctx 131072 --batch 8 --steps 20 --warmup 5 --no-b1 --no-rows > $out/bench_c3.json 2> $out/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches_b1.csv python tools/profile_step.py --batch 1 --steps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"prologue_kernel|score_reg_kernel|topk_cluster|decode_mma" -s 4 -c 4 \
    -o $out/prof_step python tools/profile_step.py --steps 2 > $out/ncu_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spread_step" -s 2 -c 1 \
    -o $out/prof_spread_b1 python tools/profile_step.py --batch 1 --steps 3 > $out/ncu_spread.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hash_keys_tc" -c 1 \
    -o $out/prof_prefill python tools/profile_step.py --steps 1 > $out/ncu_prefill.log 2>&1
timeout 1500 python tools/sweep.py --out $out/sweep.json > $out/sweep.log 2>&1
for f in bench bench_seq bench_c3; do echo "== $f"; tail -c 400 $out/$f.json; tail -2 $out/$f.err; done
ls -la $out
