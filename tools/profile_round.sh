#!/bin/bash
# usage (under gpurun): bash tools/profile_round.sh <tag>
# bench JSON + launch list (time + DRAM bytes) + ncu --set full of the step kernels
# and of the tcgen05 prefill, all from the current tree
tag=${1:-r1}
mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > gpurun_out/build_$tag.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$tag.txt
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"prologue_kernel|score_reg_kernel|topk_cluster|decode_mma" -s 4 -c 4 \
    -o gpurun_out/prof_$tag python tools/profile_step.py --steps 2 > gpurun_out/ncu_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hash_keys_tc|vnorm" -c 2 \
    -o gpurun_out/prof_prefill_$tag python tools/profile_step.py --steps 1 > gpurun_out/ncu_prefill_$tag.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:sample_decode -c 6 --log-file gpurun_out/launches_sample_$tag.csv python tools/sample_time.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_decode -s 3 -c 1 \
    -o gpurun_out/prof_sample_$tag python tools/sample_time.py > gpurun_out/ncu_sample_$tag.log 2>&1
echo done
