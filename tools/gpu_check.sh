#!/bin/bash
# usage: tools/gpu_check.sh [tag]  -- tests + bench + ncu on the GPU box (run under gpurun)
tag=${1:-x}
mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/tests_$tag.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python tools/profile_step.py --steps 2 > /dev/null 2>&1
if [ "$NCU_FULL" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_kernel|decode_split|topk_cluster|query_tables|hash_append" \
     -s 7 -c 5 -o gpurun_out/prof_$tag python tools/profile_step.py --steps 2 > gpurun_out/ncu_$tag.log 2>&1
fi
cat gpurun_out/tests_$tag.log; cat gpurun_out/bench_$tag.json | head -c 3000; echo; tail -3 gpurun_out/bench_$tag.err
