mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"score_reg|score_tma|score_kernel" -c 1 \
    -o gpurun_out/prof_sc python tools/profile_step.py --steps 1 > gpurun_out/ncu_sc.log 2>&1
echo done
