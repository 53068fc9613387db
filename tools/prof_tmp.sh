mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > gpurun_out/build_p4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"step_prologue|query_tables" -c 2 \
    -o gpurun_out/prof_p4 python tools/profile_step.py --steps 2 --unfused > gpurun_out/ncu_p4.log 2>&1
echo done
