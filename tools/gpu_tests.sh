#!/bin/bash
# usage (under gpurun): bash tools/gpu_tests.sh <tag> [pytest args...]
# build + the GPU test suite (all failures listed, not -x)
tag=${1:-t}; shift
mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf "$@" > gpurun_out/tests_$tag.log 2>&1
tail -40 gpurun_out/tests_$tag.log
