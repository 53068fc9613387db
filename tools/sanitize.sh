#!/bin/bash
# usage (under gpurun): bash tools/sanitize.sh -- compute-sanitizer over tools/sanitize.py
out=gpurun_out/san
mkdir -p $out
python -m paper_2602_06283_b200.build > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --log-file $out/$tool.txt python tools/sanitize.py > $out/${tool}_out.txt 2>&1
  echo "$tool rc=$? $(tail -1 $out/$tool.txt)"
done
