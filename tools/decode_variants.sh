#!/bin/bash
# usage (under gpurun): bash tools/decode_variants.sh -- sparse decode timing per (warps, stages, grid) variant
mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > /dev/null 2>&1
python tools/decode_time.py >> gpurun_out/decode_variants.txt 2>&1
for v in "-DSK_DECODE_STAGES=4" "-DSK_DECODE_STAGES=2" "-DSK_DECODE_WARPS=8 -DSK_DECODE_STAGES=3" "-DSK_DECODE_WARPS=8 -DSK_DECODE_STAGES=2" "-DSK_DECODE_TARGET_PCT=100" "-DSK_DECODE_TARGET_PCT=300"; do
  lib=$(python tools/variant_build.py $v 2>/dev/null | tail -1)
  name=/tmp/libsocket_$(echo "$v" | tr -c 'A-Za-z0-9' '_').so
  cp "$lib" "$name"
  echo "variant $v" >> gpurun_out/decode_variants.txt
  SOCKET_LIB_VARIANT=$name python tools/decode_time.py >> gpurun_out/decode_variants.txt 2>&1
done
cat gpurun_out/decode_variants.txt
