#!/bin/bash
# usage (under gpurun): bash tools/topk_variants.sh -- socket_topk timing per cluster-size variant
mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > /dev/null 2>&1
for B in 16 4 1; do python tools/topk_time.py --batch $B >> gpurun_out/topk_variants.txt 2>&1; done
for m in 64 512 1024; do
  lib=$(python tools/variant_build.py -DSK_TOPK_MIN_CTAS=$m 2>/dev/null | tail -1)
  cp "$lib" /tmp/libsocket_min$m.so
  for B in 16 4 1; do SOCKET_LIB_VARIANT=/tmp/libsocket_min$m.so python tools/topk_time.py --batch $B >> gpurun_out/topk_variants.txt 2>&1; done
done
cat gpurun_out/topk_variants.txt
