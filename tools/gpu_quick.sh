#!/bin/bash
# usage (under gpurun): bash tools/gpu_quick.sh <tag> [pytest -k expr]
# build, GPU parity tests, one bench line and the ncu launch list of the step
tag=${1:-q}
mkdir -p gpurun_out
python -m paper_2602_06283_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 600 python -m pytest tests -m gpu -q -x $K 2>&1 | tail -25 > gpurun_out/tests_$tag.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 2 --no-dense > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python tools/profile_step.py --steps 2 > /dev/null 2>&1
cat gpurun_out/tests_$tag.log
python - "$tag" <<'PY'
import csv, collections, json, sys
tag = sys.argv[1]
try:
    b = json.loads(open(f"gpurun_out/bench_{tag}.json").read().strip().splitlines()[-1])
    print("bench:", b["value"], b["unit"], "ms/step", b["ms_per_step"], "e2e", b["e2e"]["value"])
    print("stages:", {k: v.get("ms") for k, v in b["stages"].items()}, "prefill", b.get("prefill"))
except Exception as e:
    print("bench parse failed", e); print(open(f"gpurun_out/bench_{tag}.err").read()[-3000:])
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        h = r; start = i + 1; break
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[start:]:
    if len(r) > vi and not r[ki].startswith("void at::"):
        d[r[ki].split("(")[0][:50]].append(float(r[vi].replace(",", "")))
for k, v in d.items():
    print(f"  {k:50s} n={len(v)} mean={sum(v)/len(v)/1000:.1f} us")
PY
