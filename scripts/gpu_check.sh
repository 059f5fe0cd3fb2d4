#!/usr/bin/env bash
# One GPU round trip: parity tests, bench line, ncu launch list (shares).
TAG=${1:-x}
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
python - <<'PY' "$TAG"
import json,sys
t=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bench_{t}.json").read().strip().splitlines()[-1])
    print("value",round(d["value"],1),"e2e",round(d["e2e"]["value"],1),"ms/pair",round(d["ms_per_pair"],4),"wta frac",round(d["roofline"]["frac"],4))
    print({k:round(v,4) for k,v in d["stage_ms_per_pair"].items()}, d["exact_resolves"], d["clocks"])
except Exception as e:
    print("bench parse failed", e); print(open(f"gpurun_out/bench_{t}.err").read()[-2000:])
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --streams 1 --no-extensions > /dev/null 2>&1; echo "ncu rc=$?"
