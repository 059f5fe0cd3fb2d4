#!/usr/bin/env bash
# GPU tests plus device-only bench lines for the given workloads (quick A/B).
# Usage: scripts/quick.sh TAG [workloads...]
TAG=$1; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
for wl in "${@:-c4}"; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --no-extensions > gpurun_out/bench_${TAG}_$wl.json 2> gpurun_out/bench_${TAG}_$wl.err
  python - "gpurun_out/bench_${TAG}_$wl.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
g = {k: round(v["avg_launch_ms"], 4) for k, v in d["roofline"]["kernel_groups"].items()}
st = {k: round(v["us_per_pair"], 1) for k, v in d["roofline"]["stages"].items()}
print(d["workload"], round(d["value"], 1), "parity", (d.get("parity") or {}).get("ok"), st, g)
PY
done
