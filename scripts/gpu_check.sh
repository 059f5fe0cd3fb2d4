#!/usr/bin/env bash
# One GPU round trip: parity tests, bench line(s), ncu launch list (shares).
# usage: scripts/gpu_check.sh TAG [tests|notests] [extra workloads...]
TAG=${1:-x}
MODE=${2:-tests}
shift 2 2>/dev/null
mkdir -p gpurun_out
if [ "$MODE" = tests ]; then
  timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_${TAG}.log
fi
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
for wl in "$@"; do
  timeout 900 python bench.py --workload $wl --no-extensions > gpurun_out/bench_${TAG}_${wl}.json 2> gpurun_out/bench_${TAG}_${wl}.err; echo "bench $wl rc=$?"
done
python scripts/bench_summary.py gpurun_out/bench_${TAG}*.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --streams 1 --no-extensions > /dev/null 2>&1; echo "ncu rc=$?"
