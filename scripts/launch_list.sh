#!/usr/bin/env bash
# ncu launch list of a short single-stream bench (16-frame batches) and its
# per-kernel shares. Usage: scripts/launch_list.sh TAG [extra bench args]
TAG=${1:-ll}; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 \
    --streams 1 --no-extensions "$@" > /dev/null 2>&1; echo "ncu list rc=$?"
python scripts/launch_shares.py gpurun_out/launches_${TAG}.csv > gpurun_out/launch_shares_${TAG}.md
head -40 gpurun_out/launch_shares_${TAG}.md
