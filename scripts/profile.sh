#!/usr/bin/env bash
# Profiling recipe run on the GPU box (under gpurun, one GPU). Outputs land in
# gpurun_out/; summaries worth keeping are copied to profiles/ (tracked).
#   1. launch list: every kernel of one bench step with its device time
#   2. ncu --set full of the top kernels (one launch each)
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p "$OUT"
BENCH="python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --streams 1 --no-extensions"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_${TAG}.csv" $BENCH > "$OUT/launches_${TAG}.log" 2>&1
echo "launch list rc=$?"
for K in k_wta11 k_d_repick k_avg_b k_row_scan k_cloud_normals k_fill_disc k_remove_outliers; do
  ncu --set full --clock-control none --import-source on -k "regex:^${K}\$|${K}" -s 1 -c 1 \
      -o "$OUT/prof_${TAG}_${K}" -f $BENCH > "$OUT/prof_${TAG}_${K}.log" 2>&1
  echo "$K rc=$?"
done
