#!/usr/bin/env bash
# ncu --set full on named kernels of a short bench: args are NAME:SKIP
# (regex on the kernel function name, launches of it to skip first).
TAG=$1; shift
BENCH="python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --streams 1 --no-extensions"
for KS in "$@"; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k "regex:${K}" -s "$S" -c 1 \
      -o "gpurun_out/prof_${TAG}_${K//[^a-zA-Z0-9_]/_}" -f $BENCH > /dev/null 2>&1
  echo "$K rc=$?"
done
