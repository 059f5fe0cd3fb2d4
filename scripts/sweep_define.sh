#!/usr/bin/env bash
# Time the default bench across values of a compile-time #define: each
# argument VALUE rebuilds with `#define NAME VALUE` in FILE and prints the
# device pairs/s and the per-launch time of every kernel group.
# Usage: scripts/sweep_define.sh FILE NAME VALUE...
FILE=$1; NAME=$2; shift 2
cp "$FILE" /tmp/sweep_orig
for V in "$@"; do
  cp /tmp/sweep_orig "$FILE"
  sed -i "s/^#define ${NAME} .*/#define ${NAME} ${V}/" "$FILE"
  python -c "from paper_2007_12623_b200.build import build; build(verbose=False)" || { echo "build failed: $V"; continue; }
  timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --no-extensions > gpurun_out/sweep_${NAME}_${V}.json 2>/dev/null
  python - "$V" "gpurun_out/sweep_${NAME}_${V}.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
g = {k: round(v["avg_launch_ms"], 4) for k, v in d["roofline"]["kernel_groups"].items()}
print(f"{sys.argv[1]}: {d['value']:.1f} pairs/s  parity_ok={d['parity'].get('ok')}  {g}")
PY
done
cp /tmp/sweep_orig "$FILE"
