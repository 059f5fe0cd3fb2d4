#!/usr/bin/env bash
# Time one kernel across source variants on the box: each argument is a sed
# expression applied to FILE before a rebuild; prints the kernel's total
# ncu launch time per variant (cold, serialised: compare variants only).
FILE=$1; KERNEL=$2; shift 2
BENCH="python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --streams 1 --no-extensions"
cp "$FILE" /tmp/variant_orig
i=0
for EXPR in "$@"; do
  cp /tmp/variant_orig "$FILE"
  [ -n "$EXPR" ] && sed -i "$EXPR" "$FILE"
  python -c "from paper_2007_12623_b200.build import build; build(verbose=False)" || { echo "build failed: $EXPR"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:${KERNEL}" --csv \
      --log-file gpurun_out/variant_$i.csv $BENCH > /dev/null 2>&1
  python - "$i" "$EXPR" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/variant_{sys.argv[1]}.csv")) if r]
h = next(r for r in rows if "Kernel Name" in r)
t = [float(dict(zip(h, r))["Metric Value"].replace(",", "")) for r in rows[rows.index(h) + 1:]
     if dict(zip(h, r)).get("Metric Name") == "gpu__time_duration.sum"]
print(f"variant {sys.argv[1]} [{sys.argv[2]}]: {len(t)} launches, total {sum(t)/1000:.1f} us")
PY
  i=$((i+1))
done
cp /tmp/variant_orig "$FILE"
