#!/usr/bin/env bash
# Copy the files of an evidence run (scripts/evidence.sh TAG on the box, merged
# back into gpurun_out/) into profiles/r2/. Run here. Usage:
#   scripts/collect_evidence.sh TAG
set -e
TAG=$1
D=profiles/r2
mkdir -p $D
cp gpurun_out/bench_${TAG}.json $D/bench_c4.json
for w in c2 c3 c5; do cp gpurun_out/bench_${TAG}_${w}.json $D/bench_${w}.json; done
cp gpurun_out/bench_${TAG}_ref.json $D/bench_reference_c4.json
cp gpurun_out/launches_${TAG}.csv $D/launches_c4.csv
python scripts/launch_shares.py gpurun_out/launches_${TAG}.csv > $D/launch_shares_c4.md
python scripts/ncu_summary.py $(ls gpurun_out/prof_${TAG}_*.ncu-rep) > $D/ncu_full_summary.md
python scripts/pipe_util.py gpurun_out/prof_${TAG}_*.ncu-rep > $D/pipe_util.jsonl
[ -f gpurun_out/sanitizer_${TAG}.txt ] && cp gpurun_out/sanitizer_${TAG}.txt $D/sanitizer.txt
python scripts/bench_summary.py $D/bench_c4.json $D/bench_c2.json $D/bench_c3.json $D/bench_c5.json
