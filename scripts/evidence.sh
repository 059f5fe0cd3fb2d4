#!/usr/bin/env bash
# Round evidence on one B200: full GPU test suite, bench lines for every
# workload, the ncu launch list of the default bench, ncu --set full captures
# of the top kernels and the measured pipe rates. Usage: scripts/evidence.sh TAG
TAG=${1:-ev}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench c4 rc=$?"
for wl in c2 c3 c5; do
  timeout 900 python bench.py --workload $wl --no-extensions > gpurun_out/bench_${TAG}_${wl}.json 2> gpurun_out/bench_${TAG}_${wl}.err; echo "bench $wl rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo "ref rc=$?"
python scripts/bench_summary.py gpurun_out/bench_${TAG}*.json
[ -x scripts/pipe_rates ] && scripts/pipe_rates > gpurun_out/pipe_rates_${TAG}.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --frames 16 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --streams 1 --no-extensions > /dev/null 2>&1; echo "ncu list rc=$?"
bash scripts/profile_k.sh ${TAG} k_d_gather:3 k_repick_list:3 k_d_repick:0 k_wta11:1 k_disc_sum:3 "^k_scan_b$":3 \
    k_cloud_normals:1 k_edge_words:3 k_outlier_words:3 k_fill_radial_list:3
python scripts/launch_shares.py gpurun_out/launches_${TAG}.csv > gpurun_out/launch_shares_${TAG}.md
