#!/usr/bin/env bash
# compute-sanitizer passes (run on the GPU box): memcheck + racecheck of the
# smoke chain, memcheck of the edge-shape / odd-size / random-parameter parity
# tests. Logs in gpurun_out/.
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.log 2>&1
echo "memcheck smoke rc=$?"; grep "ERROR SUMMARY" gpurun_out/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck.log 2>&1
echo "racecheck smoke rc=$?"; grep "RACECHECK SUMMARY" gpurun_out/racecheck.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_gpu_parity.py -q -m gpu -x \
  -k "odd_frame or edge_shapes or random_parameter_sets or stereo_frame or other_windows" \
  > gpurun_out/memcheck2.log 2>&1
echo "memcheck tests rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck2.log
# round 2 paths: compact/trimmed outputs, caller-buffer outputs, normals'
# exact eigensolver path, warp-aggregated list appends (cleanup kernels)
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_outputs.py tests/test_normals.py -q -m gpu -x > gpurun_out/memcheck3.log 2>&1
echo "memcheck r2 tests rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck3.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest \
  tests/test_normals.py -q -m gpu -x > gpurun_out/racecheck3.log 2>&1
echo "racecheck normals rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/racecheck3.log
