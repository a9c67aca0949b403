#!/bin/bash
# compute-sanitizer evidence for a round (run on the GPU box through gpurun, from the repo root): memcheck
# and racecheck over the executor tests (TestExecutor + the fuzz executor tests), the fused Lloyd step
# (cluster kernel), the seeding kernels and the error-table kernel.  Output: gpurun_out/<tag>_sanitizer.txt
TAG=${1:-r02}
OUT=gpurun_out/${TAG}_sanitizer.txt
: > $OUT
run() {  # tool, pytest -k expression, files...
  local tool=$1 expr=$2; shift 2
  echo "compute-sanitizer --tool $tool python -m pytest $* -m gpu -k \"$expr\"" >> $OUT
  timeout 1500 compute-sanitizer --tool $tool python -m pytest "$@" -m gpu -q -x -k "$expr" 2>&1 | grep -v "^$" | grep -v "^=========     \|^========= $" | tail -12 >> $OUT
}
run memcheck "TestExecutor or executor_random_masks or executor_medium" tests/test_gpu_parity.py tests/test_gpu_fuzz.py
run memcheck "TestClustering or BoundedLloyd or DeviceSeeding or SeededForward or TestEstimator" tests/test_gpu_parity.py
run racecheck "TestExecutor and not large" tests/test_gpu_parity.py
run racecheck "executor_random_masks" tests/test_gpu_fuzz.py
run racecheck "duplicate_tokens_repair or BoundedLloyd or DeviceSeeding" tests/test_gpu_parity.py
run racecheck "TestEstimator" tests/test_gpu_parity.py
run memcheck "ReferenceSeeding and not benched" tests/test_gpu_parity.py
run racecheck "ReferenceSeeding and picks_equal_numpy and (9-64 or 257 or 1000)" tests/test_gpu_parity.py
cat $OUT
