#!/bin/bash
# compute-sanitizer over the -m gpu suite (run on the GPU box via gpurun).
#   bash tools/sanitize.sh [tests...]   -> gpurun_out/sanitizer_<tool>.log
# Tools: memcheck (out-of-bounds / misaligned accesses, leaks off),
# racecheck (shared-memory hazards), synccheck (barrier misuse).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
TESTS=${*:-tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_indexed.py tests/test_collisions.py tests/test_gpu_f3.py tests/test_golden_fixtures.py}
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no --report-api-errors no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  start=$(date +%s)
  timeout ${TMO:-1500} $CS --tool $tool $extra --print-limit 50 --error-exitcode 99 \
      python -m pytest $TESTS -m gpu -x -q -p no:cacheprovider > "$OUT/sanitizer_${tool}.log" 2>&1
  echo "$tool rc=$? $(( $(date +%s) - start ))s" | tee -a "$OUT/sanitizer_summary.txt"
  tail -3 "$OUT/sanitizer_${tool}.log"
done
