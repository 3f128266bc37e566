#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tests/probes/sanitize_small.py
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  timeout ${TMO:-1500} $CS --tool $tool --print-limit 20 --error-exitcode 9 python tests/probes/sanitize_small.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
