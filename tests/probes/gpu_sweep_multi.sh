#!/bin/bash
# Several probe_sweep.py runs in one box call: SWEEP_RUNS holds "tag|args" entries separated by ';;'.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
IFS=$'\n'; for run in $(echo "$SWEEP_RUNS" | sed 's/;;/\n/g'); do
  tag=${run%%|*}; args=${run#*|}
  echo "== $tag: $args" | tee gpurun_out/sweep_${tag}.log
  eval timeout ${SWEEP_TIMEOUT:-600} python tests/probes/probe_sweep.py $args 2>&1 | tee -a gpurun_out/sweep_${tag}.log
done
