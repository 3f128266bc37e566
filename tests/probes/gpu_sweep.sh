#!/bin/bash
# GPU-box wrapper for tests/probes/probe_sweep.py: SWEEP_ARGS holds its arguments.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
eval timeout ${SWEEP_TIMEOUT:-900} python tests/probes/probe_sweep.py $SWEEP_ARGS 2>&1 | tee gpurun_out/sweep_${SWEEP_TAG:-x}.log
