#!/bin/bash
# GPU-box wrapper: per-tile timelines of CTA 0 under several knob settings (TRACES = ';'-separated env sets).
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
IFS=';' read -ra sets <<< "${TRACES:-SLSP_GEMM_MSUB=2}"
for e in "${sets[@]}"; do
  echo "=== $e"
  env $e timeout 120 python tests/probes/probe_trace.py ${KIND:-sparse} ${SHOW:-8} 2>&1
done | tee gpurun_out/trace_${TAG:-x}.log
