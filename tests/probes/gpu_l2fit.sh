#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python tests/probes/probe_sweep.py --burst --layers gu4k,gu8k,gu16k,gate_up --cycles 3 --reps 10 \
  --sparse "MSUB=2;MSUB=2 DEBUG=1;MSUB=2 DEBUG=17;MSUB=2 DEBUG=3" --dense "CLUSTER=2;CLUSTER=2 DEBUG=17" 2>&1 | tee gpurun_out/l2fit.log
