#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
S="MSUB=2"; for x in 100 200 400 800 1600; do S="$S;MSUB=2 PACE=$x"; done
timeout 900 python tests/probes/probe_sweep.py --burst --layers gate_up,qkv,down --cycles 3 --reps 10 \
  --sparse "$S" --dense "CLUSTER=2;CLUSTER=2 MSUB=2" 2>&1 | tee gpurun_out/pace.log
