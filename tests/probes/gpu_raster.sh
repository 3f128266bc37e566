#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
S="MSUB=2"; for g in 1 2 3 6; do S="$S;MSUB=2 GROUP=$g"; done
for h in 0 3; do S="$S;MSUB=2 GROUP=1 HINTS=$h"; done
timeout 900 python tests/probes/probe_sweep.py --burst --layers gate_up,qkv,down --cycles 3 --reps 10 \
  --sparse "$S" --dense "CLUSTER=2;CLUSTER=2 GROUP=1;CLUSTER=2 GROUP=2" 2>&1 | tee gpurun_out/raster.log
