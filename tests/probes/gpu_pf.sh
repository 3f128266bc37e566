#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
S="MSUB=2"; for x in "2 PFAT=8" "4 PFAT=8" "6 PFAT=8" "4 PFAT=14" "8 PFAT=4" "21 PFAT=2"; do S="$S;MSUB=2 PF=$x"; done
timeout 900 python tests/probes/probe_sweep.py --burst --layers gate_up,qkv,o --cycles 3 --reps 10 \
  --sparse "$S" --dense "CLUSTER=2" 2>&1 | tee gpurun_out/pf.log
