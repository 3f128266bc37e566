#!/bin/bash
# GEMM debug-knob matrix (gate_up, M=8192): which resource bounds the kernels.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
S=""; for d in 0 1 4 5 8 9 32 33 2 3 16 17 20 21; do S="$S;MSUB=2 DEBUG=$d"; done; S=${S#;}
D=""; for d in 0 1 4 5 2 3 16 17; do D="$D;CLUSTER=2 DEBUG=$d"; done; D=${D#;}
timeout 900 python tests/probes/probe_sweep.py --burst --layers ${LAYERS:-gate_up} --cycles 2 --reps 10 \
  --sparse "$S" --dense "$D" 2>&1 | tee gpurun_out/debug_matrix.log
