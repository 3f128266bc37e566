#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python tests/probes/probe_sweep.py --burst --mn --layers gate_up,down,qkv,o --cycles 3 --reps 10 \
  --sparse "MSUB=2;MSUB=2 DEBUG=1;MSUB=1" --dense "CLUSTER=2;CLUSTER=2 DEBUG=1" 2>&1 | tee gpurun_out/mn.log
