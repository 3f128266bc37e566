#!/bin/bash
# GPU-box wrapper: ncu --set full of the 3rd GEMM launch of tests/probes/probe_one.py (KIND, LAYER, TAG; ENV extra env).
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
env $ENV timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
  -o gpurun_out/prof_${TAG:-x} python tests/probes/probe_one.py ${KIND:-sparse} ${LAYER:-gate_up} > gpurun_out/ncu_${TAG:-x}.log 2>&1
tail -3 gpurun_out/ncu_${TAG:-x}.log
