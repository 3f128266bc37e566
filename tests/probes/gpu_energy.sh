#!/bin/bash
# Energy per launch of the sparse / dense GEMM and their debug-knob variants under sustained load.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python tests/probes/probe_energy.py --layers ${LAYERS:-gate_up} --seconds ${SECS:-1.5} \
  --sparse "${SPARSE:-MSUB=2;MSUB=2 DEBUG=1;MSUB=2 DEBUG=3;MSUB=2 DEBUG=17;MSUB=1;MC=2}" \
  --dense "${DENSE:-CLUSTER=2;CLUSTER=2 DEBUG=1;CLUSTER=2 DEBUG=3;CLUSTER=2 DEBUG=17}" 2>&1 | tee gpurun_out/energy.log
