#!/bin/bash
# GPU-box: ncu --set full of the moderate-M GEMMs (M=512 down: sparse 256-token
# half-k-stage tiles + split-K vs dense), summarised on the box (reports stay in /tmp).
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for kind in sparse dense; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
    -o /tmp/prof_midm_${kind} python tests/probes/probe_one.py $kind down 512 > gpurun_out/ncu_midm_${kind}.log 2>&1
done
python tests/ncu_summary.py /tmp/prof_midm_sparse.ncu-rep /tmp/prof_midm_dense.ncu-rep > gpurun_out/r01_ncu_midm.txt 2>&1
tail -40 gpurun_out/r01_ncu_midm.txt
