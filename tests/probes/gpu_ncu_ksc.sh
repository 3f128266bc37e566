#!/bin/bash
# ncu --set full of the decode GEMMs with and without the cluster split-K
# (config 1 INT8 M=128; Llama-3.1-8B qkv BF16 M=1), summaries into gpurun_out.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out /tmp/ncu
NCU="ncu --set full --clock-control none --import-source on"
for t in cfg1_sparse cfg1_dense dec_sparse dec_dense; do
  for k in 0 1; do
    SLSP_GEMM_KSC=$k timeout 300 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/ncu/r02_ksc${k}_$t python tests/probes/probe_ncu_targets.py $t > /tmp/ncu/ksc${k}_$t.log 2>&1
  done
done
python tests/ncu_summary.py /tmp/ncu/r02_ksc*.ncu-rep > gpurun_out/r02_ncu_ksc.txt 2>&1
tail -n 1 /tmp/ncu/*.log
