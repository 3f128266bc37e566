#!/bin/bash
# ncu of the in-GEMM lift (sparse_gemm_lift) vs sparse_gemm on lifted rows, gate_up BF16 at M=64 / 1.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out /tmp/ncu
NCU="ncu --set full --clock-control none --import-source on"
for m in glift_m64 gsparse_m64 glift_m1; do
  timeout 300 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/ncu/$m python tests/probes/probe_ncu_targets.py $m > /tmp/ncu/$m.log 2>&1
done
python tests/ncu_summary.py /tmp/ncu/g*.ncu-rep > gpurun_out/glift_ncu.txt 2>&1
for m in glift_m64 gsparse_m64; do
  ncu -i /tmp/ncu/$m.ncu-rep --page raw --csv > /tmp/ncu/$m.raw.csv 2>/dev/null
  true
done
python tests/ncu_summary.py --grep "inst_executed.sum$|smsp__average_warp|dram__bytes|l1tex__m_xbar2l1tex_read_bytes.sum$|gpu__time_duration" /tmp/ncu/g*.ncu-rep > gpurun_out/glift_ncu_extra.txt 2>&1
tail -n 2 /tmp/ncu/*.log; ls -la gpurun_out | tail
