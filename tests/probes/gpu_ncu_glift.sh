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
  ncu -i /tmp/ncu/$m.ncu-rep --page source --csv --print-source sass > gpurun_out/${m}_source.csv 2>/dev/null
done
cp /tmp/ncu/glift_m64.ncu-rep gpurun_out/
tail -n 2 /tmp/ncu/*.log; ls -la gpurun_out | tail
