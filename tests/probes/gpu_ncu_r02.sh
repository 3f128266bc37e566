#!/bin/bash
# Round-2 ncu evidence: tensor-pipe metric names, full captures of the large-M GEMMs
# (sparse / dense gate_up), config 1, a BF16 decode GEMM, the amax-fold GEMM, the lift
# at M=1 / 8192. Summaries are extracted on the box (the reports exceed gpurun's
# 64 MiB pull limit); only the sparse gate_up report is kept.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out /tmp/ncu
NCU="ncu --set full --clock-control none --import-source on"
ncu --query-metrics 2>/dev/null | grep -i -E "tensor|utc|tmem|tcgen|uma|mma" > gpurun_out/ncu_metric_names.txt
timeout 600 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/ncu/r02_sgu python tests/probes/probe_one.py sparse gate_up > /tmp/ncu/sgu.log 2>&1
timeout 600 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/ncu/r02_dgu python tests/probes/probe_one.py dense gate_up > /tmp/ncu/dgu.log 2>&1
for m in cfg1_sparse cfg1_dense dec_sparse dec_dense chain_amax; do
  timeout 300 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/ncu/r02_$m python tests/probes/probe_ncu_targets.py $m > /tmp/ncu/$m.log 2>&1
done
for m in lift_m1 lift_m8192; do
  timeout 300 ncu --set full --clock-control none -k regex:act_ -s 2 -c 1 -o /tmp/ncu/r02_$m python tests/probes/probe_ncu_targets.py $m > /tmp/ncu/$m.log 2>&1
done
python tests/ncu_summary.py /tmp/ncu/r02_*.ncu-rep > gpurun_out/r02_ncu_full.txt 2>&1
python tests/ncu_summary.py --grep "tensor|pipe_uma|pipe_tma|tmem|utc|dram__bytes|xbar2l1tex_read_bytes.sum$|sm__cycles_elapsed.avg.per_second|gpu__time_duration" /tmp/ncu/r02_*.ncu-rep > gpurun_out/r02_ncu_tensor_metrics.txt 2>&1
cp /tmp/ncu/r02_sgu.ncu-rep gpurun_out/
tail -n 2 /tmp/ncu/*.log; wc -l gpurun_out/r02_ncu_*.txt
