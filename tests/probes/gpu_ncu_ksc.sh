cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for k in 1 2; do
  SLSP_GEMM_KSC=$k timeout 300 $NCU -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/ksc_cfg1_$k python tests/probes/probe_ncu_targets.py cfg1_sparse > gpurun_out/ncu_ksc_$k.log 2>&1
done
SLSP_GEMM_KSC=1 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel python tests/probes/probe_ncu_targets.py cfg1_sparse > gpurun_out/t1.log 2>&1
SLSP_GEMM_KSC=2 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel python tests/probes/probe_ncu_targets.py cfg1_sparse > gpurun_out/t2.log 2>&1
ls -la gpurun_out
