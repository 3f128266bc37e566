#!/bin/bash
# Early subtile-0 commit / reordered last k-blocks (SLSP_GEMM_TAIL0): parity, burst timing, energy.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bench_parity.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python tests/probes/probe_sweep.py --burst --sparse 'MSUB=2 TAIL0=0;MSUB=2 TAIL0=1;MSUB=2 TAIL0=2' --dense 'CLUSTER=2' \
  --cycles 3 --reps 20 --check 2>&1 | tee gpurun_out/tail0_sweep.log | tail -22
timeout 600 python tests/probes/probe_energy.py --layers gate_up,down --sparse 'TAIL0=0;TAIL0=2' --dense 'CLUSTER=2' 2>&1 | tee gpurun_out/tail0_energy.log
