#!/bin/bash
# TMA ingest experiments (tests/micro/tma_bw.cu) + GEMM loads-only variants.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
B=tests/micro/tma_bw
IT=4000
{
echo "== per-SM cap (private, 192 KB ring)"
for c in 2 8 16 32 74 148; do $B 1 0 4 3 $c $IT; done
echo "== chip cap vs ring shape (148 CTAs, private)"
for sn in "2 6" "3 4" "4 3" "6 2" "12 1" "3 2" "2 2" "1 4"; do $B 1 0 $sn 148 $IT; done
echo "== sharing: groups of G CTAs read the same region"
for g in 2 4 8 16 37; do $B 1 1 4 3 148 $IT $g; done
echo "== cluster 2 unicast private / multicast"
$B 2 0 4 3 148 $IT; $B 2 2 4 3 148 $IT
echo "== cluster 4 unicast / multicast (136 and 144 CTAs)"
$B 4 0 4 3 136 $IT; $B 4 2 4 3 136 $IT; $B 4 0 4 3 144 $IT; $B 4 2 4 3 144 $IT
echo "== cluster 8 multicast"
$B 8 2 4 3 128 $IT; $B 8 2 4 3 144 $IT
echo "== dram (private, 5376-byte rows)"
$B 1 3 4 3 148 2000
} 2>&1 | tee gpurun_out/tma_bw.log
timeout 900 python tests/probes/probe_sweep.py --burst --layers gate_up --cycles 2 --reps 10 \
  --sparse 'MSUB=2;MSUB=2 DEBUG=16;MSUB=2 DEBUG=48;MSUB=2 DEBUG=24;MC=2 DEBUG=16;MSUB=1 DEBUG=16;MSUB=2 DEBUG=2;MSUB=2 DEBUG=1' \
  --dense 'CLUSTER=2;CLUSTER=2 DEBUG=16;CLUSTER=2 DEBUG=2' 2>&1 | tee gpurun_out/loads_only.log
