#!/bin/bash
# Round measurement pass on the GPU box: GPU tests, smoke, bench (both arms),
# the ncu launch list of the bench and one `ncu --set full` capture each of
# the top kernels. Outputs under gpurun_out/ (summarised into profiles/ here
# with tests/ncu_summary.py). Numbers printed under ncu are never bench values.
cd ${GRAFT_REPO_ROOT:-.}
out=${1:-gpurun_out}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_round.log 2>&1; echo "pytest exit $?" >> $out/pytest_round.log
tail -3 $out/pytest_round.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -2 $out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_round.json 2> $out/bench_round.err; echo "bench exit $?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
# full captures (3rd launch of each: warm): sparse gate_up GEMM, dense gate_up GEMM, lift (K=3584), 6:8 packer
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/prof_sgemm python tests/probes/probe_one.py sparse gate_up > $out/ncu_s.log 2>&1
timeout 600 $NCU -k regex:gemm_kernel -s 2 -c 1 -o /tmp/prof_dgemm python tests/probes/probe_one.py dense gate_up > $out/ncu_d.log 2>&1
timeout 600 $NCU -k regex:act_row1_kernel -s 2 -c 1 -o /tmp/prof_lift python tests/probes/probe_lift.py 3584 > $out/ncu_l.log 2>&1
timeout 600 $NCU -k regex:pack68b_kernel -s 0 -c 1 -o /tmp/prof_pack python tests/probes/probe_pack.py > $out/ncu_p.log 2>&1
# the reports stay on the box (gpurun_out/ is capped at 64 MiB); bring back the summaries
python tests/ncu_summary.py /tmp/prof_sgemm.ncu-rep /tmp/prof_dgemm.ncu-rep /tmp/prof_lift.ncu-rep /tmp/prof_pack.ncu-rep \
   > $out/ncu_full.txt 2>&1
python tests/ncu_summary.py --launches $out/launches.csv > $out/launches_summary.txt 2>&1
cp /tmp/prof_sgemm.ncu-rep $out/ 2>/dev/null  # (one report: gpurun pulls at most 64 MiB)
ls -la $out/*.ncu-rep
echo done
