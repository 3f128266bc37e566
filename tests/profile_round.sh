#!/bin/bash
# Round measurement pass on the GPU box: GPU tests, bench, ncu launch list and
# full captures of the top kernels. Outputs under gpurun_out/ (summaries are
# copied into profiles/ by hand).
out=${1:-gpurun_out}
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_round.log 2>&1; echo "pytest exit $?" >> $out/pytest_round.log
tail -3 $out/pytest_round.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > $out/smoke.log 2>&1; tail -2 $out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_round.json 2> $out/bench_round.err; echo "bench exit $?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
# full captures: sparse gate_up GEMM, dense gate_up GEMM, lift (K=3584), pack (gate_up)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o $out/prof_sgemm \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $out/ncu_s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 -o $out/prof_dgemm \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $out/ncu_d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:act_warp_kernel -s 4 -c 1 -o $out/prof_lift \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-dense > $out/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack68_kernel -s 0 -c 1 -o $out/prof_pack \
   python tests/probe_pack.py > $out/ncu_p.log 2>&1
echo done
