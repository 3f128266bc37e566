cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest1.log
tail -5 gpurun_out/pytest1.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench exit $?"
tail -c 3000 gpurun_out/bench1.json
timeout 900 python tests/probes/probe_sweep.py --burst --sparse 'MSUB=2;MC=2' --dense 'CLUSTER=2' --cycles 3 --reps 20 > gpurun_out/sweep1.log 2>&1
cat gpurun_out/sweep1.log | tail -20
