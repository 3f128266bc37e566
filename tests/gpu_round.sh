cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
out=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > $out/pytest1.log 2>&1; echo "pytest exit $?" >> $out/pytest1.log; tail -3 $out/pytest1.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > $out/bench1.json 2> $out/bench1.err; echo "bench exit $?"; cat $out/bench1.json | head -c 1500
CFGS="1x2 2x2" bash tests/probe_msub.sh $out
