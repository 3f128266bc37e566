#!/bin/bash
# Round-2 final pass: smoke, GPU tests, the bench line, configs 1/4, decode steady state,
# (compute-sanitizer is closed on this pool: not run).
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1
tail -2 gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tests/bench_configs.py --cfg 1,4 --out gpurun_out/cfg14.md > gpurun_out/cfg14.log 2>&1
timeout 300 python tests/probes/probe_decode_ss.py > gpurun_out/dec_final.log 2>&1
