#!/bin/bash
# Perf probes for the GEMM kernels (GPU box): normal run, then the debug knobs
# of gemm.cu (1 = no output stores, 2 = no operand loads, 4 = L2-resident operands).
out=${1:-gpurun_out}
for dbg in 0 1 2 4 3; do
  SLSP_GEMM_DEBUG=$dbg timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/probe_$dbg.json 2> $out/probe_$dbg.err
  python - "$out/probe_$dbg.json" "$dbg" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print("debug", sys.argv[2], "value", d["value"], "dense", d["dense"]["value"], "speedup", d["speedup_vs_dense"],
      "gemm_speedup", d["gemm_speedup_vs_dense"], "clk", d["clocks"]["sm_mhz"])
for r in d["layers"]:
    print("   ", r["name"], "sparse", r["sparse_gemm_ms"], r["sparse_gemm_eff_tflops"], "dense", r["dense_gemm_ms"],
          r["dense_gemm_tflops"], "x", r["gemm_speedup"], "lift", r["lift_ms"], "quant", r["quant_ms"])
PY
done
