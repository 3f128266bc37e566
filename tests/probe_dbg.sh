#!/bin/bash
# Short-bench GEMM timings for a list of "msub cluster debug" configs.
out=${1:-gpurun_out}
for cfg in ${CFGS:-"1 2 0" "1 2 1" "2 2 0" "2 2 1" "2 2 2"}; do
  set -- $cfg
  SLSP_GEMM_MSUB=$1 SLSP_GEMM_CLUSTER=$2 SLSP_GEMM_DEBUG=$3 SLSP_GEMM_GROUP=${GROUP:-16} timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/dbg.json 2>/dev/null
  python - "$out/dbg.json" "$cfg" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"[{sys.argv[2]}] gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
done
