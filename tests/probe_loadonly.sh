#!/bin/bash
# Load-pipeline ceiling: GEMM with MMAs skipped (SLSP_GEMM_DEBUG=16|1), per config and grid size.
for cfg in ${CFGS:-"0 1" "0 2" "1 1" "1 2"}; do
  set -- $cfg
  for cl in ${CLUSTERS:-0 9}; do
    SLSP_GEMM_KHALF=$1 SLSP_GEMM_MSUB=$2 SLSP_GEMM_CLUSTERS=$cl SLSP_GEMM_DEBUG=17 timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /tmp/lo.json 2>/dev/null
    python - /tmp/lo.json "khalf $1 msub $2 clusters $cl" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"[{sys.argv[2]}] {s}")
PY
  done
done
