#!/bin/bash
for g in ${GAPS:-0 100 200 400 800}; do
  SLSP_GEMM_MSUB=2 SLSP_GEMM_STORE_GAP=$g timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-dense > /tmp/g.json 2>/dev/null
  python - /tmp/g.json "gap $g" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}" for r in d["layers"])
print(f"[{sys.argv[2]}] {s}")
PY
done
SLSP_GEMM_MSUB=2 SLSP_GEMM_STORE_GAP=${TGAP:-200} timeout 100 python tests/probe_trace.py sparse 0
