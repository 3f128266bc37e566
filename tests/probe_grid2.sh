#!/bin/bash
# Per-SM efficiency at reduced grid: normal / no-load / load-only, per MSUB.
for ms in ${MSUBS:-1 2}; do for cl in ${CLUSTERS:-9 74}; do for dbg in 0 2 17; do
  SLSP_GEMM_MSUB=$ms SLSP_GEMM_CLUSTERS=$cl SLSP_GEMM_DEBUG=$dbg timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /tmp/g.json 2>/dev/null
  python - /tmp/g.json "msub $ms clusters $cl dbg $dbg" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
r = [x for x in d["layers"] if x["name"] == "gate_up"][0]
print(f"[{sys.argv[2]}] gate_up sparse {r['sparse_gemm_ms']:.3f} dense {r['dense_gemm_ms']:.3f}")
PY
done; done; done
