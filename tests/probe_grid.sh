#!/bin/bash
# Scaling of GEMM throughput with the number of active CTA pairs (per-SM vs shared limit).
out=${1:-gpurun_out}
for c in ${CLUSTERS:-74 9}; do
  for dbg in ${DBGS:-0 8}; do
    SLSP_GEMM_CLUSTERS=$c SLSP_GEMM_DEBUG=$dbg timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > $out/grid_${c}_$dbg.json 2>/dev/null
    python - "$out/grid_${c}_$dbg.json" "$c" "$dbg" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); g = {r["name"]: r for r in d["layers"]}["gate_up"]
c = int(sys.argv[2])
print(f"clusters {c:3d} dbg {sys.argv[3]}: sparse {g['sparse_gemm_ms']:.3f} ms ({g['sparse_gemm_eff_tflops']/c/2:.2f} TF/SM)  dense {g['dense_gemm_ms']:.3f} ms ({g['dense_gemm_tflops']/c/2:.2f} TF/SM)")
PY
  done
done
