#!/bin/bash
# Pipeline-depth probe: GEMM time vs number of smem stages (SLSP_GEMM_STAGES_LESS).
out=${1:-gpurun_out}
for ms in 1 2; do for less in 0 1 2; do
  SLSP_GEMM_MSUB=$ms SLSP_GEMM_STAGES_LESS=$less timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/st.json 2>/dev/null
  python - "$out/st.json" "msub $ms less $less" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"[{sys.argv[2]}] gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
done; done
