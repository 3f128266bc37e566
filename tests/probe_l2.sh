#!/bin/bash
# L2 policy / raster-band probes for the GEMMs (gate_up at M=8192, full grid).
out=${1:-gpurun_out}
for cfg in "0 8" "1 8" "5 8" "7 8" "5 4" "5 16" "5 32" "5 148"; do
  set -- $cfg
  SLSP_GEMM_HINTS=$1 SLSP_GEMM_GROUP=$2 timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > $out/l2_$1_$2.json 2>/dev/null
  python - "$out/l2_$1_$2.json" "$1" "$2" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"hints {sys.argv[2]} group {sys.argv[3]:>3}: value {d['value']} dense {d['dense']['value']} x{d['speedup_vs_dense']} gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
done
