#!/bin/bash
# MSUB (M-subtiles per CTA pair) x cluster probes: parity first, then bench + sustained power.
out=${1:-gpurun_out}
for cfg in ${CFGS:-"2 2" "1 2"}; do
  set -- $cfg
  export SLSP_GEMM_MSUB=$1 SLSP_GEMM_CLUSTER=$2 SLSP_GEMM_GROUP=${GROUP:-16}
  echo "== msub $1 cluster $2"
  timeout 150 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
  timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/ms_$1_$2.json 2>$out/ms_$1_$2.err
  python - "$out/ms_$1_$2.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"  bench: value {d['value']} dense {d['dense']['value']} x{d['speedup_vs_dense']} gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
  timeout 120 python tests/probe_power.py gate_up 1.0 2>&1 | head -2
done
