#!/bin/bash
# Half-k-stage probe: parity + bench for KHALF x MSUB.
out=${1:-gpurun_out}
for cfg in ${CFGS:-"1 1" "1 2" "0 1" "0 2"}; do
  set -- $cfg
  export SLSP_GEMM_KHALF=$1 SLSP_GEMM_MSUB=$2
  timeout 200 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -1
  timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/kh.json 2>$out/kh.err
  python - "$out/kh.json" "khalf $1 msub $2" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"[{sys.argv[2]}] value {d['value']} x{d['speedup_vs_dense']} gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
done
