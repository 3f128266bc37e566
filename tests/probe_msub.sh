#!/bin/bash
# MSUB (M-subtiles per CTA pair) x cluster probes: parity first, then bench + sustained power.
# CFGS: space-separated list of MSUBxCLUSTER, e.g. "2x2 1x2".
out=${1:-gpurun_out}
for cfg in ${CFGS:-2x2 1x2}; do
  ms=${cfg%x*}; cl=${cfg#*x}
  export SLSP_GEMM_MSUB=$ms SLSP_GEMM_CLUSTER=$cl SLSP_GEMM_GROUP=${GROUP:-16}
  echo "== msub $ms cluster $cl"
  timeout 150 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
  timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/ms_$cfg.json 2>$out/ms_$cfg.err
  python - "$out/ms_$cfg.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"  bench: value {d['value']} dense {d['dense']['value']} x{d['speedup_vs_dense']} gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
  [ -n "$POWER" ] && timeout 120 python tests/probe_power.py gate_up 1.0 2>&1 | head -2
  for dbg in ${DBGS:-}; do
    SLSP_GEMM_DEBUG=$dbg timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > $out/ms_dbg.json 2>/dev/null
    python - "$out/ms_dbg.json" "$dbg" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"  dbg {sys.argv[2]}: gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
  done
done
