#!/bin/bash
# Cluster-of-4 (multicast B) vs cluster-of-2, both kernels; correctness first.
out=${1:-gpurun_out}
for cl in ${CLS:-4 2}; do
  SLSP_GEMM_CLUSTER=$cl timeout 120 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
  for grp in ${GRPS:-16 32}; do
    SLSP_GEMM_CLUSTER=$cl SLSP_GEMM_GROUP=$grp timeout 120 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > $out/cl_${cl}_$grp.json 2>$out/cl_${cl}_$grp.err
    python - "$out/cl_${cl}_$grp.json" "$cl" "$grp" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
s = "  ".join(f"{r['name']} {r['sparse_gemm_ms']:.3f}/{r['dense_gemm_ms']:.3f}" for r in d["layers"])
print(f"cluster {sys.argv[2]} group {sys.argv[3]:>3}: value {d['value']} dense {d['dense']['value']} x{d['speedup_vs_dense']} gemm x{d['gemm_speedup_vs_dense']} | {s}")
PY
  done
done
