"""Runs one Qwen2.5-7B GEMM (sparse or dense; layer and M from argv, default
gate_up at M=8192) a few times — a minimal target for `ncu -k
regex:gemm_kernel` captures (perf probing)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "sparse"
layer = sys.argv[2] if len(sys.argv) > 2 else "gate_up"
n, k = {"gate_up": (37888, 3584), "down": (3584, 18944), "qkv": (4608, 3584), "o": (3584, 3584)}[layer]
m = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
g = torch.Generator(device="cuda").manual_seed(0)
w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
s_ch = torch.rand(n, device="cuda", generator=g) * 0.01
out = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
if kind == "sparse":
    pw = slsp.pack_compress(w, 6, 8)
    act, s_tok = slsp.fused_quant_slide(x, 6, 8)
    fn = lambda: slsp.sparse_gemm(pw, act, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM, out=out)  # noqa: E731
else:
    q, s_tok = slsp.quantize_rows(x)
    fn = lambda: slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM, out=out)  # noqa: E731
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    fn()
torch.cuda.synchronize()
print("ok")
