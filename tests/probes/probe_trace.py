"""Per-tile timeline of CTA 0 of the sparse / dense GEMM (perf probing, B200).

Uses the kernel's SLSP_GEMM_TRACE hook: clock64 stamps per tile iteration
  0 MMA: accumulator free (tile start)   1 MMA: subtile 1 free (MSUB=2)
  2 MMA: last k-block issued             3 epilogue: accumulator full
  4/6 epilogue: subtile 0/1 released      5/7 epilogue: subtile 0/1 stored
Usage: python tests/probe_trace.py [sparse|dense] [tiles-to-print]
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "sparse"
show = int(sys.argv[2]) if len(sys.argv) > 2 else 12
N, K, M = 37888, 3584, 8192
KP = K * 3 // 2
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
s_ch = torch.rand(N, device=dev, generator=g) + 0.5
s_tok = torch.rand(M, device=dev, generator=g) + 0.5
out = torch.empty((N, M), dtype=torch.bfloat16, device=dev)
if kind == "sparsex":
    w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev, generator=g)
    w = slsp.magnitude_prune(w, 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    go = pw.gemm_order()
    act = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev, generator=g)
    run = lambda: slsp.sparse_gemm_x(go, act, s_ch, s_tok, slsp.OUT_BF16_NM, out=out)  # noqa: E731
elif kind == "sparse":
    vals = torch.randint(-127, 128, (N, KP // 2), dtype=torch.int8, device=dev, generator=g)
    meta = torch.full((N, KP // 8), 0x44, dtype=torch.uint8, device=dev)
    pw = slsp.PackedWeights(vals, meta, N, K, KP, 6, 8)
    pw.tiled()
    act = torch.randint(-127, 128, (M, KP), dtype=torch.int8, device=dev, generator=g)
    run = lambda: slsp.sparse_gemm(pw, act, s_ch, s_tok, slsp.OUT_BF16_NM, out=out)  # noqa: E731
else:
    w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev, generator=g)
    act = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev, generator=g)
    run = lambda: slsp.dense_gemm(w, act, s_ch, s_tok, slsp.OUT_BF16_NM, out=out)  # noqa: E731

for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
print(f"{kind} msub={os.environ.get('SLSP_GEMM_MSUB', '1')} dbg={os.environ.get('SLSP_GEMM_DEBUG', '0')}: "
      f"{e0.elapsed_time(e1):.3f} ms")

trace = torch.zeros(65536 + 16 * 256 * 2, dtype=torch.int64, device=dev)
os.environ["SLSP_GEMM_TRACE"] = str(trace.data_ptr())
slsp.reload_knobs()
run()
torch.cuda.synchronize()
del os.environ["SLSP_GEMM_TRACE"]
slsp.reload_knobs()
t = trace[:65536].view(-1, 16).cpu()
st = trace[65536:].view(16, 256, 2).cpu()
n = int((t[:, 0] != 0).sum())
t0 = int(t[0, 0])
rel = lambda v: (int(v) - t0) if int(v) else -1  # noqa: E731
print(f"tiles on CTA 0: {n}; cycles relative to tile 0 start")
print(" it   mma_start sub1_free mma_end | epi_full sub0_rel sub0_st sub1_rel sub1_st | "
      "mainloop  drain0 stores0 drain1  gap(start_i+1 - mma_end_i)  mma_full_wait prod_empty_wait")
for i in range(min(n, show)):
    r = [rel(v) for v in t[i][:8]]
    nxt = rel(t[i + 1, 0]) if i + 1 < n else -1
    print(f"{i:3d} " + " ".join(f"{v:9d}" for v in r[:3]) + " | " + " ".join(f"{v:8d}" for v in r[3:]) +
          f" | {r[2] - r[0]:8d} {r[4] - r[3]:7d} {r[5] - r[4]:7d} {r[6] - r[5]:7d} {nxt - r[2] if nxt >= 0 else -1:7d}"
          f"  {int(t[i, 8]):8d} {int(t[i, 9]):8d}")
if n > 2:
    tot = int(t[n - 1, 2]) - t0
    print(f"avg cycles/tile {tot / (n - 1):.0f}")
    # SM clock while the tiles ran: clock64 vs %globaltimer (ns) at the tile starts
    dc = int(t[n - 1, 0]) - t0
    dt = int(t[n - 1, 10]) - int(t[0, 10])
    if dt > 0:
        q1 = max(1, (n - 1) // 4)
        mhz = [(int(t[j + q1, 0]) - int(t[j, 0])) / max(1, int(t[j + q1, 10]) - int(t[j, 10])) * 1e3
               for j in range(0, n - 1 - q1 + 1, q1)]
        print(f"SM clock over the tiles: {dc / dt * 1e3:.0f} MHz (per quarter: {', '.join(f'{v:.0f}' for v in mhz)})")

# per-stage load latency: producer issue -> MMA sees the stage full
import statistics  # noqa: E402
lat, idle = [], []
for i in range(2, min(n, 16)):
    ks = [k for k in range(256) if int(st[i, k, 0]) and int(st[i, k, 1])]
    for k in ks:
        lat.append(int(st[i, k, 1]) - int(st[i, k, 0]))
if lat:
    lat.sort()
    q = lambda f: lat[min(len(lat) - 1, int(f * len(lat)))]  # noqa: E731
    print(f"stage latency issue->full (cycles, tiles 2..15): p10 {q(0.1)} p50 {q(0.5)} p90 {q(0.9)} max {lat[-1]}")
    i = 3
    ks = [k for k in range(256) if int(st[i, k, 0])]
    print("tile 3 per-stage latency:", [int(st[i, k, 1]) - int(st[i, k, 0]) for k in ks])
