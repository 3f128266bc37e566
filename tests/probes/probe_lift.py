"""Lift / quantize kernel timing (perf probing): fused_quant_slide and
quantize_rows at M=8192 for the workload K values, row-resident path vs warp
path (SLSP_LIFT_ROW), each launch after a 512 MiB L2-flush write; prints GB/s
of algorithmic bytes M*(2K + out + 4)."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

M = 8192
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def burst(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


for k in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["3584", "18944", "4096", "14336"])]:
    x = (torch.rand(M, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    kp = slsp.round_up(k * 3 // 2, 256)
    pay = torch.empty((M, kp // 4), dtype=torch.int32, device="cuda")
    sc = torch.empty(M, dtype=torch.float32, device="cuda")
    q = torch.empty((M, slsp.round_up(k, 128)), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    t_c = burst(lambda: y.copy_(x))
    print(f"K={k:6d} calibration: torch copy bf16 {t_c * 1e3:7.1f} us {2 * x.numel() * 2 / t_c / 1e6:7.0f} GB/s",
          flush=True)
    ref = {}
    for path in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("0", "1")):  # 0 warp, 1 row, 2 row (1024-thread), 3 persistent row
        os.environ["SLSP_LIFT_ROW"] = path
        slsp.reload_knobs()
        t_l = burst(lambda: slsp.fused_quant_slide(x, 6, 8, check=False, payload=pay, scales=sc))
        p1 = pay.clone()
        t_q = burst(lambda: slsp.quantize_rows(x, check=False, out=q, scales=sc))
        q1 = q.clone()
        same = "" if not ref else f" same={torch.equal(ref['p'], p1) and torch.equal(ref['q'], q1)}"
        ref = {"p": p1, "q": q1}
        bl, bq = M * (2 * k + kp + 4), M * (2 * k + q.shape[1] + 4)
        print(f"K={k:6d} row_path={path}: lift {t_l * 1e3:7.1f} us {bl / t_l / 1e6:7.0f} GB/s | "
              f"quant {t_q * 1e3:7.1f} us {bq / t_q / 1e6:7.0f} GB/s{same}", flush=True)
