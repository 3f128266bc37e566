"""Sustained-load probe (GPU box): runs one GEMM back-to-back for ~1 s while
sampling SM clock, power and throttle reasons via NVML every 5 ms. Tells
whether a kernel is clock/power-limited at full grid. Usage:
  python tests/probe_power.py [layer] [seconds]"""
import json
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

SHAPES = {"gate_up": (37888, 3584), "down": (3584, 18944), "qkv": (4608, 3584), "o": (3584, 3584)}


def sample(stop, out):
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)


def run(name, fn, flops, seconds):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    g.replay()
    torch.cuda.synchronize()
    t0 = time.time()
    reps = 0
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, samples))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    time.sleep(0.05)
    e0.record()
    while time.time() - t0 < seconds:
        g.replay()
        reps += 20
        if reps % 200 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    busy = [s for s in samples if s[1] > 300]
    clk = sorted(s[0] for s in busy) or [0]
    pw = sorted(s[1] for s in busy) or [0]
    reasons = 0
    for s in busy:
        reasons |= s[2]
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1),
                      "sm_mhz_median": clk[len(clk) // 2], "sm_mhz_min": clk[0], "power_w_median": pw[len(pw) // 2],
                      "power_w_max": pw[-1], "reasons_mask": hex(reasons), "samples": len(busy)}), flush=True)


def main():
    layer = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
    seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    n, k = SHAPES[layer]
    m = 8192
    gen = torch.Generator(device="cuda").manual_seed(0)
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=gen), 6, 8)
    x = (torch.rand(m, k, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    q, q_s = slsp.quantize_rows(x)
    s_ch = torch.rand(n, device="cuda") * 0.01
    out = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
    flops = 2.0 * m * n * k
    run(f"sparse_{layer}", lambda: slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM,
                                                    out=out), flops, seconds)
    run(f"dense_{layer}", lambda: slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=q_s,
                                                  out_mode=slsp.OUT_BF16_NM, out=out), flops, seconds)
    run(f"sparse_{layer}", lambda: slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=slsp.OUT_BF16_NM,
                                                    out=out), flops, seconds)


if __name__ == "__main__":
    main()
