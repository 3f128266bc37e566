"""Packer throughput, table-walk (SLSP_PACK_PATH=1) vs byte-permute (2) kernels,
gate_up 37888x3584 int8 and e4m3, L2 flushed (perf probing); outputs compared."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
n, k = 37888, 3584
g = torch.Generator(device="cuda").manual_seed(0)
for dt in ("int8", "e4m3"):
    if dt == "int8":
        w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    else:
        w = slsp.magnitude_prune(((torch.rand(n, k, device="cuda", generator=g) * 2 - 1) * 300).to(torch.float8_e4m3fn),
                                 6, 8)
    ref = None
    for path in ("1", "2"):
        os.environ["SLSP_PACK_PATH"] = path
        slsp.reload_knobs()
        pw = slsp.pack_compress(w, 6, 8, check=False)
        ts = []
        for _ in range(15):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            slsp.pack_compress(w, 6, 8, check=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        byt = n * k + n * pw.kp // 2 + n * pw.kp // 8
        same = "" if ref is None else f" same={torch.equal(pw.values.view(torch.uint8), ref[0]) and torch.equal(pw.meta, ref[1])}"
        ref = (pw.values.view(torch.uint8).clone(), pw.meta.clone())
        print(f"{dt} path {path}: {ms * 1e3:7.1f} us  {byt / ms / 1e6:7.0f} GB/s{same}", flush=True)
