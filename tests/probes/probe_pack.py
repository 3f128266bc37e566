"""Packs the Qwen2.5-7B gate_up weight once (for ncu capture of pack_kernel)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
w = torch.randint(-127, 128, (37888, 3584), dtype=torch.int8, device="cuda", generator=g)
w = slsp.magnitude_prune(w, 6, 8)
pw = slsp.pack_compress(w, 6, 8, check=False)
torch.cuda.synchronize()
print("packed", pw.values.shape, pw.meta.shape)
