"""Container -> device operands on the B200: the reference's
kind-2 file loads into the same MMA-ready values / metadata the on-GPU packer
produces, and the sparse GEMM on it equals the oracle bit for bit; the kind-3
file feeds the GEMM as the lifted activations; GEMM-ready weights round-trip
to the reference's file bytes."""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle_lib import DT_F32, DT_I8, KIND_INT8
from paper_2603_05232_b200 import container as ct

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("tag", ["even", "odd"])
def test_load_compressed_matches_packer_and_gemm(slsp, orc, tag):
    ref = np.load(GOLD / f"container_6_8_{tag}.npz")
    pw = ct.load_compressed(GOLD / f"container_6_8_{tag}.slsp")
    mine = slsp.pack_compress(torch.from_numpy(ref["w"]).cuda(), 6, 8)
    assert pw.kp == mine.kp
    assert torch.equal(pw.values, mine.values)
    assert torch.equal(pw.meta, mine.meta)
    assert torch.equal(pw.tiled(), mine.tiled())
    # the GEMM on the loaded operands == the oracle's packed-word sparse_gemm
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, size=(100, ref["w"].shape[1])).astype(np.float32)
    payload, _ = slsp.fused_quant_slide(torch.from_numpy(x).cuda(), 6, 8, kp=pw.kp)
    got = slsp.sparse_gemm(pw, payload).cpu().numpy()
    opay, _ = orc.fused_quant_slide(x, 6, 8, KIND_INT8, DT_F32)
    assert np.array_equal(got, orc.sparse_gemm_words(ref["values"], ref["codes"], opay))
    # round trip to the reference's bytes
    assert ct.serialize(ct.compressed_from_device(pw)) == (GOLD / f"container_6_8_{tag}.slsp").read_bytes()


def test_load_quantized_feeds_gemm(slsp, orc):
    ref = np.load(GOLD / "container_fqs_6_8.npz")
    c = ct.load_container(GOLD / "container_fqs_6_8.slsp")
    payload, scales = ct.quantized_to_device(c)
    k = ref["x"].shape[1]
    w = slsp.magnitude_prune(torch.randint(-127, 128, (256, k), dtype=torch.int8, device="cuda"), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    assert payload.shape[1] * 4 == pw.kp
    got = slsp.sparse_gemm(pw, payload).cpu().numpy()
    vals, codes = orc.compress(orc.pack_matrix(w.cpu().numpy(), 6, 8, DT_I8), DT_I8)
    assert np.array_equal(got, orc.sparse_gemm_words(vals, codes, ref["payload"]))
    assert torch.equal(scales.cpu(), torch.from_numpy(ref["scales"]))
