"""SLSP container host side (container.hpp) — CPU tests, pinned on files the
REFERENCE wrote (tests/golden/container_*.slsp, gen_golden.py). Cases mirror
proj/tests/test_container.cpp: round trips, byte-exact re-serialization, CRC
single-byte corruption, structural errors, payload-shape validation."""
from pathlib import Path

import numpy as np
import pytest

from paper_2603_05232_b200 import container as ct

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("tag", ["even", "odd"])
def test_reference_compressed_file_parses_and_reserializes(tag):
    data = (GOLD / f"container_6_8_{tag}.slsp").read_bytes()
    c = ct.deserialize(data)
    ref = np.load(GOLD / f"container_6_8_{tag}.npz")
    assert (c.kind, c.dtype, c.z, c.l, c.hw_m, c.hw_n) == (ct.KIND_COMPRESSED, ct.DT_INT8, 6, 8, 2, 4)
    assert c.rows == ref["values"].shape[0] and c.cols == ref["values"].shape[1] // 2
    assert np.array_equal(np.frombuffer(c.values, np.int8).reshape(ref["values"].shape), ref["values"])
    codes = np.frombuffer(c.metadata, np.uint8)
    unpacked = np.stack([(codes >> (2 * i)) & 3 for i in range(4)], axis=1).reshape(-1)[: ref["codes"].size]
    assert np.array_equal(unpacked, ref["codes"].reshape(-1))  # container.hpp:338-345 unpack_codes
    assert ct.serialize(c) == data  # FileRoundTripIsByteExact


def test_reference_quantized_file():
    data = (GOLD / "container_fqs_6_8.slsp").read_bytes()
    c = ct.deserialize(data)
    ref = np.load(GOLD / "container_fqs_6_8.npz")
    assert c.kind == ct.KIND_QUANTIZED and c.rows == ref["payload"].shape[0]
    assert np.array_equal(np.frombuffer(c.values, np.uint32).reshape(ref["payload"].shape), ref["payload"])
    assert np.array_equal(np.array(c.scales, np.float32).view(np.uint32), ref["scales"].view(np.uint32))
    assert ct.serialize(c) == data


def test_crc_detects_single_byte_corruption():
    rng = np.random.default_rng(104)
    for name in ("container_6_8_even.slsp", "container_6_8_odd.slsp", "container_fqs_6_8.slsp"):
        data = bytearray((GOLD / name).read_bytes())
        for _ in range(25):
            bad = bytearray(data)
            pos = int(rng.integers(len(bad)))
            bad[pos] ^= int(rng.integers(1, 256))
            with pytest.raises(ct.ContainerError):
                ct.deserialize(bytes(bad))


def test_structural_errors():
    data = (GOLD / "container_6_8_odd.slsp").read_bytes()
    with pytest.raises(ct.ContainerError, match="truncated"):
        ct.deserialize(b"")
    with pytest.raises(ct.ContainerError, match="truncated"):
        ct.deserialize(data[:20])
    with pytest.raises(ct.ContainerError, match="bad magic"):
        ct.deserialize(b"X" + data[1:])
    trailing = data[:-4] + b"\x00" + data[-4:]
    with pytest.raises(ct.ContainerError):
        ct.deserialize(trailing)


def test_payload_shape_validation():
    c = ct.deserialize((GOLD / "container_6_8_odd.slsp").read_bytes())
    c.values = c.values[:-1]
    with pytest.raises(ct.ContainerError, match="values payload"):
        ct.serialize(c)
    d = ct.Container(ct.KIND_DENSE, ct.DT_INT8, 6, 0, 0, 0, 1, 4, b"\x00" * 4)
    with pytest.raises(ct.ContainerError, match="zero pattern"):
        ct.serialize(d)
