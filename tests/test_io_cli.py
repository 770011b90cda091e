"""LDT1 tensor files (reference tensorio.py) with the bf16 dtype byte, and the file CLI.

Mirrors the reference's tests/test_io.py layout and error cases; the CLI tests that need no
GPU (gen, explain, decode's error path) run on CPU, the decode round trip is marked gpu.
"""

import os
import struct
import sys

import numpy as np
import pytest
import torch

from oracle import linattn_oracle as orc
from paper_2501_02573_b200 import DataError, FormatError, tensorio
from paper_2501_02573_b200.cli import main

REF_SRC = "/root/reference/pkg/src"


def test_header_layout(tmp_path):
    path = tmp_path / "t.ldt"
    tensorio.write_tensor(np.array([1.0]), path)
    raw = path.read_bytes()
    assert len(raw) == 4 + 1 + 1 + 8 + 8 and raw[:4] == b"LDT1" and raw[4] == 0 and raw[5] == 1
    assert struct.unpack("<Q", raw[6:14]) == (1,) and struct.unpack("<d", raw[14:]) == (1.0,)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_roundtrip_bitwise(tmp_path, dtype):
    t = np.random.default_rng(60).standard_normal((2, 3, 4)).astype(dtype)
    tensorio.write_tensor(t, tmp_path / "t.ldt")
    back = tensorio.read_tensor(tmp_path / "t.ldt")
    assert back.dtype == t.dtype and back.shape == t.shape and back.tobytes() == t.tobytes()


def test_bf16_dtype_byte_roundtrip(tmp_path):
    t = torch.randn(3, 5, 7).to(torch.bfloat16)
    path = tmp_path / "b.ldt"
    tensorio.write_tensor(t, path)
    raw = path.read_bytes()
    assert raw[4] == tensorio.BF16 and raw[5] == 3 and len(raw) == 6 + 3 * 8 + t.numel() * 2
    back = tensorio.read_tensor(path)
    assert back.dtype == torch.bfloat16 and torch.equal(back, t)
    tensorio.write_tensor(back, tmp_path / "c.ldt")
    assert (tmp_path / "c.ldt").read_bytes() == raw


def test_errors(tmp_path):
    p = tmp_path / "bad.ldt"
    p.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(FormatError, match="magic"):
        tensorio.read_tensor(p)
    p.write_bytes(b"LDT1" + bytes([7, 1]) + struct.pack("<Q", 1) + bytes(8))
    with pytest.raises(FormatError, match="dtype byte"):
        tensorio.read_tensor(p)
    p.write_bytes(b"LDT1" + bytes([0, 1]) + struct.pack("<Q", 16) + bytes(64))
    with pytest.raises(FormatError, match="expected"):
        tensorio.read_tensor(p)
    tensorio.write_tensor(np.array([1.0, np.nan]), p)
    with pytest.raises(DataError, match="flat index 1"):
        tensorio.read_tensor(p)
    with pytest.raises(FormatError):
        tensorio.write_tensor(np.zeros((0, 2)), p)
    with pytest.raises(FormatError):
        tensorio.write_tensor(np.zeros(3, dtype=np.int32), p)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present (GPU box)")
def test_bytes_identical_to_reference_writer(tmp_path):
    sys.path.insert(0, REF_SRC)
    try:
        from linattn import read_tensor as ref_read, write_tensor as ref_write
    finally:
        sys.path.remove(REF_SRC)
    for dt in (np.float32, np.float64):
        t = np.random.default_rng(3).standard_normal((2, 4, 3)).astype(dt)
        ref_write(t, tmp_path / "r.ldt")
        tensorio.write_tensor(t, tmp_path / "o.ldt")
        assert (tmp_path / "r.ldt").read_bytes() == (tmp_path / "o.ldt").read_bytes()
        assert np.array_equal(ref_read(tmp_path / "o.ldt"), t)


def test_cli_gen_and_explain(tmp_path, capsys):
    out = [str(tmp_path / n) for n in ("B.ldt", "C.ldt", "V.ldt")]
    assert main(["gen", "--batch", "1", "--heads", "2", "--seqlen", "33", "--rank", "4", "--dim", "5",
                 "--seed", "3", "--out-b", out[0], "--out-c", out[1], "--out-v", out[2]]) == 0
    b, c, v = orc.gen_inputs(1, 2, 33, 4, 5, np.float32, 3)
    assert np.array_equal(tensorio.read_tensor(out[0]), b) and np.array_equal(tensorio.read_tensor(out[2]), v)
    assert main(["gen", "--seqlen", "8", "--dtype", "bf16", "--out-b", out[0], "--out-c", out[1],
                 "--out-v", out[2]]) == 0
    assert tensorio.read_tensor(out[1]).dtype == torch.bfloat16
    capsys.readouterr()
    assert main(["explain", "--seqlen", "8192", "--dtype", "bf16", "--mask", "decay"]) == 0
    assert capsys.readouterr().out.startswith("b200-chunked ")
    assert main(["explain", "--seqlen", "64"]) == 0
    assert capsys.readouterr().out.startswith("b200-chunked-f32 ")


def test_cli_usage_errors(tmp_path, capsys):
    assert main(["decode", "--b", str(tmp_path / "missing.ldt"), "--c", "x", "--v", "y"]) == 2
    assert "cannot read" in capsys.readouterr().err
    assert main(["explain", "--seqlen", "8", "--policy", str(tmp_path / "nope")]) == 2
    assert main(["decode", "--b", "x", "--c", "y", "--v", "z", "--method", "fleet"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cli_decode_roundtrip(tmp_path, dtype, capsys):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    paths = [str(tmp_path / n) for n in ("B.ldt", "C.ldt", "V.ldt", "O.ldt")]
    assert main(["gen", "--batch", "2", "--heads", "2", "--seqlen", "300", "--rank", "64", "--dim", "64",
                 "--dtype", dtype, "--seed", "4", "--out-b", paths[0], "--out-c", paths[1],
                 "--out-v", paths[2]]) == 0
    assert main(["decode", "--b", paths[0], "--c", paths[1], "--v", paths[2], "--gamma", "0.9,0.999",
                 "--decay", "--out", paths[3]]) == 0
    assert "resolved: " + ("b200-chunked-f32" if dtype == "f32" else "b200-chunked") in capsys.readouterr().err
    b, c, v = (tensorio.read_tensor(p) for p in paths[:3])
    to_np = (lambda t: t.float().numpy()) if dtype == "bf16" else (lambda t: t)
    ref = orc.oracle_attn(to_np(b), to_np(c), to_np(v), [0.9, 0.999], True)
    out = tensorio.read_tensor(paths[3])
    assert orc.max_rel_error(to_np(out), ref) <= (2e-2 if dtype == "bf16" else 1e-4)
