"""Host-side parts of the CLI flows: the .bsat format
(reference tensorio.py:90-141) with its error classes, byte-compatibility
with the reference package, and CLI argument handling that fails before any
device work. The device flows themselves are in tests/test_gpu_cli.py."""

import struct

import numpy as np
import pytest

from paper_2509_07120_b200 import cli
from paper_2509_07120_b200.tensorio import (
    BadMagicError,
    TensorFileError,
    TruncatedPayloadError,
    UnsupportedDTypeError,
    as_f32,
    read_tensor,
    write_tensor,
)


def test_roundtrip_and_layout(tmp_path):
    a = np.random.default_rng(0).standard_normal((2, 5, 3)).astype(np.float32)
    p = tmp_path / "a.bsat"
    write_tensor(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"BSAT"
    assert struct.unpack_from("<IBI", raw, 4) == (1, 0, 3)
    assert struct.unpack_from("<3Q", raw, 13) == (2, 5, 3)
    assert len(raw) == 13 + 24 + a.size * 4
    b = read_tensor(p)
    assert b.dtype == np.float32 and np.array_equal(a, b)


@pytest.mark.parametrize("mutate,err", [
    (lambda r: b"XXXX" + r[4:], BadMagicError),
    (lambda r: r[:10], TruncatedPayloadError),
    (lambda r: r[:-4], TruncatedPayloadError),
    (lambda r: r + b"\0\0\0\0", TensorFileError),
    (lambda r: r[:8] + b"\x01" + r[9:], UnsupportedDTypeError),
    (lambda r: r[:4] + struct.pack("<I", 2) + r[8:], TensorFileError),
])
def test_read_errors(tmp_path, mutate, err):
    p = tmp_path / "a.bsat"
    write_tensor(p, np.ones((2, 3), np.float32))
    p.write_bytes(mutate(p.read_bytes()))
    with pytest.raises(err):
        read_tensor(p)


def test_non_finite_rejected(tmp_path):
    p = tmp_path / "a.bsat"
    write_tensor(p, np.ones((4,), np.float32))
    raw = bytearray(p.read_bytes())
    raw[-4:] = struct.pack("<f", float("nan"))
    p.write_bytes(bytes(raw))
    with pytest.raises(TensorFileError):
        read_tensor(p)
    with pytest.raises(ValueError):
        as_f32(np.array([1.0, np.inf]))
    with pytest.raises(ValueError):
        as_f32(np.zeros((0, 3)))


def test_byte_compatible_with_reference(tmp_path, reference_pkg):
    from bsattn.tensorio import read_tensor as ref_read, write_tensor as ref_write
    a = np.random.default_rng(1).standard_normal((3, 7, 4)).astype(np.float32)
    ours, theirs = tmp_path / "o.bsat", tmp_path / "r.bsat"
    write_tensor(ours, a)
    ref_write(theirs, a)
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(ref_read(ours), read_tensor(theirs))


def test_cli_argument_errors(tmp_path):
    q = tmp_path / "q.bsat"
    write_tensor(q, np.ones((1, 10, 8), np.float32))
    # sparse attend without a mask: refused before any device work
    with pytest.raises(SystemExit):
        cli.main(["attend", "--mode", "sparse", "--q", str(q), "--k", str(q), "--v", str(q),
                  "--out", str(tmp_path / "o.bsat")])
    for name in cli.OUT_OF_SCOPE:
        with pytest.raises(SystemExit):
            cli.main([name])
    with pytest.raises(SystemExit):
        cli.main(["mask", "--q", str(q), "--k", str(q), "--tau", "0.5"])  # --rho missing


def test_layout_inference():
    class A:
        frames, patches_per_frame, specials_per_frame, grid, specials_last = 2, None, 5, None, False
    lay = cli.layout_from_args(A, 2 * 1374)
    assert lay.patches_per_frame == 1369 and lay.total_tokens == 2748
    with pytest.raises(SystemExit):
        cli.layout_from_args(A, 2749)       # not divisible into 2 frames
    A.specials_per_frame = 2000
    with pytest.raises(SystemExit):
        cli.layout_from_args(A, 2748)       # inferred patches < 1
    A.specials_per_frame, A.grid = 5, "bad"
    with pytest.raises(SystemExit):
        cli.layout_from_args(A, 2748)
