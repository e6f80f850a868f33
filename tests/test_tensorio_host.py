"""The .bsat tensor file format (tensorio.py), the reference's own cases
(/root/reference/pkg/tests/test_tensorio.py, TestTensorFile) run against this
package. Host-only code: no GPU."""

import struct

import numpy as np
import pytest

from paper_2509_07120_b200.tensorio import (
    BadMagicError,
    TensorFileError,
    TruncatedPayloadError,
    UnsupportedDTypeError,
    read_tensor,
    write_tensor,
)


def test_round_trips_bit_identical(tmp_path):
    rng = np.random.default_rng(5)
    for shape in ((2, 3), (3, 5, 7)):
        t = rng.standard_normal(shape).astype(np.float32)
        path = tmp_path / "t.bsat"
        write_tensor(path, t)
        back = read_tensor(path)
        assert back.shape == shape and back.tobytes() == t.tobytes()


def test_header_bytes(tmp_path):
    path = tmp_path / "t.bsat"
    write_tensor(path, np.zeros((10, 64), dtype=np.float32))
    raw = path.read_bytes()
    assert raw[:4] == b"BSAT"
    assert struct.unpack_from("<I", raw, 4) == (1,)
    assert raw[8] == 0
    assert struct.unpack_from("<I", raw, 9) == (2,)
    assert struct.unpack_from("<2Q", raw, 13) == (10, 64)
    assert len(raw) == 13 + 16 + 10 * 64 * 4


def _corrupt(tmp_path, edit):
    path = tmp_path / "t.bsat"
    write_tensor(path, np.arange(12, dtype=np.float32).reshape(3, 4))
    path.write_bytes(edit(bytearray(path.read_bytes())))
    return path


@pytest.mark.parametrize("edit,err", [
    (lambda r: bytes(r[:-4]), TruncatedPayloadError),
    (lambda r: b"NOPE" + bytes(r[4:]), BadMagicError),
    (lambda r: bytes(r[:8]) + b"\x07" + bytes(r[9:]), UnsupportedDTypeError),
    (lambda r: bytes(r) + b"\x00\x00", TensorFileError),
])
def test_corrupt_files_rejected(tmp_path, edit, err):
    with pytest.raises(err):
        read_tensor(_corrupt(tmp_path, edit))


def test_writer_rejects_nan(tmp_path):
    with pytest.raises(ValueError, match="non-finite"):
        write_tensor(tmp_path / "t.bsat", np.array([[np.nan]], dtype=np.float32))
