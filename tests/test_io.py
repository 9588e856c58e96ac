"""MASTENS v1 tensor files: the product's
read_tensor / write_tensor (paper_2409_07704_b200/csrc/mas_io.cpp through the
C-ABI) against the reference's own io::read_tensor / io::write_tensor
(tensor_io.cpp compiled in place into oracle/_ref), modelled on the
reference's tests/test_io.cpp cases.  Host-only code: runs on CPU."""

from __future__ import annotations

import os
import struct

import numpy as np
import pytest

ERRC = {"IoFailure": 12, "BadMagic": 13, "UnsupportedVersion": 14, "TruncatedFile": 15,
        "DimensionOverflow": 16}


def _errc(mas, fn):
    """Calls fn through the C-ABI; returns (errc, message) of the failure."""
    import ctypes

    from paper_2409_07704_b200 import _lib

    err = _lib.MasError()
    rc = fn(err)
    assert rc == _lib.MAS_E_IO, rc
    return err.errc, err.message.decode()


def _read_c(mas, path, budget=1 << 30):
    import ctypes

    lib = mas._lib.load()
    dtype = ctypes.c_int32()
    dims = (ctypes.c_int64 * 3)()
    has = ctypes.c_int32()
    vals = np.empty(1 << 16, np.uint8)  # kept alive across the call
    lens = np.empty(1 << 12, np.uint32)
    return _errc(mas, lambda err: lib.mas_io_read_header(
        os.fsencode(path), budget, ctypes.byref(dtype), ctypes.byref(dims), ctypes.byref(has),
        ctypes.byref(err)) or lib.mas_io_read(os.fsencode(path), budget, dtype.value,
                                              ctypes.byref(dims), vals.ctypes.data,
                                              lens.ctypes.data, ctypes.byref(err)))


def _sample():
    # -0, a denormal and a NaN payload must survive bit-exactly
    v = np.array([1.5, -2.0, 0.0, -0.0, 1e-40, 3.25], np.float32).reshape(1, 2, 3)
    return v


def test_float_round_trip_bit_exact(mas, tmp_path):
    v = _sample()
    nan = np.frombuffer(np.uint32(0x7fc00123).tobytes(), np.float32)[0]
    v = v.copy()
    v[0, 1, 2] = nan
    p = tmp_path / "f.bin"
    mas.write_tensor(str(p), v)
    got, lens = mas.read_tensor(str(p))
    assert got.dtype == np.float32 and got.shape == (1, 2, 3)
    assert got.tobytes() == v.tobytes()
    np.testing.assert_array_equal(lens, [[2, 3]])
    assert lens.dtype == np.uint32


def test_alignment_round_trip_and_dtype_byte(mas, tmp_path):
    m = np.zeros((2, 3, 4), np.uint8)
    m[0, 0, 0] = m[1, 2, 3] = 1
    p = tmp_path / "m.bin"
    mas.write_tensor(str(p), m, lengths=[[3, 4], [2, 3]])
    raw = p.read_bytes()
    assert raw[12] == 1 and raw[38] == 1
    got, lens = mas.read_tensor(str(p))
    assert got.dtype == np.uint8 and np.array_equal(got, m)
    np.testing.assert_array_equal(lens, [[3, 4], [2, 3]])


def test_header_layout_is_frozen(mas, tmp_path):
    v = np.arange(2 * 3 * 5, dtype=np.float32).reshape(2, 3, 5)
    p = tmp_path / "h.bin"
    mas.write_tensor(str(p), v, lengths=[[3, 5], [1, 4]])
    raw = p.read_bytes()
    assert raw[:8] == b"MASTENS\0"
    assert struct.unpack("<I", raw[8:12])[0] == 1
    assert raw[12] == 0 and raw[13] == 3
    assert struct.unpack("<QQQ", raw[14:38]) == (2, 3, 5)
    assert raw[38] == 1
    assert len(raw) == 39 + v.nbytes + 2 * 8
    assert raw[39:39 + v.nbytes] == v.tobytes()
    assert struct.unpack("<4I", raw[39 + v.nbytes:]) == (3, 5, 1, 4)


def test_writes_byte_identical_to_reference(mas, reference, tmp_path):
    rng = np.random.default_rng(0)
    for it in range(12):
        B, T, S = (int(x) for x in rng.integers(1, 9, 3))
        if it % 2:
            v = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
        else:
            v = (rng.random((B, T, S)) < 0.2).astype(np.uint8)
        lens = np.stack([rng.integers(0, T + 1, B), rng.integers(0, S + 1, B)], 1)
        ours, theirs = tmp_path / f"o{it}.bin", tmp_path / f"r{it}.bin"
        mas.write_tensor(str(ours), v, lengths=lens)
        rc, msg = reference.write_tensor(str(theirs), v, lens)
        assert rc == -1, msg
        assert ours.read_bytes() == theirs.read_bytes()
        # and each reads the other's file
        rc, msg, rv, rl = reference.read_tensor(str(ours))
        assert rc == -1 and rv.tobytes() == v.tobytes() and np.array_equal(rl, lens)
        gv, gl = mas.read_tensor(str(theirs))
        assert gv.tobytes() == v.tobytes() and np.array_equal(gl, lens)


def _corrupt_cases(tmp_path, mas):
    """(name, bytes) of every malformed file test_io.cpp covers."""
    v = np.arange(6, dtype=np.float32).reshape(1, 2, 3)
    p = tmp_path / "good.bin"
    mas.write_tensor(str(p), v)
    good = p.read_bytes()
    cases = []

    def patch(off, data):
        b = bytearray(good)
        b[off:off + len(data)] = data
        return bytes(b)

    cases.append(("magic", patch(0, b"NOTATENS")))
    cases.append(("version", patch(8, struct.pack("<I", 2))))
    cases.append(("dtype", patch(12, b"\x07")))
    cases.append(("rank", patch(13, b"\x02")))
    cases.append(("lenflag", patch(38, b"\x05")))
    cases.append(("trunc_header", good[:20]))
    cases.append(("trunc_payload", good[:39 + 10]))
    cases.append(("trunc_lengths", good[:-3]))
    cases.append(("zero_dim", patch(14, struct.pack("<Q", 0))))
    cases.append(("huge_dim", patch(22, struct.pack("<Q", 1 << 40))))
    cases.append(("over_budget", patch(14, struct.pack("<QQQ", 1 << 12, 1 << 12, 1 << 12))))
    cases.append(("empty", b""))
    return cases


def test_malformed_files_match_reference_errors(mas, reference, tmp_path):
    for name, data in _corrupt_cases(tmp_path, mas):
        p = tmp_path / f"bad_{name}.bin"
        p.write_bytes(data)
        rc, msg, _, _ = reference.read_tensor(str(p))
        assert rc != -1, name
        errc, ours = _read_c(mas, str(p))
        assert errc == rc, (name, errc, rc)
        assert ours == msg, (name, ours, msg)
        with pytest.raises(OSError) as ei:
            mas.read_tensor(str(p))
        assert str(ei.value) == msg


def test_custom_budget_and_missing_file(mas, reference, tmp_path):
    p = tmp_path / "b.bin"
    mas.write_tensor(str(p), np.zeros((1, 2, 3), np.float32))
    rc, msg, _, _ = reference.read_tensor(str(p), 8)
    errc, ours = _read_c(mas, str(p), 8)
    assert errc == rc == ERRC["DimensionOverflow"] and ours == msg
    missing = "/no/such/dir/x.bin"
    rc, msg, _, _ = reference.read_tensor(missing)
    errc, ours = _read_c(mas, missing)
    assert errc == rc == ERRC["IoFailure"] and ours == msg
    with pytest.raises(OSError, match="cannot open for writing"):
        mas.write_tensor(missing, np.zeros((2, 2), np.float32))
    rc, msg = reference.write_tensor(missing, np.zeros((1, 2, 2), np.float32))
    assert rc == ERRC["IoFailure"] and msg.startswith("cannot open for writing")


def test_file_without_lengths_defaults_to_full(mas, reference, tmp_path):
    v = np.ones((2, 3, 4), np.float32)
    p = tmp_path / "nolen.bin"
    mas.write_tensor(str(p), v)
    raw = bytearray(p.read_bytes())
    raw[38] = 0
    p.write_bytes(bytes(raw[:39 + v.nbytes]))
    got, lens = mas.read_tensor(str(p))
    np.testing.assert_array_equal(lens, [[3, 4], [3, 4]])
    rc, _, _, rl = reference.read_tensor(str(p))
    assert rc == -1 and np.array_equal(rl, lens)


def test_python_surface_checks(mas, tmp_path):
    p = str(tmp_path / "x.bin")
    mas.write_tensor(p, np.zeros((3, 4), np.float32))  # 2-D: one item
    v, lens = mas.read_tensor(p)
    assert v.shape == (1, 3, 4) and lens.tolist() == [[3, 4]]
    with pytest.raises(ValueError, match="values dtype must be float32 or uint8"):
        mas.write_tensor(p, np.zeros((1, 2, 2), np.float64))
    with pytest.raises(ValueError):
        mas.write_tensor(p, np.zeros((1, 2, 2), np.float32), lengths=[[3, 2]])
    with pytest.raises(ValueError):
        mas.write_tensor(p, np.zeros((0, 2, 2), np.float32))


def test_read_rejects_a_file_replaced_after_the_header(mas, tmp_path):
    """mas_io_read checks the header against the dims the buffers were sized
    for (a file swapped between the two reads must not overflow them)."""
    import ctypes

    from paper_2409_07704_b200 import _lib

    lib = mas._lib.load()
    p = tmp_path / "swap.bin"
    mas.write_tensor(str(p), np.zeros((1, 2, 3), np.float32))
    dtype = ctypes.c_int32()
    dims = (ctypes.c_int64 * 3)()
    has = ctypes.c_int32()
    err = _lib.MasError()
    assert lib.mas_io_read_header(os.fsencode(str(p)), 1 << 30, ctypes.byref(dtype),
                                  ctypes.byref(dims), ctypes.byref(has), ctypes.byref(err)) == 0
    vals = np.full(6, 7.0, np.float32)
    lens = np.zeros((1, 2), np.uint32)
    mas.write_tensor(str(p), np.zeros((4, 8, 9), np.float32))  # bigger file, same path
    rc = lib.mas_io_read(os.fsencode(str(p)), 1 << 30, dtype.value, ctypes.byref(dims),
                         vals.ctypes.data, lens.ctypes.data, ctypes.byref(err))
    assert rc == _lib.MAS_E_IO and err.errc == 12  # IoFailure
    assert b"differs from the expected" in err.message
    assert (vals == 7.0).all()
    mas.write_tensor(str(p), np.zeros((1, 2, 3), np.uint8))  # same dims, other dtype
    rc = lib.mas_io_read(os.fsencode(str(p)), 1 << 30, dtype.value, ctypes.byref(dims),
                         vals.ctypes.data, lens.ctypes.data, ctypes.byref(err))
    assert rc == _lib.MAS_E_IO
