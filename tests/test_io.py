"""SKYC dataset files: skycell::write_bin / read_bin
(proj/src/datagen.cpp:185-221; test_datagen.cpp:98-106, :152-160).

CPU: the header checks (bin_header) against the unmodified reference's
read_bin on the same files -- same exception type, same message.
GPU: files written by the reference load into device memory bit-exactly with
the reference's dim_min / dim_max, files written from device memory are
byte-identical to the reference's, and a skyline over a loaded file equals the
reference's compute_skyline over read_bin's Dataset."""
import os
import struct

import numpy as np
import pytest

import paper_2107_09993_b200 as sky

EXC = {1: sky.InputError, 4: sky.IoError}


def _write(path, data: bytes):
    with open(path, "wb") as f:
        f.write(data)


def _bad_files(tmp_path):
    hdr = lambda v, d, n: b"SKYC" + struct.pack("<IIQ", v, d, n)
    return {
        "bad_magic": b"NOPE",                          # test_datagen.cpp:152-160
        "short_magic": b"SK",
        "version": hdr(2, 3, 1) + b"\0" * 24,
        "dims_low": hdr(1, 1, 1) + b"\0" * 8,
        "dims_high": hdr(1, 17, 1) + b"\0" * 8 * 17,
        "truncated": hdr(1, 3, 10) + b"\0" * 8 * 29,
    }


@pytest.mark.parametrize("case", ["bad_magic", "short_magic", "version", "dims_low", "dims_high"])
def test_bin_header_errors_match_reference(tmp_path, reference, case):
    from oracle.oracle import CpuError
    path = str(tmp_path / f"{case}.bin")
    _write(path, _bad_files(tmp_path)[case])
    with pytest.raises(CpuError) as ref:
        reference.read_bin(path)
    with pytest.raises(sky.SkycellError) as got:
        sky.bin_header(path)
    assert isinstance(got.value, EXC[ref.value.code])
    assert str(got.value) == str(ref.value)


def test_bin_header_missing_file(tmp_path, reference):
    from oracle.oracle import CpuError
    path = str(tmp_path / "absent.bin")
    with pytest.raises(CpuError) as ref:
        reference.read_bin(path)
    with pytest.raises(sky.IoError) as got:
        sky.bin_header(path)
    assert ref.value.code == 4 and str(got.value) == str(ref.value)


def test_bin_header_of_reference_file(tmp_path, reference, oracle):
    v = oracle.generate(1, 5000, 3, 21)  # test_datagen.cpp:98-106
    path = str(tmp_path / "roundtrip.bin")
    reference.write_bin(path, v)
    assert sky.bin_header(path) == (5000, 3)


@pytest.mark.gpu
def test_gpu_read_bin_matches_reference(tmp_path, engine, reference, oracle):
    v = oracle.generate(1, 5000, 3, 21) * 7.0 - 2.0
    v[17, 1] = -0.0
    path = str(tmp_path / "ref.bin")
    reference.write_bin(path, v)
    x, mn, mx = engine.read_bin(path)
    rx, rmn, rmx = reference.read_bin(path)
    assert np.array_equal(x.cpu().numpy().view(np.uint64), rx.view(np.uint64))
    assert np.array_equal(mn, rmn) and np.array_equal(mx, rmx)


@pytest.mark.gpu
def test_gpu_write_bin_bytes_match_reference(tmp_path, engine, reference, oracle):
    import torch
    v = oracle.generate(2, 300_000, 5, 8)
    ref_path, dev_path, host_path = (str(tmp_path / f"{k}.bin") for k in ("ref", "dev", "host"))
    reference.write_bin(ref_path, v)
    engine.write_bin(dev_path, torch.from_numpy(v).cuda())
    engine.write_bin(host_path, v)
    want = open(ref_path, "rb").read()
    assert open(dev_path, "rb").read() == want
    assert open(host_path, "rb").read() == want


@pytest.mark.gpu
def test_gpu_read_bin_multi_chunk_and_truncated(tmp_path, engine, reference, oracle):
    """> 64 MB: several pinned staging chunks; then the same file cut short."""
    v = oracle.generate(0, 2_500_000, 4, 3)  # 80 MB
    path = str(tmp_path / "big.bin")
    reference.write_bin(path, v)
    x, mn, mx = engine.read_bin(path)
    assert np.array_equal(x.cpu().numpy(), v)
    rx, rmn, rmx = reference.read_bin(path)
    assert np.array_equal(mn, rmn) and np.array_equal(mx, rmx)
    data = open(path, "rb").read()
    cut = str(tmp_path / "cut.bin")
    _write(cut, data[:-8])
    from oracle.oracle import CpuError
    with pytest.raises(CpuError) as ref:
        reference.read_bin(cut)
    with pytest.raises(sky.InputError) as got:
        engine.read_bin(cut)
    assert str(got.value) == str(ref.value)


@pytest.mark.gpu
def test_gpu_skyline_of_loaded_file(tmp_path, engine, reference, oracle):
    v = oracle.generate(2, 20000, 4, 5) * 3.0 + 1.0
    path = str(tmp_path / "q.bin")
    reference.write_bin(path, v)
    x, mn, mx = engine.read_bin(path)
    rx, rmn, rmx = reference.read_bin(path)
    rho = sky.default_rho(len(v), 4)
    got = engine.skyline_raw(x, len(v), 4, mn, mx, rho)
    want = reference.compute_skyline(rx, rmn, rmx, rho)
    assert np.array_equal(np.asarray(got.ids), want.ids)
    assert got.points_examined == want.points_examined
