"""NTFT container I/O (the reference's DenseTensor::save / load,
tensor.cpp:56-96; README.md "File formats"): byte layout pinned against the
format the reference documents, round trips, slab reads, FP32 rounding and
the reference's error behaviour. The GPU leg uploads straight from the file."""
import struct

import numpy as np
import pytest


def reference_bytes(t):
    """The container as README.md "File formats" specifies it: magic NTFT,
    u32 version 1, u32 order, u64 dims, FP64 payload, little-endian, last
    index fastest."""
    head = b"NTFT" + struct.pack("<II", 1, t.ndim) + struct.pack("<" + "Q" * t.ndim, *t.shape)
    return head + np.ascontiguousarray(t, dtype="<f8").tobytes()


def test_write_matches_reference_layout(P, tmp_path):
    t = np.random.default_rng(3).random((4, 3, 5))
    p = tmp_path / "t.ntft"
    P.save_tensor(str(p), t)
    assert p.read_bytes() == reference_bytes(t)
    # FP32 data is stored exactly upcast
    t32 = t.astype(np.float32)
    P.save_tensor(str(p), t32)
    assert p.read_bytes() == reference_bytes(t32.astype(np.float64))


@pytest.mark.parametrize("shape", [[7], [6, 5], [5, 4, 3], [4, 3, 2, 5]])
def test_round_trip_and_slabs(P, tmp_path, shape):
    t = np.random.default_rng(len(shape)).random(shape)
    p = str(tmp_path / "t.ntft")
    (tmp_path / "t.ntft").write_bytes(reference_bytes(t))  # a file "the reference wrote"
    assert P.ntft_info(p) == shape
    assert np.array_equal(P.load_tensor(p), t)
    assert np.array_equal(P.load_tensor(p, dtype=np.float32), t.astype(np.float32))
    for world in (1, 2, 3):
        for r in range(world):
            b, e = P.slab_range(shape[0], r, world)
            assert np.array_equal(P.load_tensor(p, slab=(b, e)), t[b:e])


def test_reference_error_behaviour(P, tmp_path):
    t = np.ones((2, 3))
    good = reference_bytes(t)
    cases = {
        "missing": None,
        "magic": b"NTFX" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "order": good[:8] + struct.pack("<I", 0) + good[12:],
        "truncated": good[:-8],
    }
    want = {"missing": "cannot open", "magic": "not a tensor container", "version": "unsupported version",
            "order": "bad order", "truncated": "truncated payload"}
    for name, data in cases.items():
        p = tmp_path / f"{name}.ntft"
        if data is not None:
            p.write_bytes(data)
        with pytest.raises(RuntimeError, match=want[name]):
            P.load_tensor(str(p))
    with pytest.raises(P.InvalidArgument):
        p = tmp_path / "ok.ntft"
        p.write_bytes(good)
        P.load_tensor(str(p), slab=(1, 3))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gpu_upload_from_file_equals_array(P, tmp_path, dtype):
    spec = P.SyntheticSpec(shape=[40, 36, 33], rank=4, noise_sigma=0.01, seed=9)
    t, truth = P.generate(spec)
    p = str(tmp_path / "c.ntft")
    P.save_tensor(p, t)
    a = P.GpuDenseProvider(np.asarray(t, dtype=dtype))
    b = P.GpuDenseProvider.from_ntft(p, dtype=dtype)
    assert b.shape() == [40, 36, 33] and b.norm_sq() == a.norm_sq()
    for mode in range(3):
        assert np.array_equal(b.mttkrp(truth, mode), a.mttkrp(truth, mode))
    a.close()
    b.close()
