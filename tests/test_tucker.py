"""TuckerProvider (include/ntf/tucker.hpp:60-73, src/tucker.cpp:62-77) on the
GPU and the TuckerFormat container, following the reference's
tests/test_tucker.cpp and acceptance.cpp:472-507 (criterion_tucker_parity).

CPU: the host utilities (hosvd_compress / expand / ttm, NTFK save/load and
its errors) and the oracle's compressed MTTKRP pinned against the dense
MTTKRP of the expansion (the reference's own pin, test_tucker.cpp:71-99).
GPU: the compressed MTTKRP against that oracle (1e-12), the objective
identities, and the drivers on dense vs lossless-compressed input.
"""
import os

import numpy as np
import pytest

from parity import rel_fro


def _rand(shape, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape)


# ---- CPU ----------------------------------------------------------------------

def test_full_rank_compression_is_lossless(P):
    """test_tucker.cpp:18-30."""
    t = _rand((5, 4, 3), 1)
    fmt = P.hosvd_compress(t, list(t.shape))
    fmt.validate()
    back = P.expand(fmt)
    assert np.max(np.abs(back - t)) <= 1e-10 * np.sqrt((t ** 2).sum())
    assert abs((fmt.core ** 2).sum() - (t ** 2).sum()) <= 1e-10 * (t ** 2).sum()


def test_rank_one_tensor_compresses_to_a_scalar_core(P, oracle):
    """test_tucker.cpp:32-42."""
    g = np.random.default_rng(2)
    m = [g.uniform(0.1, 1.0, (d, 1)) for d in (4, 3, 5)]
    t = oracle.reconstruct(m)
    fmt = P.hosvd_compress(t, [1, 1, 1])
    assert fmt.core.size == 1
    assert abs(abs(fmt.core.ravel()[0]) - np.sqrt((t ** 2).sum())) <= 1e-10 * np.sqrt((t ** 2).sum())
    assert np.allclose(P.expand(fmt), t, rtol=1e-10, atol=0)


def test_rank_validation(P):
    """test_tucker.cpp:63-69."""
    t = _rand((4, 3, 2), 4)
    for ranks in ([5, 3, 2], [4, 0, 2], [4, 3]):
        with pytest.raises(P.InvalidArgument):
            P.hosvd_compress(t, ranks)
    fmt = P.hosvd_compress(t, [2, 2, 2])
    fmt.bases[1] = fmt.bases[1] * 2.0
    with pytest.raises(P.InvalidArgument, match="orthonormal"):
        fmt.validate()


def test_ntfk_round_trip_and_errors(P, tmp_path):
    """TuckerFormat::save / load (tucker.cpp:106-165): bit-exact round trip,
    the reference's error texts."""
    fmt = P.hosvd_compress(_rand((6, 5, 4), 5), [3, 2, 4])
    path = str(tmp_path / "f.ntfk")
    fmt.save(path)
    back = P.TuckerFormat.load(path)
    assert np.array_equal(back.core, fmt.core)
    assert all(np.array_equal(a, b) for a, b in zip(back.bases, fmt.bases))
    raw = open(path, "rb").read()
    assert raw[:4] == b"NTFK" and len(raw) == 4 + 4 + 4 + 6 * 8 + 8 * (24 + 18 + 10 + 16)
    bad = str(tmp_path / "bad.ntfk")
    open(bad, "wb").write(b"NTFT" + raw[4:])
    with pytest.raises(RuntimeError, match="not a tucker container"):
        P.TuckerFormat.load(bad)
    open(bad, "wb").write(raw[:-8])
    with pytest.raises(RuntimeError, match="truncated payload"):
        P.TuckerFormat.load(bad)
    with pytest.raises(RuntimeError, match="cannot open"):
        P.TuckerFormat.load(str(tmp_path / "missing.ntfk"))


@pytest.mark.parametrize("ranks", [[6, 4, 5], [3, 2, 3]], ids=["lossless", "lossy"])
def test_oracle_compressed_mttkrp_equals_dense_of_expansion(P, oracle, ranks):
    """The oracle restatement of tucker.cpp:62-77 against the dense MTTKRP of
    the expanded format (the reference's pin: test_tucker.cpp:71-99, 1e-10)."""
    t = _rand((6, 4, 5), 5)
    fmt = P.hosvd_compress(t, ranks)
    dense = P.expand(fmt)
    g = np.random.default_rng(6)
    for _ in range(5):
        m = [g.uniform(-1, 1, (d, 3)) for d in (6, 4, 5)]
        for mode in range(3):
            assert rel_fro(oracle.compressed_mttkrp(fmt.core, fmt.bases, m, mode), oracle.mttkrp(dense, m, mode)) < 1e-10


# ---- GPU ----------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("shape,ranks,rank", [((6, 4, 5), [6, 4, 5], 3), ((6, 4, 5), [3, 2, 3], 2),
                                              ((40, 36, 30), [12, 10, 8], 16), ((9, 8, 7, 6), [4, 3, 3, 2], 5)],
                         ids=["lossless", "lossy", "medium", "4way"])
def test_gpu_compressed_mttkrp(P, oracle, shape, ranks, rank):
    t = _rand(shape, 7)
    fmt = P.hosvd_compress(t, ranks)
    prov = P.TuckerProvider(fmt)
    assert prov.shape() == list(shape)
    assert abs(prov.norm_sq() - (fmt.core ** 2).sum()) <= 1e-13 * (fmt.core ** 2).sum()
    dense = P.expand(fmt)
    g = np.random.default_rng(8)
    for _ in range(3):
        m = [g.uniform(0, 1, (d, rank)) for d in shape]
        allm = prov.mttkrp_all(m)
        for mode in range(len(shape)):
            want = oracle.compressed_mttkrp(fmt.core, fmt.bases, m, mode)
            got = prov.mttkrp(m, mode)
            assert rel_fro(got, want) <= 1e-12
            assert rel_fro(allm[mode], want) <= 1e-12
            assert rel_fro(got, oracle.mttkrp(dense, m, mode)) <= 1e-10
    assert "tucker" in prov.mttkrp_plan(rank, 0)
    prov.close()


@pytest.mark.gpu
def test_gpu_objective_identities(P, oracle):
    """test_tucker.cpp:115-138: a zero model leaves half the core norm; an
    exact model of the expansion has zero objective."""
    t = _rand((5, 4, 3), 9)
    fmt = P.hosvd_compress(t, [3, 3, 2])
    prov = P.TuckerProvider(fmt)
    zero = [np.zeros((d, 2)) for d in (5, 4, 3)]
    assert abs(prov.objective(zero) - 0.5 * (fmt.core ** 2).sum()) <= 1e-14 * (fmt.core ** 2).sum()
    prov.close()
    g = np.random.default_rng(7)
    m = [g.uniform(0.1, 1.0, (4, 2)) for _ in range(3)]
    t = oracle.reconstruct(m)
    prov = P.TuckerProvider(P.hosvd_compress(t, list(t.shape)))
    assert abs(prov.objective(m)) <= 1e-10 * (t ** 2).sum()
    prov.close()


@pytest.mark.gpu
def test_gpu_invalid_bases_rejected(P):
    fmt = P.hosvd_compress(_rand((6, 5, 4), 10), [3, 2, 2])
    fmt.bases[0] = fmt.bases[0] * 1.5
    with pytest.raises(P.InvalidArgument, match="orthonormal"):
        P.TuckerProvider(fmt)


@pytest.mark.gpu
@pytest.mark.parametrize("spec_shape,rank,seed,init_seed", [([8, 8, 8], 3, 11, 13), ([20, 20, 20], 4, 1015, 1016)],
                         ids=["test_tucker", "acceptance"])
def test_drivers_identical_on_dense_and_compressed(P, spec_shape, rank, seed, init_seed, tmp_path):
    """test_tucker.cpp:140-157 and acceptance.cpp:472-507: her_run on the
    dense tensor and on its lossless compression, 30 iterations, f_k within
    1e-8 relative. Also through the NTFK container (ntf_tensor_upload_ntfk)."""
    spec = P.SyntheticSpec(shape=spec_shape, rank=rank, noise_sigma=0.01, seed=seed)
    t, _ = P.generate(spec)
    init = P.random_init(spec_shape, rank, init_seed)
    fmt = P.hosvd_compress(t, spec_shape)
    cfg = P.AoConfig(max_outer_iters=30)
    _, dt = P.her_run(P.GpuDenseProvider(t), init, cfg, P.HerParams())
    prov = P.TuckerProvider(fmt)
    _, ct = P.her_run(prov, init, cfg, P.HerParams())
    assert len(dt.records) == len(ct.records) == 30
    worst = max(abs(a.f - b.f) / abs(a.f) for a, b in zip(dt.records, ct.records))
    assert worst <= 1e-8, worst
    path = str(tmp_path / "c.ntfk")
    fmt.save(path)
    pk = P.TuckerProvider.from_ntfk(path)
    _, kt = P.ao_run(pk, init, cfg)
    _, at = P.ao_run(prov, init, cfg)
    assert [r.f for r in kt.records] == [r.f for r in at.records]
    prov.close()
    pk.close()
