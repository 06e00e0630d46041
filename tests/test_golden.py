"""Golden fixtures (tests/golden/*.npz, written by tests/golden/make_golden.py
from the pinned oracle) and full-size properties at the BASELINE shapes.

CPU part: the oracle and the host-side generator still reproduce the frozen
numbers (generation is bit-exact by construction, datagen.cpp:13-80).
GPU part: the sm_100a path reproduces the frozen MTTKRPs (1e-12) and the
30-iteration HER / AO traces (parity.compare_traces bars); at the full C2 /
C3 sizes, where the oracle's per-call cost is seconds, size-independent
identities stand in: for a noiseless instance T = [[A]],
    MTTKRP(T, A, n) = A_n * (hadamard_{j != n} A_j^T A_j)      (exact algebra)
and MTTKRP is linear in T.
"""
import glob
import os

import numpy as np
import pytest

from parity import compare_traces, rel_fro

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = sorted(p for p in glob.glob(os.path.join(HERE, "*.npz")) if not os.path.basename(p).startswith(("config_", "refrun_")))


def _load(path):
    z = np.load(path)
    shape = [int(x) for x in z["shape"]]
    n = len(shape)
    get = lambda key: [z[f"{key}{i}"] for i in range(n)]  # noqa: E731
    return z, shape, get


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_oracle_reproduces_fixture(oracle, path):
    z, shape, get = _load(path)
    rank, seed, sigma = int(z["rank"]), int(z["seed"]), float(z["sigma"])
    t, truth = oracle.generate(shape, rank, sigma=sigma, seed=seed)
    assert np.array_equal(t, z["tensor"])
    for a, b in zip(truth, get("truth")):
        assert np.array_equal(a, b)
    init = oracle.random_init(shape, rank, oracle.stream_seed(seed, 1))
    for a, b in zip(init, get("init")):
        assert np.array_equal(a, b)
    for mode in range(len(shape)):
        assert rel_fro(oracle.mttkrp(t, get("init"), mode), z[f"mttkrp_init{mode}"]) < 1e-14
    fac, f0, recs = oracle.run("her", t, get("init"), max_outer_iters=len(z["her_f"]))
    assert abs(f0 - float(z["her_f0"])) <= 1e-14 * abs(f0)
    np.testing.assert_allclose([r["f"] for r in recs], z["her_f"], rtol=1e-10, atol=1e-14 * float(z["norm_sq"]))
    assert [bool(r["restarted"]) for r in recs] == list(z["her_restarted"])


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_host_generator_matches_fixture(P, path):
    z, shape, get = _load(path)
    spec = P.SyntheticSpec(shape=shape, rank=int(z["rank"]), noise_sigma=float(z["sigma"]), seed=int(z["seed"]))
    t, truth = P.generate(spec)
    assert np.array_equal(np.asarray(t), z["tensor"])
    init = P.random_init(shape, int(z["rank"]), P.stream_seed(int(z["seed"]), 1))
    for a, b in zip(init.factors, get("init")):
        assert np.array_equal(a, b)


# ---- GPU -----------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_gpu_mttkrp_matches_fixture(P, path):
    z, shape, get = _load(path)
    prov = P.GpuDenseProvider(z["tensor"])
    assert abs(prov.norm_sq() - float(z["norm_sq"])) <= 1e-13 * float(z["norm_sq"])
    for mode in range(len(shape)):
        assert rel_fro(prov.mttkrp(get("truth"), mode), z[f"mttkrp_truth{mode}"]) < 1e-12
        assert rel_fro(prov.mttkrp(get("init"), mode), z[f"mttkrp_init{mode}"]) < 1e-12


def _fixture_records(z, algo):
    f = z[f"{algo}_f"]
    out = []
    for k in range(len(f)):
        r = {"iter": k + 1, "f": float(f[k]), "restarted": None, "beta": None}
        if algo == "her":
            r["restarted"] = bool(z["her_restarted"][k])
            r["beta"] = float(z["her_beta"][k])
        out.append(r)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["her", "ao"])
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_gpu_traces_match_fixture(P, path, algo):
    z, shape, get = _load(path)
    init = P.KruskalModel(get("init"))
    cfg = P.AoConfig(max_outer_iters=len(z[f"{algo}_f"]))
    if algo == "her":
        model, trace = P.her_run(z["tensor"], init, cfg, P.HerParams())
    else:
        model, trace = P.ao_run(z["tensor"], init, cfg)
    stats = compare_traces(trace, float(z[f"{algo}_f0"]), _fixture_records(z, algo), float(z["norm_sq"]),
                           check_restarts=(algo == "her"))
    assert stats["checked"] == len(z[f"{algo}_f"])
    assert model.is_nonnegative()


@pytest.mark.gpu
@pytest.mark.parametrize("shape,rank", [([300, 300, 300], 20), ([100, 100, 100, 100], 16)],
                         ids=["C2", "C3"])
def test_full_size_noiseless_identity_and_linearity(P, shape, rank):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.0, seed=102)
    t, truth = P.generate(spec)
    a = [np.asarray(x) for x in truth.factors]
    prov = P.GpuDenseProvider(t)
    prov3 = P.GpuDenseProvider(np.asarray(t) * 3.0)  # exact scaling (power of two times 1.5: one rounding)
    grams = [x.T @ x for x in a]
    for mode in range(len(shape)):
        h = np.ones((rank, rank))
        for j, g in enumerate(grams):
            if j != mode:
                h *= g
        want = a[mode] @ h
        got = prov.mttkrp(a, mode)
        assert rel_fro(got, want) < 1e-12, mode
        assert rel_fro(prov3.mttkrp(a, mode), 3.0 * got) < 1e-14, mode
    prov.close()
    prov3.close()
