"""Host-side checks of the product library that need no GPU: the C ABI loads
and exports every symbol include/ntf_b200.h declares, host datagen is
bit-exact with the oracle (and hence the reference generator), validation
mirrors the reference's exceptions, trace CSV round-trips, and there is no
CPU fallback (a context cannot be created without a device)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(P):
    from paper_2001_04321_b200 import _lib
    header = open(os.path.join(ROOT, "include", "ntf_b200.h")).read()
    declared = sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w ]*\*?\s*\**)\b(ntf_\w+)\s*\(", header, re.M)))
    assert len(declared) >= 30
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [name for name in declared if not hasattr(lib, name)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)


@pytest.mark.parametrize("shape,rank,sigma,ill,seed", [([6, 5, 4], 3, 0.1, False, 42), ([30, 20, 10], 5, 0.01, True, 7),
                                                      ([5, 4, 3, 6], 2, 0.01, False, 404), ([12, 9], 2, 0.0, False, 1),
                                                      ([50, 50, 50], 10, 0.01, False, 101), ([7], 2, 0.5, False, 3)])
def test_generate_bit_exact_with_oracle(P, oracle, shape, rank, sigma, ill, seed):
    t, truth = P.generate(P.SyntheticSpec(shape, rank, sigma, ill, seed))
    t2, truth2 = oracle.generate(shape, rank, sigma, ill, seed)
    assert np.array_equal(t, t2)
    for a, b in zip(truth, truth2):
        assert np.array_equal(a, b)
    t32, _ = P.generate(P.SyntheticSpec(shape, rank, sigma, ill, seed), dtype=np.float32)
    assert t32.dtype == np.float32 and np.array_equal(t32, t2.astype(np.float32))


def test_collinear_rule_matches_oracle(P, oracle):
    spec = P.SyntheticSpec([9, 8, 7], 4, 0.01, False, 104, collinear=True)
    t, truth = P.generate(spec)
    t2, truth2 = oracle.generate([9, 8, 7], 4, 0.01, False, 104, collinear=True)
    assert np.array_equal(t, t2)
    # columns share one vector: pairwise column differences are 0.5 (U_j - U_k)
    _, plain = oracle.generate([9, 8, 7], 4, 0.0, False, 104)
    for a, u in zip(truth, plain):
        assert np.allclose(a[:, 0] - a[:, 1], 0.5 * (u[:, 0] - u[:, 1]), atol=1e-15)


def test_random_init_and_stream_seed(P, oracle):
    for seed in (0, 17, 2**40 + 3):
        a = P.random_init([4, 6, 3], 3, seed)
        b = oracle.random_init([4, 6, 3], 3, seed)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        assert P.stream_seed(seed, 3) == oracle.stream_seed(seed, 3)


def test_factor_error_matches_oracle(P, oracle):
    gen = np.random.default_rng(4)
    truth = [gen.random((d, 4)) for d in (5, 6, 7)]
    est = [a + 0.05 * gen.random(a.shape) for a in truth]
    assert P.factor_error(est, truth) == pytest.approx(oracle.factor_error(est, truth), rel=1e-12)
    perm = [2, 0, 3, 1]
    assert P.factor_error([a[:, perm] * 3.0 for a in truth], truth) < 1e-12


def test_validation_mirrors_reference(P):
    with pytest.raises(ValueError):
        P.HerParams(beta0=0.0).validate()
    with pytest.raises(ValueError):
        P.HerParams(gamma_bar=1.0).validate()
    with pytest.raises(ValueError):
        P.HerParams(eta=1.01).validate()
    P.HerParams().validate()
    with pytest.raises(ValueError):
        P.AoConfig().validate()
    with pytest.raises(ValueError):
        P.AoConfig(max_outer_iters=5, record_factor_error=True).validate()
    P.AoConfig(max_outer_iters=5).validate()
    with pytest.raises(ValueError):
        P.generate(P.SyntheticSpec([3, 3], 0))
    with pytest.raises(ValueError):
        P.generate(P.SyntheticSpec([3, 3], 1, ill_conditioned=True))
    with pytest.raises(ValueError):
        P.generate(P.SyntheticSpec([3, 3], 1, noise_sigma=-0.5))
    assert P.nnls_solver_from_name("as") == P.NnlsSolver.active_set
    with pytest.raises(ValueError):
        P.nnls_solver_from_name("lbfgs")


def test_update_betas_host_mirror(P, oracle):
    gen = np.random.default_rng(2)
    s = P.HerState(beta=0.5, beta_bar=1.0)
    b, bb = 0.5, 1.0
    for _ in range(1000):
        rs = bool(gen.integers(0, 2))
        P.update_betas(s, rs, P.HerParams())
        b, bb = oracle.update_betas(b, bb, rs)
        assert (s.beta, s.beta_bar) == (b, bb)


def test_slab_range_partitions_mode1(P):
    for dim0 in (1, 7, 100, 300, 2000):
        for world in (1, 2, 3, 4, 8):
            if world > dim0:
                continue
            spans = [P.slab_range(dim0, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == dim0
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        P.slab_range(10, 2, 2)


def test_trace_csv_round_trip(P, tmp_path):
    tr = P.RunTrace(1.5, [P.TraceRecord(1, 0.1, 1.25, None, False, 0.5),
                          P.TraceRecord(2, 0.2, 1.0 / 3.0, 0.25, True, 0.525)])
    path = tmp_path / "t.csv"
    tr.write_csv(str(path))
    assert open(path).readline().strip() == "iter,time_s,f,e,restarted,beta"
    back = P.RunTrace.read_csv(str(path))
    assert [(r.iter, r.f, r.e, r.restarted, r.beta) for r in back.records] == \
        [(r.iter, r.f, r.e, r.restarted, r.beta) for r in tr.records]
    back.validate()
    assert back.restart_count() == 1 and back.final_f() == 1.0 / 3.0


def test_cpp_header_api_compiles_and_runs(P, tmp_path, oracle):
    """include/ntf_b200.hpp (the reference-shaped C++ API) against the .so."""
    import subprocess
    from paper_2001_04321_b200 import _lib
    exe = tmp_path / "api_smoke"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp"), "-L", libdir, "-l:libntf_b200.so",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "cpu", str(tmp_path / "smoke.ntfk")], capture_output=True, text=True,
                         check=True).stdout
    t, _ = oracle.generate([6, 5, 4], 3, 0.1, False, 42)
    init = oracle.random_init([6, 5, 4], 3, oracle.stream_seed(42, 1))
    seq = 0.0  # the C++ side sums in flat order
    for x in t.ravel():
        seq += float(x)
    assert f"sum={seq:.17g} init00={init[0][0, 0]:.17g}" in out, out
    assert "ntfk roundtrip ok" in out
    back = P.TuckerFormat.load(str(tmp_path / "smoke.ntfk"))  # the C++ writer's container, read by Python
    assert np.array_equal(back.core, t) and all(np.array_equal(b, np.eye(d)) for b, d in zip(back.bases, (6, 5, 4)))


@pytest.mark.gpu
def test_cpp_header_drivers_on_gpu(P, tmp_path):
    """The GPU branch of tests/cpp/api_smoke.cpp: ntfb::her_run through the
    C++ header on a GpuDenseProvider gives the same bits as the Python API
    on the same inputs; on a TuckerProvider (identity bases) the same trace
    to 1e-8."""
    import subprocess
    from paper_2001_04321_b200 import _lib
    exe = tmp_path / "api_smoke"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp"), "-L", libdir, "-l:libntf_b200.so",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "gpu", str(tmp_path / "s.ntfk")], capture_output=True, text=True,
                         check=True).stdout
    spec = P.SyntheticSpec(shape=[6, 5, 4], rank=3, noise_sigma=0.1, seed=42)
    t, _ = P.generate(spec)
    init = P.random_init([6, 5, 4], 3, P.stream_seed(42, 1))
    _, tr = P.her_run(t, init, P.AoConfig(max_outer_iters=10), P.HerParams())
    assert f"f0={tr.f0:.17g} f10={tr.final_f():.17g} restarts={tr.restart_count()}" in out, out
    line = [ln for ln in out.splitlines() if ln.startswith("tucker ")][0]
    f10 = float(line.split("f10=")[1].split()[0])
    assert abs(f10 - tr.final_f()) <= 1e-8 * abs(tr.final_f())


def test_no_cpu_fallback_without_device(P):
    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.CudaError):
        P.Context(0)
    with pytest.raises(P.CudaError):
        P.GpuDenseProvider(np.ones((2, 2, 2)))


@pytest.mark.parametrize("shape,rank,sigma,dtype", [([9, 7, 5], 3, 0.05, np.float64), ([13, 4, 6, 3], 2, 0.1, np.float32),
                                                    ([11, 6], 4, 0.0, np.float64), ([7], 2, 0.2, np.float64)])
def test_generate_slab_matches_whole_instance(P, shape, rank, sigma, dtype):
    """ntf_generate_slab: every mode-1 slab (the part a sharded rank holds)
    is bit-identical to that slice of the whole instance, noise included
    (the parallel generator enters the serial noise stream at the slab's
    first entry)."""
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, seed=77)
    whole, truth = P.generate(spec, dtype=dtype)
    for world in (1, 2, 3, 4):
        for r in range(world):
            b, e = P.slab_range(shape[0], r, world)
            part, truth2 = P.generate(spec, dtype=dtype, slab=(b, e))
            assert part.shape == tuple([e - b] + shape[1:])
            assert np.array_equal(part, whole[b:e])
            assert all(np.array_equal(x, y) for x, y in zip(truth2, truth))
    with pytest.raises(P.InvalidArgument):
        P.generate(spec, dtype=dtype, slab=(0, shape[0] + 1))


def test_generate_large_chunked_noise_matches_oracle(P, oracle):
    """More entries than one generator chunk (2^20), so several OpenMP
    workers start from producer snapshots of the noise stream: still
    bit-exact with the serial oracle."""
    shape, rank = [40, 160, 200], 3
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.3, seed=5)
    t, _ = P.generate(spec)
    ref, _ = oracle.generate(shape, rank, 0.3, False, 5)
    assert np.array_equal(t, ref)
