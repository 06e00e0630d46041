"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Mirrors the reference's hot-path pins: MTTKRP vs unfold*KR
on random shapes (test_kernels.cpp:138-153), rank-one identity (:121-136),
objective vs residual (:222-248), AHALS (test_nnls.cpp:56-112), HER/AO traces
(test_her.cpp, test_ao.cpp), plus whole-trace parity with the oracle.
"""
import numpy as np
import pytest

from parity import compare_traces, rel_fro

pytestmark = pytest.mark.gpu


def _shape_gen(gen, max_order=4):
    order = 2 + int(gen.integers(0, max_order - 1))
    return [int(gen.integers(1, 7)) for _ in range(order)]


# ---- MTTKRP -----------------------------------------------------------------------

def test_mttkrp_rank_one_identity_and_zero(P, oracle):
    gen = np.random.default_rng(6)
    m = [gen.random((d, 1)) for d in (3, 4, 2)]
    t = oracle.reconstruct(m)
    prov = P.GpuDenseProvider(t)
    want = m[0] * (np.sum(m[1] ** 2) * np.sum(m[2] ** 2))
    assert rel_fro(prov.mttkrp(m, 0), want) < 1e-14
    z = P.GpuDenseProvider(np.zeros((3, 4, 2)))
    assert np.abs(z.mttkrp(m, 1)).max() == 0.0
    with pytest.raises(ValueError):
        prov.mttkrp([gen.random((d, 1)) for d in (3, 4, 3)], 0)


def test_mttkrp_random_shapes_vs_enumeration(P, oracle):
    gen = np.random.default_rng(7)
    for _ in range(40):
        shape = _shape_gen(gen)
        r = 1 + int(gen.integers(0, 4))
        t = gen.uniform(-1, 1, shape)
        m = [gen.uniform(-1, 1, (d, r)) for d in shape]
        prov = P.GpuDenseProvider(t)
        for mode in range(len(shape)):
            assert rel_fro(prov.mttkrp(m, mode), oracle.ref_mttkrp(t, m, mode)) < 1e-12


@pytest.mark.parametrize("shape,rank", [([50, 50, 50], 10), ([37, 41, 29], 20), ([20, 21, 22, 23], 16),
                                        ([300, 30, 30], 20), ([8, 200, 64], 12), ([64, 48, 32], 32),
                                        ([40, 30, 20], 64)])
def test_mttkrp_medium_f64(P, oracle, shape, rank):
    gen = np.random.default_rng(sum(shape) + rank)
    t = gen.random(shape)
    m = [gen.random((d, rank)) for d in shape]
    prov = P.GpuDenseProvider(t)
    for mode in range(len(shape)):
        assert rel_fro(prov.mttkrp(m, mode), oracle.mttkrp(t, m, mode)) < 1e-12


@pytest.mark.parametrize("mma", ["1", "0"], ids=["dmma", "dfma"])
@pytest.mark.parametrize("shape,rank", [([300, 30, 30], 20), ([64, 48, 32], 32), ([20, 21, 22, 23], 16),
                                        ([40, 30, 20], 64), ([96, 40, 50], 8)])
def test_mttkrp_f64_consumer_kinds(P, oracle, monkeypatch, shape, rank, mma):
    """FP64 fast MTTKRP with DMMA consumers (default) and with the DFMA
    register tiles (NTF_FAST_MMA=0), ROW and COL views, 1e-12 vs the oracle."""
    monkeypatch.setenv("NTF_FAST_MMA", mma)
    gen = np.random.default_rng(7 * sum(shape) + rank)
    t = gen.random(shape)
    m = [gen.random((d, rank)) for d in shape]
    prov = P.GpuDenseProvider(t)
    for mode in range(len(shape)):
        assert rel_fro(prov.mttkrp(m, mode), oracle.mttkrp(t, m, mode)) < 1e-12
    prov.close()


@pytest.mark.parametrize("shape,rank", [([50, 50, 50], 10), ([60, 50, 40], 32), ([30, 20, 40], 64)])
def test_mttkrp_f32(P, oracle, shape, rank):
    gen = np.random.default_rng(3 + rank)
    t = gen.random(shape).astype(np.float32)
    m = [gen.random((d, rank)) for d in shape]
    prov = P.GpuDenseProvider(t)
    for mode in range(len(shape)):
        assert rel_fro(prov.mttkrp(m, mode), oracle.mttkrp(t, m, mode)) < 1e-5


def test_objective_vs_residual(P, oracle):
    gen = np.random.default_rng(10)
    m = [gen.random((d, 2)) for d in (3, 4, 2)]
    t = oracle.reconstruct(m)
    prov = P.GpuDenseProvider(t)
    nsq = prov.norm_sq()
    assert abs(prov.objective(m)) <= 1e-12 * nsq
    z = [np.zeros((d, 2)) for d in (3, 4, 2)]
    assert abs(prov.objective(z) - 0.5 * nsq) <= 1e-14 * nsq
    for _ in range(30):
        shape = _shape_gen(gen)
        r = 1 + int(gen.integers(0, 4))
        rt = gen.random(shape)
        rm = [gen.random((d, r)) for d in shape]
        want = oracle.ref_objective(rt, rm)
        p = P.GpuDenseProvider(rt)
        for pivot in range(len(shape)):
            assert abs(p.objective(rm, pivot) - want) <= 1e-10 * abs(want)


def test_norm_sq(P, oracle):
    gen = np.random.default_rng(1)
    t = gen.random((37, 23, 19))
    assert abs(P.GpuDenseProvider(t).norm_sq() - oracle.norm_sq(t)) <= 1e-13 * oracle.norm_sq(t)


# ---- AHALS --------------------------------------------------------------------------

def _convex_problem(gen, rows, r):
    rm = gen.uniform(-1, 1, (r + 2, r))
    g = rm.T @ rm + 0.1 * np.eye(r)
    return g, gen.uniform(-1, 1, (rows, r)), gen.random((rows, r))


def test_ahals_basic_properties(P, oracle):
    gen = np.random.default_rng(1)
    c = gen.uniform(-1, 1, (5, 3))
    out = P.solve_nnls(P.NnlsSolver.ahals, np.eye(3), c, np.zeros((5, 3)), P.InnerStop(1, 1e-2))
    assert np.array_equal(out, np.maximum(c, 0.0))
    neg = -gen.random((5, 3))
    assert np.abs(P.solve_nnls(0, np.eye(3), neg, np.zeros((5, 3)), P.InnerStop(1, 1e-2))).max() == 0.0
    # degenerate column untouched
    g = np.zeros((2, 2))
    g[0, 0] = 1.0
    w0 = gen.random((3, 2))
    out = P.solve_nnls(0, g, gen.uniform(-1, 1, (3, 2)), w0, P.InnerStop(1, 1e-2))
    assert np.array_equal(out[:, 1], w0[:, 1])
    # fixed point stops early
    c = gen.uniform(-1, 1, (4, 3))
    assert np.array_equal(P.solve_nnls(0, np.eye(3), c, np.maximum(c, 0), P.InnerStop(50, 1e-2)), np.maximum(c, 0))
    # every solver keeps a fixed point of the NNLS (nnls.cpp:51-211 on the GPU)
    for solver in (P.NnlsSolver.admm, P.NnlsSolver.pgd, P.NnlsSolver.nesterov, P.NnlsSolver.active_set):
        got = P.solve_nnls(solver, np.eye(3), c, np.maximum(c, 0))
        assert np.abs(got - np.maximum(c, 0)).max() <= 1e-14


@pytest.mark.parametrize("rows,r", [(4, 2), (6, 3), (300, 20), (500, 32), (100, 16), (2000, 64), (1100, 10)])
def test_ahals_vs_oracle(P, oracle, rows, r):
    gen = np.random.default_rng(rows * 7 + r)
    g, c, w0 = _convex_problem(gen, rows, r)
    c = c * 10
    for it in (1, 5, 50):
        got, sw = P.solve_nnls(0, g, c, w0, P.InnerStop(it, 1e-2), return_sweeps=True)
        want, sw_o = oracle.ahals_solve(g, c, w0, it, 1e-2, return_sweeps=True)
        assert sw == sw_o
        assert rel_fro(got, want) < 1e-12


# ---- drivers -------------------------------------------------------------------------

def _instance(P, shape, rank, sigma, seed, ill=False):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, ill_conditioned=ill, seed=seed)
    t, truth = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(seed, 1))
    return t, truth, init


@pytest.mark.parametrize("shape,rank,sigma,seed", [([50, 50, 50], 10, 0.01, 101), ([30, 30, 30], 5, 0.0, 4000),
                                                   ([8, 7, 6], 3, 0.05, 7), ([20, 20, 20, 20], 4, 0.01, 103),
                                                   ([12, 9], 2, 0.01, 402), ([15, 12, 10], 4, 0.001, 97)])
@pytest.mark.parametrize("flags", [0, 8, 16], ids=["tree", "direct", "tree-no-overlap"])
def test_her_trace_parity(P, oracle, shape, rank, sigma, seed, flags):
    """Default flags = the dimension tree with the overlapped 3-way pass;
    RUN_DIRECT = N full passes; RUN_NO_OVERLAP = the tree without it."""
    t, truth, init = _instance(P, shape, rank, sigma, seed, ill=(seed == 97))
    cfg = P.AoConfig(max_outer_iters=50, flags=flags)
    model, trace = P.her_run(t, init, cfg, P.HerParams())
    fo, f0, recs = oracle.run("her", t, init.factors, max_outer_iters=50)
    stats = compare_traces(trace, f0, recs, oracle.norm_sq(t))
    assert stats["checked"] == 50
    trace.validate()
    assert model.is_nonnegative()
    # final factors and the factor-fitting error e_k (metrics.cpp:79-111)
    for a, b in zip(model, fo):
        assert rel_fro(a, b) < 1e-6
    e_gpu = P.factor_error(model, truth)
    e_ora = oracle.factor_error(fo, truth.factors)
    # e is a normalised error (<= ~2): the factors agree to 1e-6, so e to 1e-6 absolute
    assert abs(e_gpu - e_ora) <= 1e-6, (e_gpu, e_ora)


@pytest.mark.parametrize("shape,rank,sigma,seed", [([50, 50, 50], 10, 0.01, 101), ([6, 5, 4], 3, 0.1, 29),
                                                   ([5, 4, 3, 6], 2, 0.01, 404)])
def test_ao_trace_parity(P, oracle, shape, rank, sigma, seed):
    t, truth, init = _instance(P, shape, rank, sigma, seed)
    cfg = P.AoConfig(max_outer_iters=50)
    model, trace = P.ao_run(t, init, cfg)
    fo, f0, recs = oracle.run("ao", t, init.factors, max_outer_iters=50)
    compare_traces(trace, f0, recs, oracle.norm_sq(t), check_restarts=False)
    prev = trace.f0
    for r in trace.records:  # monotone (test_ao.cpp:83-104)
        assert r.f <= prev + 1e-12 * trace.f0
        prev = r.f
    for a, b in zip(model, fo):
        assert rel_fro(a, b) < 1e-6


def test_beta_zero_reduces_to_ao(P):
    """test_her.cpp:113-135 / acceptance.cpp:387-415 on the GPU path."""
    for seed in (101, 102, 103, 104, 105):
        t, _, _ = _instance(P, [6, 5, 4], 2, 0.05, seed)
        init = P.random_init([6, 5, 4], 2, seed + 1000)
        cfg = P.AoConfig(max_outer_iters=50)
        _, at = P.ao_run(t, init, cfg)
        _, ht = P.her_run(t, init, cfg, P.HerParams(beta0=1e-300))
        assert len(at.records) == len(ht.records) == 50
        for a, h in zip(at.records, ht.records):
            assert abs(h.f - a.f) <= 1e-12 * max(abs(a.f), abs(h.f))


def test_her_bookkeeping_observer(P):
    """test_her.cpp:137-179."""
    t, _, _ = _instance(P, [8, 7, 6], 3, 0.05, 7)
    init = P.random_init([8, 7, 6], 3, 71)
    seen = []

    def obs(info):
        assert info.factors.is_nonnegative() and info.hat_factors.is_nonnegative()
        if info.restarted:
            for a, h in zip(info.factors, info.hat_factors):
                assert np.array_equal(a, h)
        seen.append(info.restarted)

    model, trace = P.her_run(t, init, P.AoConfig(max_outer_iters=200), P.HerParams(), observer=obs)
    trace.validate()
    assert len(seen) == 200 and trace.restart_count() == sum(seen)
    prev = trace.f0
    for r in trace.records:
        if not r.restarted:
            assert r.f <= prev + 1e-12 * trace.f0
            prev = r.f


def test_her_beats_ao_noiseless(P):
    """test_her.cpp:181-204."""
    her_f, ao_f = [], []
    for s in range(5):
        t, _, _ = _instance(P, [15, 15, 15], 3, 0.0, 200 + s)
        init = P.random_init([15, 15, 15], 3, 300 + s)
        cfg = P.AoConfig(max_outer_iters=150)
        ao_f.append(P.ao_run(t, init, cfg)[1].final_f())
        her_f.append(P.her_run(t, init, cfg, P.HerParams())[1].final_f())
    assert sorted(her_f)[2] < sorted(ao_f)[2]


def test_identical_inputs_identical_traces(P):
    t, _, _ = _instance(P, [6, 6, 6], 2, 0.01, 83)
    init = P.random_init([6, 6, 6], 2, 89)
    cfg = P.AoConfig(max_outer_iters=40)
    _, a = P.her_run(t, init, cfg)
    _, b = P.her_run(t, init, cfg)
    assert [(r.f, r.beta, r.restarted) for r in a.records] == [(r.f, r.beta, r.restarted) for r in b.records]


def test_time_budget_and_factor_error(P):
    t, truth, _ = _instance(P, [10, 10, 10], 3, 0.0, 47)
    cfg = P.AoConfig(max_time_s=0.05)
    _, trace = P.ao_run(t, P.random_init([10, 10, 10], 3, 51), cfg)
    assert trace.records and trace.records[-1].time_s >= 0.05
    t, truth, _ = _instance(P, [6, 6, 6], 2, 0.0, 53)
    cfg = P.AoConfig(max_outer_iters=30, record_factor_error=True, ground_truth=truth)
    _, trace = P.ao_run(t, P.random_init([6, 6, 6], 2, 57), cfg)
    assert trace.records[-1].e is not None and trace.records[-1].e < trace.records[0].e


def test_rank_one_fit_and_exact_factorization(P, oracle):
    """test_ao.cpp:35-54."""
    t, _, _ = _instance(P, [2, 2, 2], 1, 0.0, 3)
    _, trace = P.ao_run(t, P.random_init([2, 2, 2], 1, 17), P.AoConfig(max_outer_iters=50))
    nsq = oracle.norm_sq(t)
    assert trace.final_f() <= 1e-12 * nsq and len(trace.records) == 50
    gen = np.random.default_rng(5)
    exact = [gen.uniform(0.1, 1.0, (d, 2)) for d in (4, 3, 3)]
    t = oracle.reconstruct(exact)
    _, trace = P.ao_run(t, exact, P.AoConfig(max_outer_iters=10))
    for r in trace.records:
        assert abs(r.f) <= 1e-12 * oracle.norm_sq(t)


def test_driver_validation(P):
    t, _, init = _instance(P, [5, 5, 5], 2, 0.0, 1)
    with pytest.raises(ValueError):
        P.her_run(t, init, P.AoConfig())  # no budget
    with pytest.raises(ValueError):
        P.her_run(t, init, P.AoConfig(max_outer_iters=3), P.HerParams(beta0=0.0))
    bad = [f.copy() for f in init]
    bad[0][0, 0] = -1.0
    with pytest.raises(ValueError):
        P.her_run(t, bad, P.AoConfig(max_outer_iters=3))
    with pytest.raises(P.LogicError, match="unknown solver"):
        P.her_run(t, init, P.AoConfig(solver=7, max_outer_iters=3))


@pytest.mark.parametrize("shape,rank,seed", [([5000, 6, 5], 3, 1), ([9, 4500, 7], 4, 2), ([6, 5, 4100], 2, 3)])
@pytest.mark.parametrize("algo", ["her", "ao"])
def test_factors_taller_than_one_cluster(P, oracle, algo, shape, rank, seed):
    """The reference has no factor-height limit (nnls.cpp:15-49 loops over all
    rows). A mode beyond one 16-CTA cluster (4096 rows) takes the grid-kernel
    block update (kernels_nnls_tall.cu) -- first, middle or last mode -- with
    the same trace, decisions, factors and e_k as the oracle."""
    t, truth, init = _instance(P, shape, rank, 0.01, seed)
    cfg = P.AoConfig(max_outer_iters=12)
    if algo == "her":
        model, trace = P.her_run(t, init, cfg, P.HerParams())
    else:
        model, trace = P.ao_run(t, init, cfg)
    fo, f0, recs = oracle.run(algo, t, init.factors, max_outer_iters=12)
    stats = compare_traces(trace, f0, recs, oracle.norm_sq(t), n_check=12, check_restarts=(algo == "her"))
    assert stats["checked"] == 12
    for a, b in zip(model, fo):
        assert rel_fro(a, b) < 1e-6
    assert abs(P.factor_error(model, truth) - oracle.factor_error(fo, truth.factors)) <= 1e-6


def test_tall_standalone_ahals_and_solver_limits(P, oracle):
    """ntf_solve_nnls on 6000 rows: the same iterate and sweep count as the
    oracle; the other inner solvers still refuse factors beyond one cluster."""
    gen = np.random.default_rng(11)
    rows, r = 6000, 8
    b = gen.random((rows // 10, r))
    g = b.T @ b
    c = gen.random((rows, r)) * r
    w0 = gen.random((rows, r))
    for max_iters, tol in ((50, 1e-2), (5, 0.0)):
        want, sweeps = oracle.ahals_solve(g, c, w0, max_iters, tol, return_sweeps=True)
        got, got_sweeps = P.ahals_solve(g, c, w0, P.InnerStop(max_iters, tol), return_sweeps=True)
        assert got_sweeps == sweeps
        assert rel_fro(got, want) < 1e-12
    t, _, init = _instance(P, [5000, 2, 2], 1, 0.0, 1)
    with pytest.raises(P.UnsupportedError, match="4096"):
        P.her_run(t, init, P.AoConfig(max_outer_iters=2, solver=P.NnlsSolver.pgd))


@pytest.mark.parametrize("shape,rank", [([40, 30, 20], 100), ([60, 20, 12], 128), ([12, 10, 9, 8], 72)])
def test_ranks_above_the_fused_kernels_limit(P, oracle, shape, rank):
    """The reference has no rank limit. Ranks above 64 (the fused kernels'
    register budget) run the generic MTTKRP and the grid-kernel block update,
    up to r = 128: per-call MTTKRP, HER trace and standalone AHALS against
    the oracle; r = 129 and the other inner solvers above 64 are refused."""
    t, truth, init = _instance(P, shape, rank, 0.01, 5)
    prov = P.GpuDenseProvider(t)
    for mode in range(len(shape)):
        assert rel_fro(prov.mttkrp(init, mode), oracle.mttkrp(np.asarray(t), init.factors, mode)) < 1e-12
    model, trace = P.her_run(prov, init, P.AoConfig(max_outer_iters=8), P.HerParams())
    prov.close()
    fo, f0, recs = oracle.run("her", t, init.factors, max_outer_iters=8)
    compare_traces(trace, f0, recs, oracle.norm_sq(t), n_check=8)
    gen = np.random.default_rng(rank)
    b = gen.random((400, rank))
    g = b.T @ b
    c = gen.random((90, rank)) * rank
    w0 = gen.random((90, rank))
    want, sweeps = oracle.ahals_solve(g, c, w0, 20, 1e-3, return_sweeps=True)
    got, got_sweeps = P.ahals_solve(g, c, w0, P.InnerStop(20, 1e-3), return_sweeps=True)
    assert got_sweeps == sweeps and rel_fro(got, want) < 1e-11
    t2, _, init2 = _instance(P, [6, 5, 4], 129, 0.0, 1)
    with pytest.raises(P.UnsupportedError, match="128"):
        P.her_run(t2, init2, P.AoConfig(max_outer_iters=2))
    with pytest.raises(P.UnsupportedError, match="64"):
        P.her_run(t, init, P.AoConfig(max_outer_iters=2, solver=P.NnlsSolver.admm))


def test_tall_path_forced_on_small_instances_matches_the_fused_kernels():
    """NTF_NNLS_TALL=1 routes every block update through the grid-kernel path:
    the trace and AHALS parity tests of this module, re-run that way in a
    child process (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, NTF_NNLS_TALL="1")
    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_parity.py"), "-m", "gpu", "-q",
                          "-x", "-k", "her_trace_parity or ao_trace_parity or ahals_vs_oracle or bookkeeping"],
                         env=env, capture_output=True, text=True, timeout=1500)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


@pytest.mark.parametrize("shape,rank,dtype", [([120, 100, 80], 20, np.float64), ([40, 36, 34, 32], 16, np.float64),
                                              ([96, 80, 64], 32, np.float32)], ids=["3way-f64", "4way-f64", "3way-f32"])
def test_production_path_is_bitwise_deterministic(P, shape, rank, dtype):
    """test_her.cpp:251-271 on the production kernels (TMA/DMMA or FFMA
    MTTKRP with the in-kernel split-K grid barrier, tree contractions with
    self-resetting arrival counters, the stream NNLS with its st.async
    cluster exchange, graph replay): two runs from identical inputs give
    identical bits -- in traces, decisions and factors. compute-sanitizer is
    not available on the GPU pool (runs under it are refused), so this and
    the oracle parity are the race evidence."""
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=61)
    t, _ = P.generate(spec, dtype=dtype)
    init = P.random_init(shape, rank, P.stream_seed(61, 1))
    prov = P.GpuDenseProvider(t)
    runs = [P.her_run(prov, init, P.AoConfig(max_outer_iters=30), P.HerParams()) for _ in range(2)]
    (ma, ta), (mb, tb) = runs
    assert ta.f0 == tb.f0
    assert [(r.f, r.beta, r.restarted, r.inner_sweeps) for r in ta.records] == \
        [(r.f, r.beta, r.restarted, r.inner_sweeps) for r in tb.records]
    for a, b in zip(ma, mb):
        assert np.array_equal(a, b)
    prov.close()


@pytest.mark.gpu
def test_async_upload_from_pinned_memory_matches_the_blocking_upload(P):
    """ntf_tensor_upload_async (what GpuDenseProvider uses for host arrays):
    the run starts while the tensor is still in flight from pinned memory --
    session setup and graph capture overlap the copy, every consumer is
    ordered after it on the device -- and gives bit for bit the trace, factors
    and ||T||^2 of the blocking ntf_tensor_upload path."""
    import ctypes as C

    from paper_2001_04321_b200 import _lib as L
    shape, rank = [200, 160, 120], 20
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=77)
    t, _ = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(77, 1))
    host = P.pinned_empty(shape, np.float64)  # ntf_pinned_alloc: page-locked, so the copy is truly asynchronous
    np.copyto(host, t)
    cfg = P.AoConfig(max_outer_iters=12)
    runs = []
    for _ in range(2):  # the asynchronous path, run immediately after the enqueue
        prov = P.GpuDenseProvider(host)
        model, trace = P.her_run(prov, init, cfg, P.HerParams())
        runs.append((model, trace, prov.norm_sq()))
        prov.wait()
        prov.close()
    # the blocking C entry point
    ctx = P.default_context()
    h = C.c_void_p()
    arr = (C.c_int64 * 3)(*shape)
    assert L.lib().ntf_tensor_upload(ctx.handle, host.ctypes.data_as(C.c_void_p), L.NTF_DTYPE_F64, 3, arr, C.byref(h)) == 0
    prov = P.GpuDenseProvider.__new__(P.GpuDenseProvider)
    prov.ctx, prov.handle, prov._shape, prov.dtype, prov._source = ctx, h, list(shape), np.float64, host
    model, trace = P.her_run(prov, init, cfg, P.HerParams())
    nsq = prov.norm_sq()
    prov.close()
    for m2, t2, n2 in runs:
        assert n2 == nsq
        assert t2.f0 == trace.f0
        assert [r.f for r in t2.records] == [r.f for r in trace.records]
        assert [r.restarted for r in t2.records] == [r.restarted for r in trace.records]
        for a, b in zip(m2, model):
            assert np.array_equal(a, b)
