"""The reference's other inner NNLS solvers (src/nnls.cpp:51-211: PGD,
Nesterov, ADMM, active set) behind solve_nnls (nnls.cpp:213-222), on the GPU
(kernels_solvers.cu) and in the oracle restatement, following the
reference's tests/test_nnls.cpp and tests/test_ao.cpp:83-104 (monotone f for
every solver).

CPU: the oracle's solvers all reach the AHALS optimum on a strictly convex
problem, its spectral norm matches numpy's, and the reference's error texts.
GPU: per-solve parity with the oracle, the drivers with every solver against
the oracle's traces, and the error paths.
"""
import numpy as np
import pytest

from parity import compare_traces, rel_fro

SOLVERS = ["pgd", "nesterov", "admm", "active_set"]


def _problem(rows, r, seed):
    g = np.random.default_rng(seed)
    a = g.random((3 * r, r))
    G = a.T @ a + 0.1 * np.eye(r)
    C = g.random((rows, r)) * 3.0 - 0.5
    W0 = g.random((rows, r))
    return G, C, W0


def _obj(G, C, W):
    return 0.5 * np.sum((W.T @ W) * G) - np.sum(W * C)  # nnls.cpp:11-13


# ---- CPU: the oracle restatement -------------------------------------------------

def test_oracle_spectral_norm(oracle):
    """kernels.cpp:262-280 against numpy's eigen-solve."""
    for seed in range(5):
        G, _, _ = _problem(4, 7, seed)
        assert abs(oracle.spectral_norm(G) - np.linalg.eigvalsh(G).max()) <= 1e-9 * np.linalg.eigvalsh(G).max()


@pytest.mark.parametrize("solver", SOLVERS)
def test_oracle_solvers_reach_the_ahals_optimum(oracle, solver):
    """Every solver converges to the unique minimiser of the strictly convex
    NNLS (test_nnls.cpp's cross-solver checks)."""
    G, C, W0 = _problem(30, 6, 1)
    want = oracle.solve_nnls("ahals", G, C, W0, max_iters=2000, tol=1e-14)
    got = oracle.solve_nnls(solver, G, C, W0, max_iters=5000, tol=1e-14)
    assert got.min() >= 0.0
    assert abs(_obj(G, C, got) - _obj(G, C, want)) <= 1e-9 * abs(_obj(G, C, want))


def test_oracle_pgd_step_formula(oracle):
    """One PGD sweep is max(0, W - (W G - C) / L) (nnls.cpp:51-57)."""
    G, C, W0 = _problem(10, 5, 2)
    lip = oracle.spectral_norm(G)
    one = oracle.solve_nnls("pgd", G, C, W0, max_iters=1, tol=0.0)
    assert np.allclose(one, np.maximum(0.0, W0 - (W0 @ G - C) / lip), rtol=1e-14, atol=1e-15)


def test_oracle_solver_errors(oracle):
    Z = np.zeros((4, 4))
    C = np.ones((3, 4))
    for solver, msg in (("pgd", "pgd_solve: zero Gram matrix"), ("nesterov", "nesterov_solve: zero Gram matrix"),
                        ("admm", "admm_solve: zero Gram matrix"),
                        ("active_set", "active_set_solve: Gram matrix is not positive definite")):
        with pytest.raises(oracle.OracleError, match=msg):
            oracle.solve_nnls(solver, Z, C, np.ones((3, 4)))


# ---- GPU ------------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("rows,r", [(37, 5), (300, 20), (700, 32), (90, 64)])
@pytest.mark.parametrize("solver", SOLVERS)
def test_gpu_solver_matches_oracle(P, oracle, solver, rows, r):
    if solver == "active_set" and r > 32:
        pytest.skip("the GPU active set serves r <= 32")
    G, C, W0 = _problem(rows, r, rows + r)
    stop = P.InnerStop(max_iters=50, rel_change_tol=1e-2)
    got = P.solve_nnls(P.nnls_solver_from_name(solver), G, C, W0, stop)
    want = oracle.solve_nnls(solver, G, C, W0, max_iters=50, tol=1e-2)
    assert got.min() >= 0.0
    assert rel_fro(got, want) <= 1e-10, rel_fro(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["her", "ao"])
@pytest.mark.parametrize("solver", SOLVERS)
def test_gpu_drivers_with_every_solver(P, oracle, solver, algo):
    """her_run / ao_run with cfg.solver (her.cpp:65-70 calls solve_nnls):
    traces against the oracle's; AO monotone (test_ao.cpp:83-104)."""
    shape, rank = [20, 18, 16], 4
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=71)
    t, _ = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(71, 1))
    cfg = P.AoConfig(solver=P.nnls_solver_from_name(solver), max_outer_iters=15)
    if algo == "her":
        _, trace = P.her_run(t, init, cfg, P.HerParams())
    else:
        _, trace = P.ao_run(t, init, cfg)
    _, f0, recs = oracle.run(algo, t, init.factors, max_outer_iters=15, solver=solver)
    compare_traces(trace, f0, recs, oracle.norm_sq(t), n_check=15, check_restarts=(algo == "her"))
    if algo == "ao":
        prev = trace.f0
        for rec in trace.records:
            assert rec.f <= prev + 1e-12 * trace.f0
            prev = rec.f


@pytest.mark.gpu
def test_gpu_solver_errors(P):
    """A zero Gram (an all-zero factor) fails like the reference: the
    std::runtime_error texts of nnls.cpp:53,61,90 / :195."""
    Z = np.zeros((4, 4))
    C = np.ones((3, 4))
    for solver, msg in (("pgd", "pgd_solve: zero Gram matrix"), ("admm", "admm_solve: zero Gram matrix"),
                        ("active_set", "not positive definite")):
        with pytest.raises(RuntimeError, match=msg):
            P.solve_nnls(P.nnls_solver_from_name(solver), Z, C, np.ones((3, 4)))
    spec = P.SyntheticSpec(shape=[8, 7, 6], rank=2, noise_sigma=0.0, seed=3)
    t, _ = P.generate(spec)
    init = P.random_init([8, 7, 6], 2, 5)
    init.factors[1][:] = 0.0
    with pytest.raises(RuntimeError, match="nesterov_solve: zero Gram matrix"):
        P.ao_run(t, init, P.AoConfig(solver=P.NnlsSolver.nesterov, max_outer_iters=3))
