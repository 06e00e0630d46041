"""The oracle restatement against THE REFERENCE ITSELF (CPU; TEST INFRASTRUCTURE).

`oracle/_ref/libntf_ref.so` is built by `oracle/ref_build/Makefile` from the
reference's own unmodified sources where they lie under /root/reference/proj
(kernels.cpp, nnls.cpp, her.cpp, ao.cpp, kruskal.cpp, tensor.cpp,
provider.cpp, datagen.cpp, metrics.cpp, trace.cpp, reference.cpp, tucker.cpp)
against a small Eigen stand-in (`oracle/ref_build/shim/Eigen/Dense`; Eigen3
is not in this image). This module

  1. runs the reference's OWN unit suites (tests/test_{tensor,kernels,nnls,
     metrics,datagen,ao,her,tucker}.cpp, doctest stand-in) over that build --
     the build is the reference as far as its own tests can tell;
  2. pins the oracle (`oracle/pyoracle.py`) to it function by function on the
     same seeded inputs: datagen bit for bit, MTTKRP, Grams, HALS / every inner
     solver, extrapolation, beta updates, factor error, and whole HER / AO
     traces (restart decisions identical, final factors, e_k);
  3. checks the committed reference-produced golden runs at the BASELINE
     configs (tests/golden/refrun_c{2,3,4}.npz, written by
     `make_config_golden.py --ref`) against the oracle's fixtures, so the GPU
     parity tests (which use both) stand on reference output.

Where /root/reference is absent (the GPU box) and no prebuilt library
travelled, parts 1-2 skip; part 3 only reads committed files.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as O  # noqa: E402
import pyref  # noqa: E402

HAVE_REF_SOURCES = os.path.isdir(pyref.REF_ROOT)
needs_ref = pytest.mark.skipif(not pyref.available(), reason="no oracle/_ref build and no /root/reference")

EPS = 2.0 ** -52


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def R():
    if not pyref.available():
        pytest.skip("no oracle/_ref build and no /root/reference")
    assert pyref.is_reference_build()
    return pyref


# ------------------------------------------------------------------ part 1
@pytest.mark.skipif(not HAVE_REF_SOURCES, reason="/root/reference is absent")
def test_reference_unit_suites_pass_over_the_build():
    """78 doctest cases / ~8700 assertions of the reference's own tests."""
    out = subprocess.run(["make", "-s", "-j", "8", "-C", os.path.join(ROOT, "oracle", "ref_build"), "check"],
                         capture_output=True, text=True, timeout=1500)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("[shim-doctest]")]
    assert len(lines) == 8, out.stdout[-4000:]
    cases = asserts = 0
    for ln in lines:
        parts = [p.strip() for p in ln.replace("[shim-doctest]", "").split("|")]
        assert parts[1] == "failed: 0" and parts[3] == "failed: 0", ln
        cases += int(parts[0].split(":")[1])
        asserts += int(parts[2].split(":")[1])
    assert cases >= 70 and asserts >= 8000, (cases, asserts)


# ------------------------------------------------------------------ part 2
@needs_ref
def test_rng_and_datagen_bit_for_bit(R):
    assert R.mt19937_64_draw(5489, 9999) == O.mt19937_64_draw(5489, 9999) == 9981545732273789042
    for base, stream in ((0, 0), (102, 1), (2 ** 63 + 11, 7)):
        assert R.stream_seed(base, stream) == O.stream_seed(base, stream)
    uo, zo = O.uniform_normal(12345, 500)
    ur, zr = R.uniform_normal(12345, 500)
    assert np.array_equal(uo, ur) and np.array_equal(zo, zr)
    for shape, rank, sigma, ill, seed in (([9, 8, 7], 3, 0.0, False, 1), ([12, 5, 6, 4], 4, 0.05, False, 2),
                                          ([10, 11, 6], 5, 0.01, True, 3), ([30, 20], 2, 0.1, False, 4)):
        to, tro = O.generate(shape, rank, sigma, ill, seed)
        tr, trr = R.generate(shape, rank, sigma, ill, seed)
        assert np.array_equal(to, tr)
        assert all(np.array_equal(a, b) for a, b in zip(tro, trr))
        io = O.random_init(shape, rank, O.stream_seed(seed, 1))
        ir = R.random_init(shape, rank, R.stream_seed(seed, 1))
        assert all(np.array_equal(a, b) for a, b in zip(io, ir))
    with pytest.raises(ValueError):
        R.generate([4, 4, 4], 0)
    with pytest.raises(ValueError):
        R.generate([4, 4, 4], 1, ill_conditioned=True)


@needs_ref
@pytest.mark.parametrize("shape,rank", [([7, 6, 5], 3), ([5, 4, 6, 3], 2), ([16, 9], 4), ([3, 4, 2, 5, 3], 2),
                                        ([40, 30, 20], 8)])
def test_mttkrp_and_objective_parts(R, shape, rank):
    rng = np.random.default_rng(sum(shape) + rank)
    t = rng.random(shape)
    model = [rng.random((d, rank)) for d in shape]
    for mode in range(len(shape)):
        a, b = O.mttkrp(t, model, mode), R.mttkrp(t, model, mode)
        assert rel(a, b) <= 4 * EPS, (mode, rel(a, b))
        assert rel(R.ref_mttkrp(t, model, mode), b) <= 1e-13  # the reference's own serial oracle
    assert np.array_equal(O.reconstruct(model), R.reconstruct(model))
    assert O.norm_sq(t) == R.norm_sq(t)
    grams = [O.gram(a) for a in model]
    for a, go in zip(model, grams):
        assert rel(go, R.gram(a)) <= 4 * EPS
    for skip in range(len(shape)):
        assert np.array_equal(O.hadamard_of_grams(grams, skip), R.hadamard_of_grams(grams, skip))
    last = len(shape) - 1
    g = O.hadamard_of_grams(grams, last)
    c = O.mttkrp(t, model, last)
    fo = O.cheap_objective(O.norm_sq(t), model[last], g, c)
    fr = R.cheap_objective(R.norm_sq(t), model[last], g, c)
    assert abs(fo - fr) <= 64 * EPS * O.norm_sq(t)
    assert abs(R.ref_objective(t, model) - fr) <= 1e-10 * abs(fr) + 64 * EPS * O.norm_sq(t)
    bad = [a[:-1] if i == 0 else a for i, a in enumerate(model)]
    for M in (O, R):
        with pytest.raises(ValueError):  # mttkrp: model/tensor shape mismatch (kernels.cpp:162)
            M.mttkrp(t, bad, 0)


@needs_ref
@pytest.mark.parametrize("rows,r,seed", [(30, 4, 1), (200, 10, 2), (64, 20, 3), (17, 1, 4)])
def test_hals_and_inner_solvers(R, rows, r, seed):
    rng = np.random.default_rng(seed)
    b = rng.random((rows + 40, r))
    g = b.T @ b
    c = rng.random((rows, r)) * r
    w0 = rng.random((rows, r))
    assert rel(O.hals_pass(g, c, w0), R.hals_pass(g, c, w0)) <= 8 * EPS
    wo, so = O.ahals_solve(g, c, w0, 50, 1e-2, return_sweeps=True)
    wr, sr = R.ahals_solve(g, c, w0, 50, 1e-2, return_sweeps=True)
    assert so == sr and rel(wo, wr) <= 64 * EPS
    wo, so = O.ahals_solve(g, c, w0, 7, 1e-9, return_sweeps=True)
    wr, sr = R.ahals_solve(g, c, w0, 7, 1e-9, return_sweeps=True)
    assert so == sr and (so == 7 or r == 1) and rel(wo, wr) <= 64 * EPS
    for solver in ("ahals", "pgd", "nesterov", "admm", "active_set"):
        a, bb = O.solve_nnls(solver, g, c, w0, 30, 1e-3), R.solve_nnls(solver, g, c, w0, 30, 1e-3)
        assert rel(a, bb) <= 1e-9, (solver, rel(a, bb))
    assert abs(O.spectral_norm(g) - R.spectral_norm(g)) <= 1e-9 * R.spectral_norm(g)
    # a zero diagonal entry: the column is skipped (nnls.cpp:16-19)
    g2 = g.copy()
    g2[:, 0] = 0.0
    g2[0, :] = 0.0
    assert rel(O.hals_pass(g2, c, w0), R.hals_pass(g2, c, w0)) <= 8 * EPS
    assert np.array_equal(R.hals_pass(g2, c, w0)[:, 0], w0[:, 0])


@needs_ref
def test_her_building_blocks(R):
    rng = np.random.default_rng(9)
    a_new, a_old = rng.random((40, 6)), rng.random((40, 6))
    for beta in (0.0, 0.5, 0.97, 3.0):
        assert np.array_equal(O.extrapolate_block(a_new, a_old, beta), R.extrapolate_block(a_new, a_old, beta))
    st_o, st_r = (0.5, 1.0), (0.5, 1.0)
    for restarted in (False, False, True, False, True, True, False, False, False):
        st_o = O.update_betas(*st_o, restarted)
        st_r = R.update_betas(*st_r, restarted)
        assert st_o == st_r
    for bad in ((0.0, 1.05, 1.01, 1.5), (1.0, 1.05, 1.01, 1.5), (0.5, 1.0, 1.01, 1.5), (0.5, 1.05, 1.1, 1.5),
                (0.5, 1.6, 1.01, 1.5)):
        with pytest.raises(ValueError):
            O.validate_her_params(*bad)
        with pytest.raises(ValueError):
            R.validate_her_params(*bad)
    R.validate_her_params()
    est = [rng.random((d, 4)) for d in (9, 8, 7)]
    truth = [rng.random((d, 4)) for d in (9, 8, 7)]
    assert abs(O.factor_error(est, truth) - R.factor_error(est, truth)) <= 1e-13
    perm = [a[:, [2, 0, 3, 1]] * np.array([3.0, 0.5, 2.0, 7.0]) for a in truth]
    assert R.factor_error(perm, truth) <= 1e-12 and O.factor_error(perm, truth) <= 1e-12
    cost = rng.random((6, 6))
    assert O.hungarian(cost)[0] == R.hungarian(cost)[0]


RUNS = [  # shape, rank, sigma, ill, seed, iters
    ([20, 16, 12], 5, 0.01, False, 7, 50),
    ([8, 7, 6, 5], 3, 0.0, False, 8, 50),
    ([30, 24, 18], 8, 0.05, True, 9, 40),
    ([50, 50, 50], 10, 0.0, False, 101, 50),  # BASELINE config 1
]


@needs_ref
@pytest.mark.parametrize("shape,rank,sigma,ill,seed,iters", RUNS)
@pytest.mark.parametrize("algo", ["her", "ao"])
def test_whole_traces(R, algo, shape, rank, sigma, ill, seed, iters):
    """her_run / ao_run of the reference against the restatement: f0 equal,
    restart decisions and beta_k identical, f_k to 1e-10, final factors and
    e_k to rounding."""
    t, truth = O.generate(shape, rank, sigma, ill, seed)
    init = O.random_init(shape, rank, O.stream_seed(seed, 1))
    fo, f0o, ro = O.run(algo, t, init, max_outer_iters=iters, truth=truth)
    fr, f0r, rr = R.run(algo, t, init, max_outer_iters=iters, truth=truth)
    nsq = O.norm_sq(t)
    assert abs(f0o - f0r) <= 64 * EPS * nsq
    assert len(ro) == len(rr) == iters
    for a, b in zip(ro, rr):
        assert a["iter"] == b["iter"]
        assert abs(a["f"] - b["f"]) <= 1e-10 * abs(b["f"]) + 64 * EPS * nsq, (a, b)
        assert a["restarted"] == b["restarted"]
        if algo == "her":
            assert a["beta"] == b["beta"]
        else:
            assert b["restarted"] is None and b["beta"] is None
        assert abs(a["e"] - b["e"]) <= 1e-9 * max(b["e"], 1e-12), (a, b)
    for a, b in zip(fo, fr):
        assert rel(a, b) <= 1e-10


@needs_ref
@pytest.mark.parametrize("solver", ["pgd", "nesterov", "admm", "active_set"])
def test_other_solvers_inside_the_drivers(R, solver):
    shape, rank = [14, 12, 10], 4
    t, _ = O.generate(shape, rank, 0.02, False, 21)
    init = O.random_init(shape, rank, O.stream_seed(21, 1))
    for algo in ("her", "ao"):
        _, f0o, ro = O.run(algo, t, init, max_outer_iters=15, solver=solver)
        _, f0r, rr = R.run(algo, t, init, max_outer_iters=15, solver=solver)
        assert abs(f0o - f0r) <= 1e-12 * abs(f0r)
        for a, b in zip(ro, rr):
            assert abs(a["f"] - b["f"]) <= 1e-8 * abs(b["f"]), (solver, algo, a, b)
            assert a["restarted"] == b["restarted"]


@needs_ref
def test_observer_and_input_checks(R):
    shape, rank = [10, 9, 8], 3
    t, _ = O.generate(shape, rank, 0.01, False, 31)
    init = O.random_init(shape, rank, O.stream_seed(31, 1))
    seen = {"o": [], "r": []}
    O.run("her", t, init, max_outer_iters=12, observer=lambda k, f, rs, b, acc, hat: seen["o"].append((k, rs, b, acc, hat)))
    R.run("her", t, init, max_outer_iters=12, observer=lambda k, f, rs, b, acc, hat: seen["r"].append((k, rs, b, acc, hat)))
    assert len(seen["o"]) == len(seen["r"]) == 12
    for a, b in zip(seen["o"], seen["r"]):
        assert a[:3] == b[:3]
        assert all(rel(x, y) <= 1e-10 for x, y in zip(a[3], b[3]))
        assert all(rel(x, y) <= 1e-10 for x, y in zip(a[4], b[4]))
    bad = [a.copy() for a in init]
    bad[1][0, 0] = -1.0
    for M in (O, R):
        with pytest.raises(ValueError):
            M.run("her", t, bad, max_outer_iters=2)  # entrywise nonnegative init
        with pytest.raises(ValueError):
            M.run("ao", t, init)  # no budget
        with pytest.raises(ValueError):
            M.run("her", t, init, max_outer_iters=2, beta0=1.5)


@needs_ref
def test_compressed_mttkrp(R):
    rng = np.random.default_rng(17)
    full, ranks, r = [12, 10, 9], [4, 3, 5], 3
    core = rng.random(ranks)
    bases = [np.linalg.qr(rng.standard_normal((d, k)))[0] for d, k in zip(full, ranks)]
    model = [rng.random((d, r)) for d in full]
    for mode in range(3):
        assert rel(O.compressed_mttkrp(core, bases, model, mode), R.compressed_mttkrp(core, bases, model, mode)) <= 1e-12


# ------------------------------------------------------------------ part 3
def _npz(kind, name):
    return dict(np.load(os.path.join(HERE, "golden", f"{kind}_{name}.npz"), allow_pickle=False))


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_reference_runs_at_the_baseline_configs_match_the_oracle_fixtures(name):
    """The committed reference-produced runs (50 iterations of her_run and
    ao_run by the reference itself at BASELINE configs 2, 3, collinear 4)
    against the oracle's fixtures of the same instances."""
    ref, ora = _npz("refrun", name), _npz("config", name)
    for k in ("shape", "rank", "sigma", "seed", "iters", "t_head", "t_tail"):
        assert np.array_equal(ref[k], ora[k]), k
    nsq = float(ora["norm_sq"])
    assert abs(float(ref["norm_sq"]) - nsq) <= 1e-13 * nsq
    assert np.array_equal(ref["her_restarted"], ora["her_restarted"])
    assert np.array_equal(ref["her_beta"], ora["her_beta"])
    for algo in ("her", "ao"):
        assert abs(float(ref[f"{algo}_f0"]) - float(ora[f"{algo}_f0"])) <= 64 * EPS * nsq
        dev = np.abs(ref[f"{algo}_f"] - ora[f"{algo}_f"])
        assert np.all(dev <= 1e-10 * np.abs(ref[f"{algo}_f"]) + 64 * EPS * nsq), dev.max()
        for i in range(len(ora["shape"])):
            assert rel(ora[f"{algo}_final{i}"], ref[f"{algo}_final{i}"]) <= 1e-10
        assert abs(float(ref[f"{algo}_e"]) - float(ora[f"{algo}_e"])) <= 1e-9 * float(ref[f"{algo}_e"])
