"""Pins the CPU oracle (test infrastructure) against every known answer and
property the reference's own test suites hold for the hot path.

Each test cites the reference test it restates (/root/reference/proj/tests).
These run without a GPU.
"""
import itertools

import numpy as np
import pytest

from parity import rel_fro


def _rand_shape(gen, max_order=4):
    order = 2 + int(gen.integers(0, max_order - 1))
    return [int(gen.integers(1, 7)) for _ in range(order)]


# ---- datagen (test_datagen.cpp) ------------------------------------------------------

def test_mt19937_64_pinned_by_the_standard(oracle):
    """test_datagen.cpp:10-16: 10000th draw of the default-seeded engine."""
    assert oracle.mt19937_64_draw(5489, 9999) == 9981545732273789042


def test_noiseless_instances_factor_exactly(oracle):
    """test_datagen.cpp:18-31."""
    t, truth = oracle.generate([6, 5, 4], 3, seed=42)
    assert np.array_equal(t, oracle.reconstruct(truth))
    assert oracle.ref_objective(t, truth) <= 1e-12 * oracle.norm_sq(t)


def test_entries_nonnegative_under_large_noise(oracle):
    t, truth = oracle.generate([5, 5, 5], 2, sigma=2.0, seed=7)
    assert (t >= 0).all() and all((a >= 0).all() for a in truth)


def test_generation_deterministic_per_seed(oracle):
    a, ma = oracle.generate([4, 3, 5], 2, sigma=0.1, seed=1234)
    b, mb = oracle.generate([4, 3, 5], 2, sigma=0.1, seed=1234)
    c, _ = oracle.generate([4, 3, 5], 2, sigma=0.1, seed=1235)
    assert np.array_equal(a, b) and all(np.array_equal(x, y) for x, y in zip(ma, mb))
    assert not np.array_equal(a, c)


def test_random_init_deterministic_in_unit_interval(oracle):
    a = oracle.random_init([4, 6], 3, 99)
    b = oracle.random_init([4, 6], 3, 99)
    c = oracle.random_init([4, 6], 3, 100)
    for x, y in zip(a, b):
        assert np.array_equal(x, y) and (x >= 0).all() and (x < 1).all()
    assert not np.array_equal(a[0], c[0])


def test_ill_conditioning_transform(oracle):
    """test_datagen.cpp:44-61 (column rule)."""
    _, plain = oracle.generate([12, 10, 8], 4, seed=5)
    _, sick = oracle.generate([12, 10, 8], 4, seed=5, ill_conditioned=True)
    for p, s in zip(plain, sick):
        assert np.array_equal(s[:, 0], 0.99 * p[:, 1] + 0.01 * p[:, 0])
        assert np.array_equal(s[:, 1], p[:, 1])


def test_datagen_validation(oracle):
    with pytest.raises(ValueError):
        oracle.generate([3, 3], 0)
    with pytest.raises(ValueError):
        oracle.generate([3, 3], 1, ill_conditioned=True)
    with pytest.raises(ValueError):
        oracle.generate([3, 3], 1, sigma=-0.5)


def test_stream_seed_is_splitmix64(oracle):
    """datagen.cpp:30-35: sub-stream k = (k+1)-th SplitMix64 output."""
    def splitmix(state):
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return state, z ^ (z >> 31)
    for base in (0, 1, 101, 2**63 + 5):
        s = base
        for k in range(4):
            s, out = splitmix(s)
            assert oracle.stream_seed(base, k) == out


# ---- kernels (test_kernels.cpp) ------------------------------------------------------

def test_mttkrp_rank_one_zero_and_mismatch(oracle):
    """test_kernels.cpp:121-136."""
    gen = np.random.default_rng(6)
    m = [gen.random((d, 1)) for d in (3, 4, 2)]
    t = oracle.reconstruct(m)
    assert rel_fro(oracle.mttkrp(t, m, 0), m[0] * np.sum(m[1] ** 2) * np.sum(m[2] ** 2)) < 1e-14
    assert np.abs(oracle.mttkrp(np.zeros((3, 4, 2)), m, 1)).max() == 0.0
    with pytest.raises(ValueError):
        oracle.mttkrp(t, [gen.random((d, 1)) for d in (3, 4, 3)], 0)


def test_mttkrp_vs_enumeration_40_shapes(oracle):
    """test_kernels.cpp:138-153 — and against numpy's own einsum."""
    gen = np.random.default_rng(7)
    for _ in range(40):
        shape = _rand_shape(gen)
        r = 1 + int(gen.integers(0, 4))
        t = gen.uniform(-1, 1, shape)
        m = [gen.uniform(-1, 1, (d, r)) for d in shape]
        for mode in range(len(shape)):
            got = oracle.mttkrp(t, m, mode)
            assert rel_fro(got, oracle.ref_mttkrp(t, m, mode)) < 1e-12
            letters = "abcdefgh"[:len(shape)]
            spec = letters + "," + ",".join(f"{c}z" for i, c in enumerate(letters) if i != mode)
            want = np.einsum(spec + "->" + letters[mode] + "z", t, *[m[i] for i in range(len(shape)) if i != mode])
            assert rel_fro(got, want) < 1e-12


def test_hadamard_of_grams_equals_kr_gram(oracle):
    """test_kernels.cpp:155-191."""
    gen = np.random.default_rng(8)
    for _ in range(30):
        shape = [int(gen.integers(1, 7)) for _ in range(3)]
        r = 1 + int(gen.integers(0, 4))
        m = [gen.uniform(-1, 1, (d, r)) for d in shape]
        grams = [oracle.gram(a) for a in m]
        for mode in range(3):
            others = [m[l] for l in range(3) if l != mode]
            kr = np.einsum("ir,jr->ijr", others[0], others[1]).reshape(-1, r)
            assert rel_fro(oracle.hadamard_of_grams(grams, mode), kr.T @ kr) < 1e-12


def test_cheap_objective_vs_residual_every_pivot(oracle):
    """test_kernels.cpp:222-248."""
    gen = np.random.default_rng(10)
    m = [gen.random((d, 2)) for d in (3, 4, 2)]
    t = oracle.reconstruct(m)
    nsq = oracle.norm_sq(t)
    grams = [oracle.gram(a) for a in m]
    c = oracle.mttkrp(t, m, 2)
    assert abs(oracle.cheap_objective(nsq, m[2], oracle.hadamard_of_grams(grams, 2), c)) <= 1e-12 * nsq
    for _ in range(30):
        shape = _rand_shape(gen)
        r = 1 + int(gen.integers(0, 4))
        rt = gen.random(shape)
        rm = [gen.random((d, r)) for d in shape]
        want = oracle.ref_objective(rt, rm)
        gr = [oracle.gram(a) for a in rm]
        for pivot in range(len(shape)):
            got = oracle.cheap_objective(oracle.norm_sq(rt), rm[pivot], oracle.hadamard_of_grams(gr, pivot),
                                         oracle.mttkrp(rt, rm, pivot))
            assert abs(got - want) <= 1e-10 * abs(want)


# ---- NNLS (test_nnls.cpp) ---------------------------------------------------------------

def _convex(gen, rows, r):
    rm = gen.uniform(-1, 1, (r + 2, r))
    return rm.T @ rm + 0.1 * np.eye(r), gen.uniform(-1, 1, (rows, r)), gen.random((rows, r))


def test_hals_pass_column_formula(oracle):
    """test_nnls.cpp:56-100."""
    gen = np.random.default_rng(1)
    c = gen.uniform(-1, 1, (5, 3))
    assert np.array_equal(oracle.hals_pass(np.eye(3), c, np.zeros((5, 3))), np.maximum(c, 0))
    assert np.abs(oracle.hals_pass(np.eye(3), -gen.random((5, 3)), np.zeros((5, 3)))).max() == 0.0
    g, c, w0 = _convex(gen, 4, 2)
    w = w0.copy()
    for j in range(2):
        for i in range(4):
            numer = c[i, j] - sum(w[i, l] * g[l, j] for l in range(2) if l != j)
            w[i, j] = max(0.0, numer / g[j, j])
    assert rel_fro(oracle.hals_pass(g, c, w0), w) < 1e-15
    g, c, cur = _convex(gen, 6, 3)
    obj = lambda w: 0.5 * np.sum((w.T @ w) * g) - np.sum(w * c)  # noqa: E731
    for _ in range(10):
        nxt = oracle.hals_pass(g, c, cur)
        assert obj(nxt) <= obj(cur) + 1e-14
        cur = nxt
    d = np.zeros((2, 2))
    d[0, 0] = 1.0
    w0 = gen.random((3, 2))
    assert np.array_equal(oracle.hals_pass(d, gen.uniform(-1, 1, (3, 2)), w0)[:, 1], w0[:, 1])


def test_ahals_fixed_point_and_brute_force(oracle):
    """test_nnls.cpp:102-112 and the 2^r active-set brute force (:25-52)."""
    gen = np.random.default_rng(2)
    c = gen.uniform(-1, 1, (4, 3))
    assert np.array_equal(oracle.ahals_solve(np.eye(3), c, np.maximum(c, 0)), np.maximum(c, 0))
    assert np.array_equal(oracle.ahals_solve(np.eye(3), c, np.zeros((4, 3))), np.maximum(c, 0))
    g, c, w0 = _convex(gen, 5, 3)
    w = oracle.ahals_solve(g, c, w0, max_iters=5000, tol=1e-14)
    for i in range(5):
        best, best_obj = np.zeros(3), 0.0
        for mask in range(1, 8):
            s = [j for j in range(3) if mask >> j & 1]
            z = np.linalg.solve(g[np.ix_(s, s)], c[i, s])
            if (z < -1e-12).any():
                continue
            x = np.zeros(3)
            x[s] = np.maximum(z, 0)
            o = 0.5 * x @ g @ x - c[i] @ x
            if o < best_obj:
                best, best_obj = x, o
        assert np.abs(w[i] - best).max() < 1e-8


# ---- HER / AO (test_her.cpp, test_ao.cpp) --------------------------------------------------

def test_extrapolate_block(oracle):
    """test_her.cpp:17-28."""
    gen = np.random.default_rng(1)
    a, b = gen.random((3, 2)), gen.random((3, 2))
    assert np.array_equal(oracle.extrapolate_block(a, b, 0.0), a)
    assert np.array_equal(oracle.extrapolate_block(a, a, 0.7), a)
    assert oracle.extrapolate_block(np.array([[1.0]]), np.array([[3.0]]), 0.5)[0, 0] == 0.0


def test_update_betas_arithmetic_and_fuzz(oracle):
    """test_her.cpp:30-67."""
    b, bb = oracle.update_betas(0.5, 1.0, True)
    assert b == pytest.approx(0.5 / 1.5) and bb == pytest.approx(0.5)
    b, bb = oracle.update_betas(0.5, 1.0, False)
    assert b == pytest.approx(0.525) and bb == pytest.approx(1.0)
    b, bb = oracle.update_betas(0.99, 1.0, False)
    assert b == pytest.approx(1.0) and bb == pytest.approx(1.0)
    gen = np.random.default_rng(2)
    b, bb = 0.5, 1.0
    for _ in range(1000):
        b, bb = oracle.update_betas(b, bb, bool(gen.integers(0, 2)))
        assert 0 < b <= bb <= 1.0


def test_her_param_validation(oracle):
    """test_her.cpp:69-79."""
    with pytest.raises(ValueError):
        oracle.validate_her_params(beta0=0.0)
    with pytest.raises(ValueError):
        oracle.validate_her_params(gamma_bar=1.0)
    with pytest.raises(ValueError):
        oracle.validate_her_params(eta=1.01)
    oracle.validate_her_params()


def test_f_hat_equals_residual_at_mixed_point(oracle):
    """test_her.cpp:81-111: cheap criterion at (hat blocks 0..N-2, plain last)."""
    gen = np.random.default_rng(3)
    for _ in range(20):
        shape = [3, 4, 2, 3]
        hat = [gen.random((d, 3)) for d in shape]
        t = gen.random(shape)
        c = oracle.mttkrp(t, hat, 3)
        a_last = gen.random((3, 3))
        g = oracle.hadamard_of_grams([oracle.gram(a) for a in hat], 3)
        mixed = hat[:3] + [a_last]
        assert abs(oracle.cheap_objective(oracle.norm_sq(t), a_last, g, c) - oracle.ref_objective(t, mixed)) \
            <= 1e-10 * oracle.ref_objective(t, mixed)


def test_beta_zero_reduces_to_ao(oracle):
    """test_her.cpp:113-135."""
    for seed in (101, 102, 103, 104, 105):
        t, _ = oracle.generate([6, 5, 4], 2, sigma=0.05, seed=seed)
        init = oracle.random_init([6, 5, 4], 2, seed + 1000)
        _, _, ar = oracle.run("ao", t, init, max_outer_iters=50)
        _, _, hr = oracle.run("her", t, init, max_outer_iters=50, beta0=1e-300)
        assert len(ar) == len(hr) == 50
        for a, h in zip(ar, hr):
            assert abs(h["f"] - a["f"]) <= 1e-12 * max(abs(a["f"]), abs(h["f"]))


def test_restart_bookkeeping(oracle):
    """test_her.cpp:137-179."""
    t, _ = oracle.generate([8, 7, 6], 3, sigma=0.05, seed=7)
    init = oracle.random_init([8, 7, 6], 3, 71)
    seen = []

    def obs(k, f, restarted, beta, acc, hat):
        assert all((a >= 0).all() for a in acc) and all((h >= 0).all() for h in hat)
        if restarted:
            assert all(np.array_equal(a, h) for a, h in zip(acc, hat))
        seen.append(restarted)

    _, f0, recs = oracle.run("her", t, init, max_outer_iters=200, observer=obs)
    assert sum(seen) == sum(r["restarted"] for r in recs) and len(seen) == 200
    prev = f0
    for r in recs:
        if not r["restarted"]:
            assert r["f"] <= prev + 1e-12 * f0
            prev = r["f"]


def test_one_ao_iteration_is_n_block_solves(oracle):
    """test_ao.cpp:56-81 (bitwise)."""
    t, _ = oracle.generate([5, 4, 3], 2, sigma=0.05, seed=11)
    init = oracle.random_init([5, 4, 3], 2, 23)
    got, _, recs = oracle.run("ao", t, init, max_outer_iters=1)
    manual = [a.copy() for a in init]
    grams = [oracle.gram(a) for a in manual]
    for i in range(3):
        g = oracle.hadamard_of_grams(grams, i)
        manual[i] = oracle.ahals_solve(g, oracle.mttkrp(t, manual, i), manual[i])
        grams[i] = oracle.gram(manual[i])
    for a, b in zip(got, manual):
        assert np.array_equal(a, b)
    assert recs[-1]["f"] == pytest.approx(oracle.ref_objective(t, manual), rel=1e-10)


def test_ao_monotone_and_exact_fits(oracle):
    """test_ao.cpp:35-54, :83-104."""
    t, _ = oracle.generate([2, 2, 2], 1, seed=3)
    _, _, recs = oracle.run("ao", t, oracle.random_init([2, 2, 2], 1, 17), max_outer_iters=50)
    assert recs[-1]["f"] <= 1e-12 * oracle.norm_sq(t)
    t, _ = oracle.generate([6, 5, 4], 3, sigma=0.1, seed=29)
    _, f0, recs = oracle.run("ao", t, oracle.random_init([6, 5, 4], 3, 31), max_outer_iters=50)
    prev = f0
    for r in recs:
        assert r["f"] <= prev + 1e-12 * f0
        prev = r["f"]


def test_her_beats_ao_noiseless(oracle):
    """test_her.cpp:181-204."""
    hf, af = [], []
    for s in range(5):
        t, _ = oracle.generate([15, 15, 15], 3, seed=200 + s)
        init = oracle.random_init([15, 15, 15], 3, 300 + s)
        af.append(oracle.run("ao", t, init, max_outer_iters=150)[2][-1]["f"])
        hf.append(oracle.run("her", t, init, max_outer_iters=150)[2][-1]["f"])
    assert sorted(hf)[2] < sorted(af)[2]


def test_identical_traces(oracle):
    t, _ = oracle.generate([6, 6, 6], 2, sigma=0.01, seed=83)
    init = oracle.random_init([6, 6, 6], 2, 89)
    a = oracle.run("her", t, init, max_outer_iters=40)[2]
    b = oracle.run("her", t, init, max_outer_iters=40)[2]
    assert [(r["f"], r["beta"], r["restarted"]) for r in a] == [(r["f"], r["beta"], r["restarted"]) for r in b]


def test_factor_error_invariances(oracle):
    """test_metrics.cpp:84-131: permutation + scaling invariance, joint optimum."""
    gen = np.random.default_rng(4)
    truth = [gen.random((d, 4)) for d in (5, 6, 7)]
    perm = [2, 0, 3, 1]
    est = [a[:, perm] * gen.uniform(0.5, 2.0, 4) for a in truth]
    assert oracle.factor_error(est, truth) < 1e-12
    for n in range(1, 6):
        cost = gen.random((n, n))
        mapping, total = oracle.hungarian(cost)
        best = min(sum(cost[i, p[i]] for i in range(n)) for p in itertools.permutations(range(n)))
        assert total == pytest.approx(best, rel=1e-12)
        assert sorted(mapping) == list(range(n))
