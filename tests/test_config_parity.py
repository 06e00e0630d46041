"""Parity at the BASELINE.json configs through the production path.

The north star's correctness clause: "over the first 50 iterations, f_k
within 1e-8 relative (FP64) with identical HER restart decisions; final
factor-fitting error e_k matching" -- checked here at config 2 (300^3, r=20,
FP64, sigma=0), config 3 (100^4, r=16, FP64, sigma=0.01) and the collinear
config 4 (500^3, r=32, FP32, sigma=0.01), for HER-AHALS (her.cpp:40-110)
and AO-AHALS (ao.cpp:17-52), with the default (production) flags: dimension
tree, CUDA-graph replay, the 16-CTA stream NNLS. The oracle's runs are the
committed fixtures tests/golden/config_*.npz (tests/golden/
make_config_golden.py); the instances are regenerated here by the host
generator, which is bit-identical to the oracle's (test_host_api.py), and
their fingerprint (||T||^2, first/last entries) is checked first.

Bars:
  * FP64 (c2, c3): |f_k - f_k^ora| <= 1e-8 |f_k^ora| + 64 eps ||T||^2
    (tests/parity.py: the cancellation floor of the cheap objective),
    identical restart decisions wherever |F_k - F_{k-1}| exceeds that floor,
    beta_k to 1e-12; final factors 1e-6 relative Frobenius; e_50 (metrics.cpp:
    79-111) within 1e-6 relative.
  * FP32 (c4): the kernels multiply in FP32 (per-call MTTKRP bar 1e-5), so
    f_k carries FP32 rounding of <A, C> ~ 1e-7 ||T||^2: |f_k - f_k^ora| <=
    1e-6 ||T||^2, restart decisions identical wherever |F_k - F_{k-1}| > 4e-6
    ||T||^2 (beyond the combined error of two evaluations), e_50 within 1e-2
    relative.
"""
import os

import numpy as np
import pytest

from parity import F_FLOOR, rel_fro

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS = ["c2", "c3", "c4"]


def _fixture(name):
    path = os.path.join(HERE, "golden", f"config_{name}.npz")
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture(scope="module")
def instances(P):
    cache = {}

    def get(name):
        if name not in cache:
            cache.clear()  # one full-size instance at a time (host memory)
            g = _fixture(name)
            shape = [int(x) for x in g["shape"]]
            spec = P.SyntheticSpec(shape=shape, rank=int(g["rank"]), noise_sigma=float(g["sigma"]),
                                   seed=int(g["seed"]), collinear=bool(g["collinear"]))
            dtype = np.float32 if str(g["dtype"]) == "f32" else np.float64
            t, truth = P.generate(spec, dtype=dtype)
            init = P.random_init(shape, spec.rank, P.stream_seed(spec.seed, 1))
            cache[name] = (g, t, truth, init)
        return cache[name]
    return get


def test_config_fixtures_cover_the_north_star_configs():
    for name in CONFIGS:
        g = _fixture(name)
        assert int(g["iters"]) == 50
        assert len(g["her_f"]) == 50 and len(g["ao_f"]) == 50
        assert g["her_restarted"].dtype == bool
        assert np.all(np.diff(g["ao_f"]) <= 1e-12 * float(g["ao_f0"]))  # AO is monotone (test_ao.cpp:83-104)
    assert bool(_fixture("c4")["collinear"]) and str(_fixture("c4")["dtype"]) == "f32"


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["her", "ao"])
@pytest.mark.parametrize("name", CONFIGS)
def test_config_trace_parity(P, instances, name, algo):
    g, t, truth, init = instances(name)
    flat = t.reshape(-1)
    assert np.array_equal(np.asarray(flat[:64], np.float64), g["t_head"])
    assert np.array_equal(np.asarray(flat[-64:], np.float64), g["t_tail"])
    prov = P.GpuDenseProvider(t)
    nsq = prov.norm_sq()
    # ||T||^2 sums |T| positive squares in FP64 in another order: 4 sqrt(|T|) eps relative
    assert abs(nsq - float(g["norm_sq"])) <= 4 * np.sqrt(t.size) * 2.0 ** -52 * float(g["norm_sq"])
    cfg = P.AoConfig(max_outer_iters=50)  # production defaults: dimension tree, graph replay
    if algo == "her":
        model, trace = P.her_run(prov, init, cfg, P.HerParams())
    else:
        model, trace = P.ao_run(prov, init, cfg)
    prov.close()
    f0o = float(g[f"{algo}_f0"])
    fo = g[f"{algo}_f"]
    fp32 = str(g["dtype"]) == "f32"
    assert len(trace.records) == 50
    if fp32:
        bar = lambda ref: 1e-6 * nsq  # noqa: E731
        decision_floor = 4e-6 * nsq
    else:
        bar = lambda ref: 1e-8 * abs(ref) + F_FLOOR * nsq  # noqa: E731
        decision_floor = 4 * F_FLOOR * nsq
    assert abs(trace.f0 - f0o) <= (1e-6 * nsq if fp32 else 1e-12 * abs(f0o) + F_FLOOR * nsq), (trace.f0, f0o)
    worst = 0.0
    decided = 0
    prev = f0o
    for k, rec in enumerate(trace.records):
        assert rec.iter == k + 1
        dev = abs(rec.f - fo[k])
        worst = max(worst, dev / abs(fo[k]))
        assert dev <= bar(fo[k]), f"{name} {algo} iter {k + 1}: gpu {rec.f!r} oracle {fo[k]!r}"
        if algo == "her" and abs(fo[k] - prev) > decision_floor:
            decided += 1
            assert rec.restarted == bool(g["her_restarted"][k]), f"{name} iter {k + 1}: restart decision differs"
            if not fp32:
                assert abs(rec.beta - g["her_beta"][k]) <= 1e-12 * abs(g["her_beta"][k])
        prev = fo[k]
    if algo == "her":
        assert decided >= 40, decided  # the decisions really were compared
    finals = [g[f"{algo}_final{i}"] for i in range(len(init.factors))]
    if not fp32:
        for a, b in zip(model, finals):
            assert rel_fro(a, b) < 1e-6
    e_gpu = P.factor_error(model, truth)
    e_ora = float(g[f"{algo}_e"])
    assert abs(e_gpu - e_ora) <= (1e-2 if fp32 else 1e-6) * e_ora, (e_gpu, e_ora)
    print(f"{name} {algo}: worst rel f dev {worst:.2e}, decisions compared {decided}, e {e_gpu:.6e} vs {e_ora:.6e}")
