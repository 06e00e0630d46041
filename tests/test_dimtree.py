"""Dimension-tree MTTKRP reuse (NTF_RUN_DIMTREE).

With split h, blocks 0..h-1 of an outer iteration contract
Y_L = T x_h A_h .. x_{N-1} A_{N-1} and blocks h..N-1 contract
Y_R = T x_0 A_0 .. x_{h-1} A_{h-1} instead of the tensor (default h = N-1
for 3-way, h = N/2 from 4-way; NTF_TREE_SPLIT overrides). Results differ
from the direct MTTKRPs only by summation order,
so the traces must meet the same parity bars against the oracle
(parity.compare_traces: f_k within 1e-8 relative + the cancellation floor,
identical restart decisions), for HER and AO, 3-way and 4-way.
"""
import numpy as np
import pytest

from parity import compare_traces, rel_fro

pytestmark = pytest.mark.gpu


def _instance(P, shape, rank, sigma, seed):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, seed=seed)
    t, truth = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(seed, 1))
    return t, truth, init


CASES = [([50, 50, 50], 10, 0.01, 101), ([40, 36, 32], 8, 0.0, 11), ([20, 18, 16, 16], 6, 0.01, 103),
         ([64, 40, 48], 20, 0.001, 5), ([24, 20, 18, 16], 16, 0.01, 9)]


@pytest.mark.parametrize("shape,rank,sigma,seed", CASES)
def test_dimtree_her_trace_parity(P, oracle, shape, rank, sigma, seed):
    t, truth, init = _instance(P, shape, rank, sigma, seed)
    cfg = P.AoConfig(max_outer_iters=50, flags=P.RUN_DIMTREE)
    model, trace = P.her_run(t, init, cfg, P.HerParams())
    fo, f0, recs = oracle.run("her", np.asarray(t), init.factors, max_outer_iters=50)
    stats = compare_traces(trace, f0, recs, oracle.norm_sq(np.asarray(t)))
    assert stats["checked"] == 50
    assert model.is_nonnegative()


@pytest.mark.parametrize("split", [1, 2, 3])
@pytest.mark.parametrize("shape,rank,sigma,seed", [([20, 18, 16, 16], 6, 0.01, 103), ([64, 40, 48], 20, 0.001, 5)])
def test_dimtree_every_split_her_parity(P, oracle, monkeypatch, shape, rank, sigma, seed, split):
    """Every split point h of the tree (Y_L with merged rows and shifted
    factors, Y_R with factor-offset tree contractions) meets the trace bars."""
    if split >= len(shape):
        pytest.skip("split must be < N")
    monkeypatch.setenv("NTF_TREE_SPLIT", str(split))
    t, truth, init = _instance(P, shape, rank, sigma, seed)
    prov = P.GpuDenseProvider(t)
    model, trace = P.her_run(prov, init, P.AoConfig(max_outer_iters=30, flags=P.RUN_DIMTREE), P.HerParams())
    fo, f0, recs = oracle.run("her", np.asarray(t), init.factors, max_outer_iters=30)
    stats = compare_traces(trace, f0, recs, oracle.norm_sq(np.asarray(t)))
    assert stats["checked"] == 30
    prov.close()


@pytest.mark.parametrize("shape,rank,sigma,seed", CASES[:3])
def test_dimtree_ao_trace_parity(P, oracle, shape, rank, sigma, seed):
    t, truth, init = _instance(P, shape, rank, sigma, seed)
    cfg = P.AoConfig(max_outer_iters=50, flags=P.RUN_DIMTREE)
    model, trace = P.ao_run(t, init, cfg)
    fo, f0, recs = oracle.run("ao", np.asarray(t), init.factors, max_outer_iters=50)
    compare_traces(trace, f0, recs, oracle.norm_sq(np.asarray(t)), check_restarts=False)
    for a, b in zip(model, fo):
        assert rel_fro(a, b) < 1e-6


@pytest.mark.parametrize("shape,rank", [([300, 300, 300], 20), ([100, 100, 100, 100], 16)], ids=["C2", "C3"])
def test_dimtree_matches_direct_at_full_size(P, shape, rank):
    t, truth, init = _instance(P, shape, rank, 0.01, 102)
    prov = P.GpuDenseProvider(t)
    _, direct = P.her_run(prov, init, P.AoConfig(max_outer_iters=8, flags=P.RUN_DIRECT), P.HerParams())
    _, tree = P.her_run(prov, init, P.AoConfig(max_outer_iters=8, flags=P.RUN_DIMTREE), P.HerParams())
    assert abs(direct.f0 - tree.f0) <= 1e-14 * abs(direct.f0)
    for a, b in zip(direct.records, tree.records):
        assert abs(a.f - b.f) <= 1e-10 * abs(a.f) + 64 * 2.0 ** -52 * prov.norm_sq()
        assert a.restarted == b.restarted
    prov.close()


@pytest.mark.parametrize("shape,rank", [([64, 48, 40], 32), ([40, 36, 34, 32], 8)], ids=["3way", "4way-split"])
def test_dimtree_f32_ao_trace(P, oracle, shape, rank):
    """FP32 tensors through the dimension tree (the path BASELINE configs 4/5
    run: FP32 partial passes with FP64 partials, FP64 tree contractions):
    AO traces match the oracle on the float values upcast (ao.cpp:17-52) and
    the direct GPU path to 1e-6 ||T||^2 (r01h: tree vs oracle <= 3.2e-8,
    direct vs tree <= 1.6e-7: the FP32 factor mirrors bound it)."""
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=21)
    t, _ = P.generate(spec, dtype=np.float32)
    init = P.random_init(shape, rank, P.stream_seed(21, 1))
    prov = P.GpuDenseProvider(t)
    nsq = prov.norm_sq()
    _, tree = P.ao_run(prov, init, P.AoConfig(max_outer_iters=20, flags=P.RUN_DIMTREE))
    _, direct = P.ao_run(prov, init, P.AoConfig(max_outer_iters=20, flags=P.RUN_DIRECT))
    t64 = np.asarray(t, dtype=np.float64)
    _, f0, recs = oracle.run("ao", t64, init.factors, max_outer_iters=20)
    dev_o = max(abs(a.f - w["f"]) for a, w in zip(tree.records, recs)) / nsq
    dev_d = max(abs(a.f - b.f) for a, b in zip(tree.records, direct.records)) / nsq
    print(f"f0 dev {abs(tree.f0 - f0) / nsq:.2e}, trace dev vs oracle {dev_o:.2e}, vs direct {dev_d:.2e}")
    assert abs(tree.f0 - f0) <= 1e-6 * nsq
    assert len(tree.records) == len(recs) == 20
    assert dev_o <= 1e-6 and dev_d <= 1e-6
    assert dev_d > 0.0  # the tree path really ran (different summation order)
    prov.close()
