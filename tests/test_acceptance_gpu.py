"""The reference's end-to-end acceptance criteria for the HER-AHALS path
(tests/acceptance.cpp), run through the GPU drivers with the same instances
(generator seeds, init seeds, budgets) and the same thresholds:

  * criterion_ao_monotone (acceptance.cpp:223-248), AHALS row: AO's f never
    rises by more than 1e-12 f0 over 200 iterations (10x9x8, r=3, sigma=0.1);
  * criterion_exact_recovery (:250-269): median over 10 seeds of
    f/||T||^2 after 500 HER-AHALS iterations at 30^3, r=5 (noiseless) <= 1e-10;
  * criterion_her_acceleration (:271-293): median final f of HER over median
    final f of AO, 20 seeds at 50^3, r=10, 200 iterations, shared init <= 1e-2
    (the reference expects order 1e-4).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_ao_monotone(P):
    worst = -1e300
    for seed in range(5):
        spec = P.SyntheticSpec(shape=[10, 9, 8], rank=3, noise_sigma=0.1, seed=2000 + seed)
        t, _ = P.generate(spec)
        _, trace = P.ao_run(t, P.random_init(spec.shape, 3, 3000 + seed), P.AoConfig(max_outer_iters=200))
        prev = trace.f0
        for rec in trace.records:
            worst = max(worst, (rec.f - prev) / trace.f0)
            prev = rec.f
    assert worst <= 1e-12, worst


def test_exact_recovery(P):
    ratios = []
    for seed in range(10):
        spec = P.SyntheticSpec(shape=[30, 30, 30], rank=5, seed=4000 + seed)
        t, _ = P.generate(spec)
        prov = P.GpuDenseProvider(t)
        _, trace = P.her_run(prov, P.random_init(spec.shape, 5, 5000 + seed), P.AoConfig(max_outer_iters=500),
                             P.HerParams())
        ratios.append(trace.final_f() / prov.norm_sq())
        prov.close()
    med = float(np.median(ratios))
    print(f"median f/||T||^2 = {med:.2e} (tol 1e-10)")
    assert med <= 1e-10, med


def test_her_acceleration(P):
    ao_final, her_final = [], []
    for seed in range(20):
        spec = P.SyntheticSpec(shape=[50, 50, 50], rank=10, seed=6000 + seed)
        t, _ = P.generate(spec)
        prov = P.GpuDenseProvider(t)
        init = P.random_init(spec.shape, 10, 7000 + seed)  # shared
        cfg = P.AoConfig(max_outer_iters=200)
        ao_final.append(P.ao_run(prov, init, cfg)[1].final_f())
        her_final.append(P.her_run(prov, init, cfg, P.HerParams())[1].final_f())
        prov.close()
    ratio = float(np.median(her_final) / np.median(ao_final))
    print(f"median-f ratio her/plain = {ratio:.2e} (tol 1e-2, expected order 1e-4)")
    assert ratio <= 1e-2, ratio
