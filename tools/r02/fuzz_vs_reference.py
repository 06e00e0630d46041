"""Randomised parity sweep of the GPU drivers against the reference build (QA,
run on the GPU box): random orders, shapes, ranks, noise levels, HER and AO,
every case through tests/parity.compare_traces. usage: fuzz_vs_reference.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import paper_2001_04321_b200 as P  # noqa: E402
import pyref as R  # noqa: E402
from parity import compare_traces, rel_fro  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
gen = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
for case in range(cases):
    order = int(gen.integers(2, 5))
    hi = {2: 90, 3: 40, 4: 14}[order]
    shape = [int(gen.integers(2, hi)) for _ in range(order)]
    rank = int(gen.choice([1, 2, 3, 4, 5, 7, 8, 10, 12, 16, 20, 24, 32, 33, 48, 64]))
    sigma = float(gen.choice([0.0, 0.001, 0.01, 0.1]))
    ill = bool(gen.integers(0, 4) == 0) and rank >= 2
    seed = int(gen.integers(1, 10 ** 6))
    algo = "her" if gen.integers(0, 3) else "ao"
    iters = 15
    try:
        spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, seed=seed, ill_conditioned=ill)
        t, truth = P.generate(spec)
        init = P.random_init(shape, rank, P.stream_seed(seed, 1))
        fr, f0, recs = R.run(algo, np.asarray(t), init.factors, max_outer_iters=iters)
        cfg = P.AoConfig(max_outer_iters=iters)
        model, trace = P.her_run(t, init, cfg, P.HerParams()) if algo == "her" else P.ao_run(t, init, cfg)
        compare_traces(trace, f0, recs, R.norm_sq(np.asarray(t)), n_check=iters, check_restarts=(algo == "her"))
        worst = max(rel_fro(a, b) for a, b in zip(model, fr))
        assert worst < 1e-5, worst
    except Exception as exc:  # report and go on
        bad += 1
        print(f"FAIL case {case}: {algo} shape={shape} r={rank} sigma={sigma} ill={ill} seed={seed}: "
              f"{type(exc).__name__}: {str(exc)[:200]}", flush=True)
print(f"{cases} cases, {bad} failures")
