"""Conditioning of the 50-iteration traces at the BASELINE configs, two
experiments against the committed fixture (the oracle in the reference's
summation order):
  ulp:   the oracle from an init perturbed by one ulp (relative 2^-52 on a
         random half of the entries);
  order: the oracle with every MTTKRP summed in descending order (the same
         algorithm rounded differently, as any other correct implementation
         -- the GPU kernels included -- rounds differently).
Both show how far two faithful FP64 runs drift apart by iteration k, i.e.
the floor a trace-parity bar can be set at. TEST INFRASTRUCTURE (oracle only)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")]
import pyoracle as O  # noqa: E402
from make_config_golden import CONFIGS  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c2"]:
    shape, rank, sigma, dt, seed, collinear = CONFIGS[name]
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"config_{name}.npz")))
    t, truth = O.generate(shape, rank, sigma=sigma, seed=seed, collinear=collinear)
    if dt == "f32":
        t = t.astype(np.float32)
    init = O.random_init(shape, rank, O.stream_seed(seed, 1))
    rng = np.random.default_rng(1)
    pert = [a * np.where(rng.random(a.shape) < 0.5, 1.0 + 2.0 ** -52, 1.0) for a in init]
    nsq = O.norm_sq(t)
    exps = [("ulp", "her"), ("ulp", "ao"), ("order", "her"), ("order", "ao")]
    if dt == "f32":  # FP32 factor mirrors: Khatri-Rao rows rounded to float
        exps += [("f32kr", "her"), ("f32kr", "ao")]
    for exp, algo in exps:
        O.set_sum_order({"order": 1, "f32kr": 2}.get(exp, 0))
        fac_p, f0, recs = O.run(algo, t, pert if exp == "ulp" else init, max_outer_iters=50)
        O.set_sum_order(0)
        f = np.array([r["f"] for r in recs])
        ref = g[f"{algo}_f"]
        rel = np.abs(f - ref) / np.abs(ref)
        absn = np.abs(f - ref) / nsq
        res = {"e_rel": abs(O.factor_error(fac_p, truth) - float(g[f"{algo}_e"])) / float(g[f"{algo}_e"]), "f0_rel": abs(f0 - float(g[f"{algo}_f0"])) / abs(float(g[f"{algo}_f0"])), "max_rel": float(rel.max()), "argmax": int(rel.argmax()) + 1, "max_abs_over_nsq": float(absn.max()),
               "rel_at": {k: float(rel[k - 1]) for k in (1, 5, 10, 20, 30, 40, 50)}}
        if algo == "her":
            res["restart_flips"] = int(sum(bool(r["restarted"]) != bool(x) for r, x in zip(recs, g["her_restarted"])))
        out[f"{name}_{exp}_{algo}"] = res
        print(name, exp, algo, json.dumps(res), flush=True)
