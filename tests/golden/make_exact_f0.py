"""Writes tests/golden/config_f0_exact.json: f0 (the pivot objective at the
init, driver_common.hpp:50-56 / kernels.cpp:298-311) of the BASELINE configs
in extended precision (numpy longdouble, 64-bit mantissa, on the same
instance and init as tests/golden/config_*.npz). It is the yardstick for how
close the oracle's and the GPU's FP64 values each are to the exact value: the
reference's sequential sums carry ~1e-12 relative error at these sizes.
TEST INFRASTRUCTURE. Run: python tests/golden/make_exact_f0.py [c2 c3 c4]"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [os.path.join(ROOT, "oracle"), HERE]
import pyoracle as O  # noqa: E402
from make_config_golden import CONFIGS  # noqa: E402

LD = np.longdouble
path = os.path.join(HERE, "config_f0_exact.json")
table = json.load(open(path)) if os.path.exists(path) else {}
for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    shape, rank, sigma, dt, seed, collinear = CONFIGS[name]
    t, _ = O.generate(shape, rank, sigma=sigma, seed=seed, collinear=collinear)
    if dt == "f32":
        t = t.astype(np.float32)
    init = O.random_init(shape, rank, O.stream_seed(seed, 1))
    n = len(shape)
    p = n - 1
    # C = T_(p) KR(A_0..A_{p-1}) with the last listed mode fastest (kernels.cpp:90-113)
    w = np.ones((1, rank), LD)
    for a in init[:p]:
        w = (w[:, None, :] * a.astype(LD)[None, :, :]).reshape(-1, rank)
    tm = t.reshape(-1, shape[p])
    c = np.zeros((shape[p], rank), LD)
    step = 1 << 16
    for b in range(0, tm.shape[0], step):
        blk = tm[b:b + step].astype(LD)
        c += blk.T @ w[b:b + step]
    nsq = np.sum(t.reshape(-1).astype(LD) ** 2)
    a = init[p].astype(LD)
    g = np.ones((rank, rank), LD)
    for j in range(p):
        aj = init[j].astype(LD)
        g *= aj.T @ aj
    f0 = 0.5 * nsq - np.sum(a * c) + 0.5 * np.sum((a.T @ a) * g)
    fx = dict(np.load(os.path.join(ROOT, "tests", "golden", f"config_{name}.npz")))
    ora = float(fx["her_f0"])
    terms = float(0.5 * nsq + abs(np.sum(a * c)) + 0.5 * np.sum((a.T @ a) * g))
    print(f"{name}: f0 exact {float(f0)!r} (|terms| {terms:.6e}); oracle {ora!r} rel err "
          f"{abs(ora - float(f0)) / float(f0):.2e}", flush=True)
    table[name] = {"f0_exact": float(f0), "terms": terms, "oracle_f0": ora,
                   "oracle_rel_err": abs(ora - float(f0)) / float(f0)}
    with open(path, "w") as fh:
        json.dump(table, fh, indent=1)
