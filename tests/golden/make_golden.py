#!/usr/bin/env python
"""Writes the golden fixtures under tests/golden/ from the CPU oracle.

The reference itself cannot be built in this image (Eigen3, doctest and CLI11
are absent), so the fixtures are produced by the oracle
restatement in oracle/ after it has been pinned against every known-answer
test the reference ships (tests/test_oracle.py: the mt19937_64 10,000th draw,
the noiseless factorisation identity, rank-one MTTKRP, the HALS column
formula, the update_betas arithmetic, ...). They freeze small end-to-end
cases so any later change of the oracle or of the CUDA path that moves a
number is caught:

  * instance generation (datagen.cpp:13-80) for a 3-way and a 4-way shape;
  * every mode's MTTKRP at the truth factors and at the init (kernels.cpp:161-191);
  * 30 HER-AHALS and 30 AO-AHALS outer iterations from the seeded init
    (her.cpp:40-110, ao.cpp:17-52): f0, f_k, restart flags, beta_k, final factors.

Run: python tests/golden/make_golden.py   (rewrites *.npz; commit them)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as ora  # noqa: E402

CASES = {
    # name: (shape, rank, sigma, seed, iterations)
    "her3_8x7x6_r3": ([8, 7, 6], 3, 0.05, 7, 30),
    "her4_6x5x4x3_r2": ([6, 5, 4, 3], 2, 0.01, 404, 30),
    "her3_20x16x12_r5_noiseless": ([20, 16, 12], 5, 0.0, 4000, 30),
}


def make(name, shape, rank, sigma, seed, iters):
    t, truth = ora.generate(shape, rank, sigma=sigma, seed=seed)
    init = ora.random_init(shape, rank, ora.stream_seed(seed, 1))
    out = {"tensor": t, "shape": np.array(shape), "rank": np.array(rank), "sigma": np.array(sigma),
           "seed": np.array(seed)}
    for i, a in enumerate(truth):
        out[f"truth{i}"] = a
    for i, a in enumerate(init):
        out[f"init{i}"] = a
    for mode in range(len(shape)):
        out[f"mttkrp_truth{mode}"] = ora.mttkrp(t, truth, mode)
        out[f"mttkrp_init{mode}"] = ora.mttkrp(t, init, mode)
    out["norm_sq"] = np.array(ora.norm_sq(t))
    for algo in ("her", "ao"):
        fac, f0, recs = ora.run(algo, t, init, max_outer_iters=iters)
        out[f"{algo}_f0"] = np.array(f0)
        out[f"{algo}_f"] = np.array([r["f"] for r in recs])
        if algo == "her":
            out["her_restarted"] = np.array([bool(r["restarted"]) for r in recs])
            out["her_beta"] = np.array([r["beta"] for r in recs])
        for i, a in enumerate(fac):
            out[f"{algo}_final{i}"] = a
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{path}: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    for name, args in CASES.items():
        make(name, *args)
