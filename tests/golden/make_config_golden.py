#!/usr/bin/env python
"""Writes tests/golden/config_*.npz: the oracle's 50-iteration HER-AHALS and
AO-AHALS runs at the BASELINE.json configs 2, 3 and 4 (TEST INFRASTRUCTURE).

The north star's correctness clause is stated at these configs: "over the
first 50 iterations, f_k within 1e-8 relative (FP64) with identical HER
restart decisions; final factor-fitting error e_k matching". The oracle
(oracle/, pinned by tests/test_oracle.py against every known answer the
reference ships) restates her.cpp:40-110, ao.cpp:17-52, nnls.cpp:15-49 and
metrics.cpp:79-111. Each fixture stores, per algorithm:

  f0, f_k (k = 1..50), restart flags and beta_k (HER), the
  final factors, and e_50 = factor_error(final, truth) (metrics.cpp:79-111).

The tensors themselves are NOT stored (216 MB - 800 MB): the host generator
(`ntf_generate`, bit-identical to datagen.cpp:13-80 and to the oracle, see
tests/test_host_api.py) regenerates them from the seed on the GPU box. A
sha-free fingerprint (||T||^2 and the first/last entries) is stored so a
drift of the generator is caught before the trace comparison.

Configs (BASELINE.json; seeds S = 101.. per SURVEY.md §8(d); init =
random_init(shape, r, stream_seed(S, 1))):
  c2: 300^3, r=20, FP64, sigma=0,    seed 102
  c3: 100^4, r=16, FP64, sigma=0.01, seed 103
  c4: 500^3, r=32, FP32, sigma=0.01, seed 104, collinear factors
      (A_i[:, j] = 0.5 s_i + 0.5 U_i[:, j]); generated in FP64, rounded to
      float, the oracle consumes the float values upcast.

Run: OMP_NUM_THREADS=<cores> python tests/golden/make_config_golden.py [c2 c3 c4]
(about 1-10 minutes per config on 8 cores; commit the .npz files).

`--ref` runs THE REFERENCE ITSELF instead of the oracle: oracle/_ref/
libntf_ref.so, the unmodified /root/reference/proj sources compiled by
oracle/ref_build/Makefile (Eigen stand-in; the reference's own unit suites
pass over that build), through oracle/pyref.py, and writes refrun_*.npz with
the same layout. Those are the reference-produced golden vectors the GPU
parity tests and tests/test_ref_build.py compare against. (The collinear c4
instance comes from this repo's generator -- the rule is SURVEY 8(d)'s, not a
reference option -- and is handed to the reference as data.)
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as ora  # noqa: E402

REF = "--ref" in sys.argv
if REF:
    import pyref as run_impl  # noqa: E402
else:
    run_impl = ora

ITERS = 50
CONFIGS = {
    # name: (shape, rank, sigma, dtype, seed, collinear)
    "c2": ([300, 300, 300], 20, 0.0, "f64", 102, False),
    "c3": ([100, 100, 100, 100], 16, 0.01, "f64", 103, False),
    "c4": ([500, 500, 500], 32, 0.01, "f32", 104, True),
}


def make(name):
    shape, rank, sigma, dt, seed, collinear = CONFIGS[name]
    t0 = time.time()
    t, truth = ora.generate(shape, rank, sigma=sigma, seed=seed, collinear=collinear)
    if dt == "f32":
        t = t.astype(np.float32)
    init = ora.random_init(shape, rank, ora.stream_seed(seed, 1))
    flat = t.reshape(-1)
    out = {"shape": np.array(shape), "rank": np.array(rank), "sigma": np.array(sigma),
           "seed": np.array(seed), "dtype": np.array(dt), "collinear": np.array(collinear),
           "iters": np.array(ITERS), "norm_sq": np.array(run_impl.norm_sq(t)),
           "t_head": np.array(flat[:64], np.float64), "t_tail": np.array(flat[-64:], np.float64)}
    for algo in ("her", "ao"):
        fac, f0, recs = run_impl.run(algo, t, init, max_outer_iters=ITERS)
        out[f"{algo}_f0"] = np.array(f0)
        out[f"{algo}_f"] = np.array([r["f"] for r in recs])
        if algo == "her":
            out["her_restarted"] = np.array([bool(r["restarted"]) for r in recs])
            out["her_beta"] = np.array([r["beta"] for r in recs])
        for i, a in enumerate(fac):
            out[f"{algo}_final{i}"] = a
        out[f"{algo}_e"] = np.array(run_impl.factor_error(fac, truth))
        print(f"{name} {algo}: f0={f0:.6e} f50={recs[-1]['f']:.6e} e50={float(out[f'{algo}_e']):.6e}",
              flush=True)
    path = os.path.join(HERE, f"{'refrun' if REF else 'config'}_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{path}: {os.path.getsize(path)} bytes, {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    for name in ([a for a in sys.argv[1:] if not a.startswith("--")] or list(CONFIGS)):
        make(name)
