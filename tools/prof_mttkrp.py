"""Per-call fast-MTTKRP pipeline counters (diagnostics): run with a library
built with -DNTF_FAST_PROFILE=1 (NTF_B200_LIB) and NTF_FAST_PROF=1; the
launcher prints producer/consumer wait cycles and epilogue phases per call.
usage: python tools/prof_mttkrp.py c2|c3 [calls]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04321_b200 as P  # noqa: E402

cfgs = {"c2": ([300, 300, 300], 20, 0.0, 102), "c3": ([100, 100, 100, 100], 16, 0.01, 103)}
shape, rank, sigma, seed = cfgs[sys.argv[1]]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t, _ = P.generate(P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, seed=seed))
init = P.random_init(shape, rank, P.stream_seed(seed, 1))
prov = P.GpuDenseProvider(t)
for mode in range(len(shape)):
    for _ in range(calls):
        prov.mttkrp(init, mode)
    print(f"mode {mode} done", file=sys.stderr, flush=True)
prov.close()
