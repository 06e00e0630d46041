"""Probe: the fast MTTKRP on a 2-way (L x I) view = the TTM T x_N A_N (diagnostics)."""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2001_04321_b200 as P  # noqa: E402

L, I, r = 90000, 300, 20
gen = np.random.default_rng(1)
t = gen.random((L, I))
a0 = gen.random((L, r))
a1 = gen.random((I, r))
prov = P.GpuDenseProvider(t)
print(prov.mttkrp_plan(r, 0))
got = prov.mttkrp([a0, a1], 0)
want = t @ a1
print("rel err", np.linalg.norm(got - want) / np.linalg.norm(want))
