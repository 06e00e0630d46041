"""Repeated MTTKRP calls on a BASELINE config for ncu captures (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04321_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shapes = {"c2": ([300, 300, 300], 20, np.float64), "c3": ([100, 100, 100, 100], 16, np.float64),
          "c4": ([500, 500, 500], 32, np.float32)}
shape, r, dt = shapes[cfg]
gen = np.random.default_rng(0)
t = gen.random(shape).astype(dt)
m = [gen.random((d, r)) for d in shape]
p = P.GpuDenseProvider(t)
for mode in range(len(shape)):
    print(mode, p.mttkrp_plan(r, mode))
    for _ in range(reps):
        p.mttkrp(m, mode)
print("ok")
