"""Print the MTTKRP kernel plan per mode for the BASELINE configs (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04321_b200 as P

for name, shape, r, dt in [("c1", [50, 50, 50], 10, np.float64), ("c2", [300, 300, 300], 20, np.float64),
                           ("c3", [100, 100, 100, 100], 16, np.float64), ("c4", [500, 500, 500], 32, np.float32)]:
    t = np.zeros(shape, dtype=dt)
    p = P.GpuDenseProvider(t)
    for m in range(len(shape)):
        print(name, m, p.mttkrp_plan(r, m))
    p.close()
