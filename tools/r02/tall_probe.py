import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2001_04321_b200 as P
for shape, rank in (([10000, 100, 100], 16), ([20000, 64, 48], 20)):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=5)
    t, truth = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(5, 1))
    prov = P.GpuDenseProvider(t)
    P.her_run(prov, init, P.AoConfig(max_outer_iters=5), P.HerParams())
    model, trace = P.her_run(prov, init, P.AoConfig(max_outer_iters=50), P.HerParams())
    dt = trace.records[-1].time_s
    print(f"{shape} r={rank}: 50 HER iterations in {dt*1e3:.1f} ms of run clock = {50/dt:.0f} iters/s; f0 {trace.f0:.4e} -> f50 {trace.final_f():.4e}, "
          f"restarts {trace.restart_count()}, e50 {P.factor_error(model, truth):.3e}")
    prov.close()
