"""The two API paths the bench line does not time (diagnostics, C2 instance):
  * per-call provider MTTKRP (a reference-side
    her_run calling GpuDenseProvider::mttkrp once per block) -- seconds per
    call and mode, host factors in, host result out;
  * the time-budget driver (AoConfig.max_time_s: one host synchronisation per
    outer iteration instead of graph replay) -- iterations/s it sustains.
usage: python tools/r02/paths_probe.py > profiles/r02/paths_probe_<tag>.json"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2001_04321_b200 as P  # noqa: E402

shape, rank = [300, 300, 300], 20
spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.0, seed=102)
t, truth = P.generate(spec)
init = P.random_init(shape, rank, P.stream_seed(102, 1))
prov = P.GpuDenseProvider(t)
out = {"config": "BASELINE config 2: 300x300x300 r=20 f64"}
per_mode = []
for mode in range(3):
    for _ in range(5):
        prov.mttkrp(init, mode)
    ts = []
    for _ in range(50):
        a = time.perf_counter()
        prov.mttkrp(init, mode)
        ts.append(time.perf_counter() - a)
    per_mode.append({"mode": mode, "median_us": 1e6 * float(np.median(ts)), "best_us": 1e6 * min(ts)})
out["per_call_mttkrp"] = per_mode
a = time.perf_counter()
for _ in range(20):
    prov.mttkrp_all(init) if hasattr(prov, "mttkrp_all") else [prov.mttkrp(init, m) for m in range(3)]
out["mttkrp_all_us"] = 1e6 * (time.perf_counter() - a) / 20
for budget in (0.05, 0.2):
    P.her_run(prov, init, P.AoConfig(max_time_s=budget), P.HerParams())  # warm
    a = time.perf_counter()
    model, trace = P.her_run(prov, init, P.AoConfig(max_time_s=budget), P.HerParams())
    wall = time.perf_counter() - a
    out[f"time_budget_{budget}"] = {"iterations": len(trace.records), "run_clock_s": trace.records[-1].time_s,
                                    "iters_per_s": len(trace.records) / trace.records[-1].time_s, "wall_s": wall}
a = time.perf_counter()
model, trace = P.her_run(prov, init, P.AoConfig(max_outer_iters=200), P.HerParams())
out["iteration_budget_200"] = {"iters_per_s_run_clock": 200 / trace.records[-1].time_s, "wall_s": time.perf_counter() - a}
seen = []
a = time.perf_counter()
P.her_run(prov, init, P.AoConfig(max_outer_iters=200), P.HerParams(), observer=lambda info: seen.append(info.iter))
out["observer_200"] = {"wall_s": time.perf_counter() - a, "callbacks": len(seen)}
prov.close()
print(json.dumps(out, indent=1))
