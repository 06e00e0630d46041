"""BASELINE config 4 as specified: the ill-conditioned (collinear) 500^3,
r = 32, FP32 instance, HER-AHALS vs AO-AHALS for 1000 outer iterations on
the production path (the reference pattern: tests/acceptance.cpp:271-293,
HER/AO final-f comparison). Prints one JSON object: per algorithm the
device-timed iterations/s, f at checkpoints, restarts, final f / ||T||^2 and
the factor-fitting error e (metrics.cpp:79-111) of the final model.
usage: python tools/r02/c4_her_vs_ao.py [iters] > profiles/r02/c4_her_vs_ao.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2001_04321_b200 as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
t, truth, init = bench.make_instance(P, "c4")
prov = P.GpuDenseProvider(t)
nsq = prov.norm_sq()
out = {"config": bench.workload_config("c4", "her")["workload"].replace(" HER-AHALS", ""), "iterations": iters,
       "norm_sq": nsq}
for algo in ("her", "ao"):
    sess = P.Session(prov, init, P.AoConfig(max_outer_iters=iters), P.HerParams(), algo=algo)
    t0 = time.perf_counter()
    sess.step(iters)
    sess.sync()
    wall = time.perf_counter() - t0
    tr = sess.trace()
    model = sess.factors() if hasattr(sess, "factors") else None
    recs = tr.records
    cps = [k for k in (1, 10, 50, 100, 200, 500, 1000, iters) if k <= len(recs)]
    res = {"iters_per_s_device": len(recs) / recs[-1].time_s, "wall_s": wall, "f0": tr.f0,
           "f_at": {str(k): recs[k - 1].f for k in sorted(set(cps))}, "final_f_over_nsq": recs[-1].f / nsq,
           "restarts": tr.restart_count() if algo == "her" else None}
    if model is not None:
        res["factor_error"] = P.factor_error(model, truth)
    out[algo] = res
    sess.close()
out["her_over_ao_final_f"] = out["her"]["f_at"][str(iters)] / out["ao"]["f_at"][str(iters)]
print(json.dumps(out))
