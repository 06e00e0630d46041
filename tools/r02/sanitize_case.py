"""Small production-path runs for compute-sanitizer (memcheck / racecheck /
synccheck): a tree HER solve on the fast kernels (TMA/DMMA MTTKRP with the
in-kernel split-K grid barrier, tree contractions on clusters, the stream
NNLS with st.async cluster traffic), a 4-way split-tree AO solve, an FP32
instance and a standalone AHALS solve; each checked against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import paper_2001_04321_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402
from parity import compare_traces  # noqa: E402

iters = int(os.environ.get("SAN_ITERS", "4"))
for shape, rank, algo, dt in (([64, 48, 40], 20, "her", np.float64), ([24, 22, 20, 18], 8, "ao", np.float64),
                              ([64, 48, 40], 32, "her", np.float32)):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=3)
    t, _ = P.generate(spec, dtype=dt)
    init = P.random_init(shape, rank, P.stream_seed(3, 1))
    prov = P.GpuDenseProvider(t)
    cfg = P.AoConfig(max_outer_iters=iters)
    model, tr = P.her_run(prov, init, cfg, P.HerParams()) if algo == "her" else P.ao_run(prov, init, cfg)
    _, f0, recs = O.run(algo, np.asarray(t, np.float64) if dt == np.float64 else t, init.factors, max_outer_iters=iters)
    if dt == np.float64:
        compare_traces(tr, f0, recs, O.norm_sq(t), n_check=iters, check_restarts=(algo == "her"))
    print(f"{shape} r={rank} {algo} {np.dtype(dt).name}: f0 {tr.f0:.6e} vs {f0:.6e}, f{iters} {tr.final_f():.6e}",
          flush=True)
    prov.close()
rng = np.random.default_rng(0)
a = rng.random((300, 20))
g = a.T @ a
c = rng.random((300, 20)) * 50
w, sw = P.solve_nnls(P.NnlsSolver.ahals, g, c, rng.random((300, 20)), return_sweeps=True)
print("standalone AHALS sweeps", sw)
