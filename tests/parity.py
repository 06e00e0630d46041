"""Shared parity helpers for the GPU-vs-oracle tests.

Tolerances (north star, BASELINE.json): per-call MTTKRP and objective within
1e-12 relative (FP64) / 1e-5 (FP32); over the first 50 outer iterations f_k
within 1e-8 relative with identical HER restart decisions.

f_k is assembled as 0.5||T||^2 - <A,C> + 0.5<A^T A, G> (kernels.cpp:298-303):
each term is O(||T||^2), so when f_k/||T||^2 approaches machine epsilon the
relative bar is unattainable by ANY two correct implementations that sum in
different orders (the reference's own tests switch to ||T||^2-scaled bars there,
test_kernels.cpp:229, test_ao.cpp:53). The f_k bar is therefore
    |f_gpu - f_oracle| <= 1e-8 |f_oracle| + F_FLOOR * ||T||^2,
with F_FLOOR = 64 * 2^-52 (a cancellation floor of a few ulps of ||T||^2).
Restart decisions must agree wherever |F-hat_k - F-hat_{k-1}| exceeds that
floor; ties inside the floor are reported, not failed.
"""
import numpy as np

F_REL = 1e-8
F_FLOOR = 64 * 2.0 ** -52


def rel_fro(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(1e-300, np.linalg.norm(want)))


def compare_traces(gpu_trace, ora_f0, ora_recs, nsq, n_check=50, check_restarts=True):
    """Returns a dict of the worst deviations; asserts the bars above."""
    floor = F_FLOOR * nsq
    assert abs(gpu_trace.f0 - ora_f0) <= 1e-12 * abs(ora_f0) + floor, (gpu_trace.f0, ora_f0)
    n = min(n_check, len(ora_recs), len(gpu_trace.records))
    worst_rel = 0.0
    ambiguous = 0
    prev_g, prev_o = gpu_trace.f0, ora_f0
    for k in range(n):
        g, o = gpu_trace.records[k], ora_recs[k]
        assert g.iter == o["iter"]
        dev = abs(g.f - o["f"])
        assert dev <= F_REL * abs(o["f"]) + floor, f"iter {k + 1}: gpu f={g.f!r} oracle f={o['f']!r}"
        worst_rel = max(worst_rel, dev / max(abs(o["f"]), 1e-300))
        if check_restarts and o["restarted"] is not None:
            if abs(o["f"] - prev_o) > 4 * floor:
                assert g.restarted == o["restarted"], f"iter {k + 1}: restart decision differs"
                if g.beta is not None:
                    assert abs(g.beta - o["beta"]) <= 1e-12 * abs(o["beta"]) + 1e-300, (g.beta, o["beta"])
            elif g.restarted != o["restarted"]:
                ambiguous += 1
        prev_g, prev_o = g.f, o["f"]
    return {"checked": n, "worst_rel_f": worst_rel, "ambiguous_restarts": ambiguous}
