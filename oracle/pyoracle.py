"""TEST INFRASTRUCTURE ONLY — ctypes view of oracle/liboracle.so.

Imported by tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / ``--impl reference`` legs. The product package never imports
this module. Factor models are lists of row-major (I_n, r) float64 arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LIB_FILE = "liboracle.so"  # oracle/pyref.py re-instantiates this module over oracle/_ref/libntf_ref.so

_dptr = C.POINTER(C.c_double)
_iptr = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    pass


class TraceRec(C.Structure):
    _fields_ = [("iter", C.c_int), ("has_e", C.c_int), ("has_restart", C.c_int),
                ("restarted", C.c_int), ("has_beta", C.c_int), ("pad", C.c_int),
                ("time_s", C.c_double), ("f", C.c_double), ("e", C.c_double), ("beta", C.c_double)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_double, _dptr, _dptr)


def build():
    if _LIB_FILE == "liboracle.so":
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    else:  # the reference build (needs /root/reference; the GPU box uses the prebuilt file)
        subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "ref_build")], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, _LIB_FILE)
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.ora_last_error.restype = C.c_char_p
        L.ora_stream_seed.restype = C.c_ulonglong
        L.ora_stream_seed.argtypes = [C.c_ulonglong, C.c_ulonglong]
        L.ora_mt19937_64_draw.restype = C.c_ulonglong
        L.ora_mt19937_64_draw.argtypes = [C.c_ulonglong, C.c_ulonglong]
        L.ora_norm_sq.restype = C.c_double
        L.ora_norm_sq.argtypes = [C.c_void_p, C.c_int, C.c_longlong]
        L.ora_cheap_objective.restype = C.c_double
        L.ora_cheap_objective.argtypes = [C.c_double, _dptr, _dptr, _dptr, C.c_int, C.c_int]
        L.ora_factor_error.restype = C.c_double
        L.ora_ahals_solve.restype = C.c_int
        L.ora_update_betas.argtypes = [_dptr, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]
        L.ora_validate_her_params.argtypes = [C.c_double] * 4
        L.ora_extrapolate.argtypes = [_dptr, _dptr, C.c_int, C.c_int, C.c_double, _dptr]
        L.ora_set_threads.restype = C.c_int
        L.ora_set_threads.argtypes = [C.c_int]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(_dptr)


def _shape(shape):
    return (C.c_int * len(shape))(*shape)


def _check(rc):
    if rc == 0:
        return
    msg = lib().ora_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise OracleError(msg)


def _flat(model):
    return np.ascontiguousarray(np.concatenate([np.ascontiguousarray(a, np.float64).ravel() for a in model]))


def _split(flat, shape, rank):
    out, off = [], 0
    for d in shape:
        out.append(flat[off:off + d * rank].reshape(d, rank).copy())
        off += d * rank
    return out


def set_sum_order(order):
    """MTTKRP summation order: 0 = the reference's, 1 = descending (same
    algorithm, different rounding; conditioning experiments only)."""
    lib().ora_set_sum_order(int(order))


def set_threads(n):
    """OpenMP threads of the oracle's parallel loops; returns the previous maximum."""
    return int(lib().ora_set_threads(int(n)))


def stream_seed(base, stream):
    return int(lib().ora_stream_seed(base, stream))


def mt19937_64_draw(seed, skip):
    return int(lib().ora_mt19937_64_draw(seed, skip))


def uniform_normal(seed, n):
    u = np.empty(n)
    z = np.empty(n)
    lib().ora_uniform_normal(C.c_ulonglong(seed), n, _p(u), _p(z))
    return u, z


def generate(shape, rank, sigma=0.0, ill_conditioned=False, seed=0, collinear=False):
    """(tensor float64 ndarray of `shape`, truth factors)."""
    t = np.empty(int(np.prod(shape)))
    truth = np.empty(sum(shape) * rank)
    _check(lib().ora_generate(_shape(shape), len(shape), rank, C.c_double(sigma), int(ill_conditioned),
                              int(collinear), C.c_ulonglong(seed), _p(t), _p(truth)))
    return t.reshape(shape), _split(truth, shape, rank)


def random_init(shape, rank, seed):
    out = np.empty(sum(shape) * rank)
    _check(lib().ora_random_init(_shape(shape), len(shape), rank, C.c_ulonglong(seed), _p(out)))
    return _split(out, shape, rank)


def _dtype_code(t):
    if t.dtype == np.float32:
        return 1
    if t.dtype == np.float64:
        return 0
    raise TypeError("tensor must be float32 or float64")


def _check_model(shape, model):
    if [a.shape[0] for a in model] != list(shape) or len({a.shape[1] for a in model}) != 1:
        raise ValueError("mttkrp: model/tensor shape mismatch")


def mttkrp(tensor, model, mode):
    t = np.ascontiguousarray(tensor)
    shape = list(t.shape)
    _check_model(shape, model)
    rank = model[0].shape[1]
    out = np.empty((shape[mode], rank))
    _check(lib().ora_mttkrp(t.ctypes.data_as(C.c_void_p), _dtype_code(t), _shape(shape), len(shape),
                            _p(_flat(model)), rank, mode, _p(out)))
    return out


def compressed_mttkrp(core, bases, model, mode):
    """tucker.cpp:62-77 (core: ndarray, bases: list of I_l x r_l)."""
    core = np.ascontiguousarray(core, np.float64)
    order = core.ndim
    rank = model[0].shape[1]
    full = [b.shape[0] for b in bases]
    flat_b = np.ascontiguousarray(np.concatenate([np.ascontiguousarray(b, np.float64).ravel() for b in bases]))
    out = np.empty((full[mode], rank))
    _check(lib().ora_compressed_mttkrp(_p(core), _shape(list(core.shape)), _p(flat_b), _shape(full), order,
                                       _p(_flat(model)), rank, mode, _p(out)))
    return out


def ref_mttkrp(tensor, model, mode):
    t = np.ascontiguousarray(tensor, np.float64)
    shape = list(t.shape)
    rank = model[0].shape[1]
    out = np.empty((shape[mode], rank))
    _check(lib().ora_ref_mttkrp(_p(t), _shape(shape), len(shape), _p(_flat(model)), rank, mode, _p(out)))
    return out


def ref_objective(tensor, model):
    t = np.ascontiguousarray(tensor, np.float64)
    out = C.c_double()
    _check(lib().ora_ref_objective(_p(t), _shape(list(t.shape)), t.ndim, _p(_flat(model)),
                                   model[0].shape[1], C.byref(out)))
    return out.value


def reconstruct(model):
    shape = [a.shape[0] for a in model]
    out = np.empty(int(np.prod(shape)))
    _check(lib().ora_reconstruct(_shape(shape), len(shape), _p(_flat(model)), model[0].shape[1], _p(out)))
    return out.reshape(shape)


def norm_sq(tensor):
    t = np.ascontiguousarray(tensor)
    return lib().ora_norm_sq(t.ctypes.data_as(C.c_void_p), _dtype_code(t), t.size)


def gram(a):
    a = np.ascontiguousarray(a, np.float64)
    out = np.empty((a.shape[1], a.shape[1]))
    lib().ora_gram(_p(a), a.shape[0], a.shape[1], _p(out))
    return out


def hadamard_of_grams(grams, skip):
    g = np.ascontiguousarray(np.stack(grams), np.float64)
    r = g.shape[1]
    out = np.empty((r, r))
    lib().ora_hadamard_of_grams(_p(g), len(grams), r, skip, _p(out))
    return out


def cheap_objective(nsq, a, g, c):
    a = np.ascontiguousarray(a, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    return lib().ora_cheap_objective(nsq, _p(a), _p(g), _p(c), a.shape[0], a.shape[1])


def hals_pass(g, c, w):
    g, c, w = (np.ascontiguousarray(x, np.float64) for x in (g, c, w))
    out = np.empty_like(w)
    lib().ora_hals_pass(_p(g), _p(c), _p(w), w.shape[0], w.shape[1], _p(out))
    return out


def ahals_solve(g, c, w0, max_iters=50, tol=1e-2, return_sweeps=False):
    g, c, w0 = (np.ascontiguousarray(x, np.float64) for x in (g, c, w0))
    out = np.empty_like(w0)
    sweeps = lib().ora_ahals_solve(_p(g), _p(c), _p(w0), w0.shape[0], w0.shape[1], max_iters,
                                   C.c_double(tol), _p(out))
    return (out, sweeps) if return_sweeps else out


def extrapolate_block(a_new, a_old, beta):
    a_new = np.ascontiguousarray(a_new, np.float64)
    a_old = np.ascontiguousarray(a_old, np.float64)
    out = np.empty_like(a_new)
    lib().ora_extrapolate(_p(a_new), _p(a_old), a_new.shape[0], a_new.shape[1], beta, _p(out))
    return out


def update_betas(beta, beta_bar, restarted, beta0=0.5, gamma=1.05, gamma_bar=1.01, eta=1.5):
    st = np.array([beta, beta_bar], np.float64)
    lib().ora_update_betas(_p(st), int(restarted), beta0, gamma, gamma_bar, eta)
    return float(st[0]), float(st[1])


def validate_her_params(beta0=0.5, gamma=1.05, gamma_bar=1.01, eta=1.5):
    _check(lib().ora_validate_her_params(beta0, gamma, gamma_bar, eta))


def factor_error(est, truth):
    shape = [a.shape[0] for a in est]
    L = lib()
    L.ora_factor_error.argtypes = [_dptr, _dptr, _iptr, C.c_int, C.c_int]
    return L.ora_factor_error(_p(_flat(est)), _p(_flat(truth)), _shape(shape), len(shape), est[0].shape[1])


def hungarian(cost):
    cost = np.ascontiguousarray(cost, np.float64)
    n = cost.shape[0]
    mapping = (C.c_int * n)()
    total = C.c_double()
    _check(lib().ora_hungarian(_p(cost), n, mapping, C.byref(total)))
    return list(mapping), total.value


SOLVERS = {"ahals": 0, "admm": 1, "nesterov": 2, "pgd": 3, "active_set": 4, "as": 4}


def solve_nnls(solver, g, c, w0, max_iters=50, tol=1e-2):
    """solve_nnls (nnls.cpp:213-222) with any solver name."""
    g, c, w0 = (np.ascontiguousarray(x, np.float64) for x in (g, c, w0))
    out = np.empty_like(w0)
    _check(lib().ora_solve_nnls(SOLVERS[solver], _p(g), _p(c), _p(w0), w0.shape[0], w0.shape[1], max_iters,
                                C.c_double(tol), _p(out)))
    return out


def spectral_norm(g):
    """kernels.cpp:262-280."""
    g = np.ascontiguousarray(g, np.float64)
    L = lib()
    L.ora_spectral_norm.restype = C.c_double
    return L.ora_spectral_norm(_p(g), g.shape[0])


def run(algo, tensor, init, max_outer_iters=0, max_time_s=0.0, inner_max_iters=50, inner_tol=1e-2,
        truth=None, beta0=0.5, gamma=1.05, gamma_bar=1.01, eta=1.5, observer=None, solver="ahals"):
    """Oracle her_run (algo='her') / ao_run (algo='ao').

    Returns (factors, f0, records) with records a list of dicts in the
    reference trace schema (iter, time_s, f, e, restarted, beta)."""
    t = np.ascontiguousarray(tensor)
    shape = list(t.shape)
    rank = init[0].shape[1]
    cap = max_outer_iters if max_outer_iters > 0 else 1_000_000
    recs = (TraceRec * cap)()
    out = np.empty(sum(shape) * rank)
    f0 = C.c_double()
    n = C.c_int()
    cb = C.cast(None, OBSERVER)
    if observer is not None:
        def _tramp(_user, k, f, rs, b, acc, hat):
            tot = sum(shape) * rank
            a = np.ctypeslib.as_array(acc, (tot,)).copy()
            h = np.ctypeslib.as_array(hat, (tot,)).copy()
            observer(k, f, bool(rs), b, _split(a, shape, rank), _split(h, shape, rank))
        cb = OBSERVER(_tramp)
    L = lib()
    truth_ptr = _p(_flat(truth)) if truth is not None else C.cast(None, _dptr)
    _check(L.ora_run(0 if algo == "her" else 1, SOLVERS[solver], t.ctypes.data_as(C.c_void_p), _dtype_code(t),
                     _shape(shape), len(shape), _p(_flat(init)), rank, inner_max_iters, C.c_double(inner_tol),
                     max_outer_iters, C.c_double(max_time_s), truth_ptr, C.c_double(beta0), C.c_double(gamma),
                     C.c_double(gamma_bar), C.c_double(eta), _p(out), C.byref(f0), recs, cap, C.byref(n),
                     cb, None))
    records = []
    for i in range(min(n.value, cap)):
        r = recs[i]
        records.append({"iter": r.iter, "time_s": r.time_s, "f": r.f,
                        "e": r.e if r.has_e else None,
                        "restarted": bool(r.restarted) if r.has_restart else None,
                        "beta": r.beta if r.has_beta else None})
    return _split(out, shape, rank), f0.value, records
