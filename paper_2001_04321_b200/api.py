"""Python mirror of the reference toolkit's solver API for the HER-AHALS path.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/ntf/*.hpp): ``AoConfig``, ``HerParams``,
``InnerStop``, ``NnlsSolver``, ``SyntheticSpec``, ``generate``,
``random_init``, ``stream_seed``, ``her_run``, ``ao_run``, ``RunTrace`` and the
``ObjectiveProvider`` surface (``shape``, ``norm_sq``, ``mttkrp``) of
``GpuDenseProvider``. Every call goes through the C ABI of libntf_b200.so;
the compute runs in the sm_100a kernels. Exceptions map the reference's
classes: std::invalid_argument -> ValueError (``InvalidArgument``),
std::logic_error -> ``LogicError``, std::runtime_error -> RuntimeError.

Factor models are ``KruskalModel`` objects (or plain lists) of row-major
(I_n, r) float64 numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
import math
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib as L


# ---- errors -------------------------------------------------------------------

class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference."""


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


class UnsupportedError(RuntimeError):
    pass


def _err_text():
    buf = C.create_string_buffer(2048)
    L.lib().ntf_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def _check(rc):
    if rc == L.NTF_OK:
        return
    msg = _err_text()
    cls = {L.NTF_ERR_INVALID_ARGUMENT: InvalidArgument, L.NTF_ERR_LOGIC: LogicError,
           L.NTF_ERR_CUDA: CudaError, L.NTF_ERR_NCCL: NcclError,
           L.NTF_ERR_UNSUPPORTED: UnsupportedError}.get(rc, RuntimeError)
    raise cls(msg)


def _dp(a):
    return a.ctypes.data_as(L.dptr)


# ---- configuration (nnls.hpp, ao.hpp, her.hpp) ----------------------------------

class NnlsSolver(enum.IntEnum):
    """include/ntf/nnls.hpp:53. All run on the GPU: ``ahals`` in the fused
    block-update kernel, the others in kernels_solvers.cu (nnls.cpp:51-211)."""
    ahals = 0
    admm = 1
    nesterov = 2
    pgd = 3
    active_set = 4


def nnls_solver_from_name(name: str) -> NnlsSolver:
    """src/nnls.cpp:224-231."""
    table = {"ahals": NnlsSolver.ahals, "admm": NnlsSolver.admm, "nesterov": NnlsSolver.nesterov,
             "pgd": NnlsSolver.pgd, "as": NnlsSolver.active_set, "active_set": NnlsSolver.active_set}
    if name not in table:
        raise InvalidArgument("unknown NNLS solver: " + name)
    return table[name]


# NTF_RUN_* performance options of AoConfig.flags (include/ntf_b200.h). The
# dimension tree (2 full tensor passes per outer iteration instead of N; the
# same algorithm up to MTTKRP summation order) is the default.
RUN_DIMTREE = 1   # accepted for compatibility: the tree is the default
RUN_NO_GRAPH = 2  # enqueue every iteration directly (no CUDA graph)
RUN_GENERIC = 4   # generic MTTKRP kernel only (diagnostics)
RUN_DIRECT = 8    # N full MTTKRP passes per iteration (the reference's loop shape)
RUN_NO_OVERLAP = 16  # 3-way: block N-1's pass on the critical path, not beside block 1's NNLS


@dataclasses.dataclass
class InnerStop:
    """include/ntf/nnls.hpp:20-23."""
    max_iters: int = 50
    rel_change_tol: float = 1e-2


@dataclasses.dataclass
class AoConfig:
    """include/ntf/ao.hpp:15-24 (+ ``flags``: NTF_RUN_* performance options)."""
    solver: NnlsSolver = NnlsSolver.ahals
    inner_stop: InnerStop = dataclasses.field(default_factory=InnerStop)
    max_outer_iters: int = 0
    max_time_s: float = 0.0
    record_factor_error: bool = False
    ground_truth: Optional["KruskalModel"] = None
    flags: int = 0

    def validate(self):
        """src/ao.cpp:10-15."""
        if self.max_outer_iters <= 0 and self.max_time_s <= 0.0:
            raise InvalidArgument("set an iteration or time budget")
        if self.record_factor_error and self.ground_truth is None:
            raise InvalidArgument("factor error recording needs ground truth factors")


@dataclasses.dataclass
class HerParams:
    """include/ntf/her.hpp:13-21."""
    beta0: float = 0.5
    gamma: float = 1.05
    gamma_bar: float = 1.01
    eta: float = 1.5

    def validate(self):
        _check(L.lib().ntf_her_params_validate(C.byref(self._c())))

    def _c(self):
        return L.HerParamsC(self.beta0, self.gamma, self.gamma_bar, self.eta)


@dataclasses.dataclass
class SyntheticSpec:
    """include/ntf/datagen.hpp:14-20 (+ ``collinear``: the build's config-4 rule)."""
    shape: Sequence[int] = ()
    rank: int = 1
    noise_sigma: float = 0.0
    ill_conditioned: bool = False
    seed: int = 0
    collinear: bool = False


# ---- models and traces ----------------------------------------------------------

class KruskalModel:
    """include/ntf/kruskal.hpp:10-33: one (I_i, r) factor per mode."""

    def __init__(self, factors=None):
        self.factors: List[np.ndarray] = [np.ascontiguousarray(f, np.float64) for f in (factors or [])]

    def order(self):
        return len(self.factors)

    def rank(self):
        return self.factors[0].shape[1] if self.factors else 0

    def shape(self):
        return [f.shape[0] for f in self.factors]

    def factor(self, mode):
        return self.factors[mode]

    def validate(self):
        if not self.factors:
            raise InvalidArgument("model must have at least one factor")
        r = self.factors[0].shape[1]
        if any(f.ndim != 2 or f.shape[1] != r for f in self.factors):
            raise InvalidArgument("factor column counts disagree")

    def matches_shape(self, shape):
        return list(self.shape()) == list(shape)

    def is_nonnegative(self):
        return all(bool((f >= 0).all()) for f in self.factors)

    def flat(self):
        return np.ascontiguousarray(np.concatenate([f.ravel() for f in self.factors]))

    @classmethod
    def from_flat(cls, flat, shape, rank):
        out, off = [], 0
        for d in shape:
            out.append(np.array(flat[off:off + d * rank]).reshape(d, rank))
            off += d * rank
        return cls(out)

    def __len__(self):
        return len(self.factors)

    def __getitem__(self, i):
        return self.factors[i]

    def __iter__(self):
        return iter(self.factors)


def _as_model(m) -> KruskalModel:
    return m if isinstance(m, KruskalModel) else KruskalModel(list(m))


@dataclasses.dataclass
class TraceRecord:
    """include/ntf/trace.hpp:11-18."""
    iter: int = 0
    time_s: float = 0.0
    f: float = 0.0
    e: Optional[float] = None
    restarted: Optional[bool] = None
    beta: Optional[float] = None
    inner_sweeps: Optional[int] = None  # diagnostics: AHALS passes summed over modes


@dataclasses.dataclass
class RunTrace:
    """include/ntf/trace.hpp:22-37 and src/trace.cpp."""
    f0: float = 0.0
    records: List[TraceRecord] = dataclasses.field(default_factory=list)

    def validate(self):
        for a, b in zip(self.records, self.records[1:]):
            if b.iter <= a.iter:
                raise LogicError("trace iterations must strictly increase")
            if b.time_s < a.time_s:
                raise LogicError("trace time must not decrease")

    def restart_count(self):
        return sum(1 for r in self.records if r.restarted)

    def final_f(self):
        if not self.records:
            raise LogicError("empty trace")
        return self.records[-1].f

    def write_csv(self, path):
        """Schema iter,time_s,f,e,restarted,beta with %.17g (trace.cpp:43-57)."""
        g = lambda v: "%.17g" % v  # noqa: E731
        with open(path, "w") as fh:
            fh.write("iter,time_s,f,e,restarted,beta\n")
            for r in self.records:
                fh.write(f"{r.iter},{g(r.time_s)},{g(r.f)},{'' if r.e is None else g(r.e)},"
                         f"{'' if r.restarted is None else int(r.restarted)},"
                         f"{'' if r.beta is None else g(r.beta)}\n")

    @staticmethod
    def read_csv(path):
        with open(path) as fh:
            if fh.readline().rstrip("\n") != "iter,time_s,f,e,restarted,beta":
                raise RuntimeError(path + ": unexpected CSV header")
            t = RunTrace()
            for line in fh:
                line = line.rstrip("\n")
                if not line:
                    continue
                c = (line.split(",") + [""] * 6)[:6]
                t.records.append(TraceRecord(int(c[0]), float(c[1]), float(c[2]),
                                             float(c[3]) if c[3] else None,
                                             (c[4] != "0") if c[4] else None,
                                             float(c[5]) if c[5] else None))
            return t


@dataclasses.dataclass
class HerIterationInfo:
    """include/ntf/her.hpp:50-57."""
    iter: int
    f_hat: float
    restarted: bool
    beta_used: float
    factors: KruskalModel
    hat_factors: KruskalModel


# ---- datagen (datagen.hpp) -------------------------------------------------------

def stream_seed(base: int, stream: int) -> int:
    """src/datagen.cpp:30-35."""
    return int(L.lib().ntf_stream_seed(base, stream))


def random_init(shape, rank, seed) -> KruskalModel:
    """src/datagen.cpp:72-80."""
    shape = [int(d) for d in shape]
    out = np.empty(sum(shape) * rank)
    _check(L.lib().ntf_random_init((C.c_int * len(shape))(*shape), len(shape), rank, seed, _dp(out)))
    return KruskalModel.from_flat(out, shape, rank)


def generate(spec: SyntheticSpec, dtype=np.float64, slab=None):
    """src/datagen.cpp:48-70 -> (tensor ndarray, truth KruskalModel).

    ``slab=(b, e)`` returns only the mode-1 rows [b, e) of the tensor (the
    part a rank of a sharded context holds), bit-identical to that slice of
    the whole instance; the truth is always whole."""
    shape = [int(d) for d in spec.shape]
    if not shape:
        raise InvalidArgument("tensor shape must have order >= 1")
    dtype = np.dtype(dtype)
    code = L.NTF_DTYPE_F32 if dtype == np.float32 else L.NTF_DTYPE_F64
    b, e = (0, shape[0]) if slab is None else (int(slab[0]), int(slab[1]))
    if not 0 <= b <= e <= shape[0]:
        raise InvalidArgument("slab outside the first mode")
    n = e - b
    for d in shape[1:]:
        n *= max(d, 0)
    t = np.empty(max(n, 0), dtype=np.float32 if code == L.NTF_DTYPE_F32 else np.float64)
    truth = np.empty(max(sum(shape) * max(spec.rank, 0), 1))
    sh = (C.c_int * len(shape))(*shape)
    if slab is None:
        _check(L.lib().ntf_generate(sh, len(shape), spec.rank, spec.noise_sigma, int(spec.ill_conditioned),
                                    int(spec.collinear), spec.seed, code, t.ctypes.data_as(C.c_void_p), _dp(truth)))
    else:
        _check(L.lib().ntf_generate_slab(sh, len(shape), spec.rank, spec.noise_sigma, int(spec.ill_conditioned),
                                         int(spec.collinear), spec.seed, code, b, e, t.ctypes.data_as(C.c_void_p),
                                         _dp(truth)))
    return t.reshape([e - b] + shape[1:]), KruskalModel.from_flat(truth, shape, spec.rank)


def ntft_info(path):
    """Shape stored in an NTFT container (tensor.cpp:73-88)."""
    order = C.c_int()
    shape = (C.c_int64 * 8)()
    _check(L.lib().ntf_ntft_info(os.fsencode(path), C.byref(order), shape))
    return [int(shape[i]) for i in range(order.value)]


def save_tensor(path, tensor):
    """DenseTensor::save (tensor.cpp:56-71): NTFT container, FP64 payload
    (FP32 data is written exactly upcast)."""
    t = np.ascontiguousarray(tensor)
    if t.dtype not in (np.float32, np.float64):
        t = t.astype(np.float64)
    code = L.NTF_DTYPE_F32 if t.dtype == np.float32 else L.NTF_DTYPE_F64
    shape = (C.c_int64 * t.ndim)(*t.shape)
    _check(L.lib().ntf_ntft_write(os.fsencode(path), t.ctypes.data_as(C.c_void_p), code, t.ndim, shape))


def load_tensor(path, dtype=np.float64, slab=None):
    """DenseTensor::load (tensor.cpp:73-96); ``slab=(b, e)`` reads only the
    mode-1 rows [b, e) (one seek), ``dtype=np.float32`` rounds to nearest."""
    shape = ntft_info(path)
    b, e = (0, shape[0]) if slab is None else (int(slab[0]), int(slab[1]))
    if not 0 <= b <= e <= shape[0]:
        raise InvalidArgument("slab outside the first mode")
    out = np.empty([e - b] + shape[1:], dtype=np.float32 if np.dtype(dtype) == np.float32 else np.float64)
    code = L.NTF_DTYPE_F32 if out.dtype == np.float32 else L.NTF_DTYPE_F64
    _check(L.lib().ntf_ntft_read(os.fsencode(path), code, b, e, out.ctypes.data_as(C.c_void_p)))
    return out


def factor_error(est, truth) -> float:
    """src/metrics.cpp:79-111."""
    est, truth = _as_model(est), _as_model(truth)
    if est.order() != truth.order() or est.rank() != truth.rank() or est.shape() != truth.shape():
        raise InvalidArgument("factor_error: model shapes disagree")
    shape = est.shape()
    out = C.c_double()
    _check(L.lib().ntf_factor_error(_dp(est.flat()), _dp(truth.flat()), (C.c_int * len(shape))(*shape),
                                    len(shape), est.rank(), C.byref(out)))
    return out.value


# ---- contexts and the dense provider (provider.hpp) --------------------------------

class Context:
    """One GPU (or one rank of an NCCL world) — owns streams and the NCCL comm."""

    def __init__(self, device=0, rank=0, world=1, nccl_id: Optional[bytes] = None):
        """``nccl_id`` with world 1 makes a one-rank NCCL communicator (the
        sharded code path on one GPU)."""
        h = C.c_void_p()
        if world == 1 and nccl_id is None:
            _check(L.lib().ntf_ctx_create(device, C.byref(h)))
        else:
            if nccl_id is None or len(nccl_id) != 128:
                raise InvalidArgument("a 128-byte NCCL unique id is required for world > 1")
            _check(L.lib().ntf_ctx_create_dist(device, rank, world, nccl_id, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(L.lib().ntf_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self.handle:
            L.lib().ntf_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT_CTX = {}


def default_context(device=0) -> Context:
    if device not in _DEFAULT_CTX:
        _DEFAULT_CTX[device] = Context(device)
    return _DEFAULT_CTX[device]


def device_count() -> int:
    n = C.c_int()
    _check(L.lib().ntf_device_count(C.byref(n)))
    return n.value


def slab_range(dim0, rank, world):
    """Mode-1 rows [begin, end) of `rank`."""
    b, e = C.c_int64(), C.c_int64()
    _check(L.lib().ntf_slab_range(dim0, rank, world, C.byref(b), C.byref(e)))
    return b.value, e.value


class ObjectiveProvider:
    """include/ntf/provider.hpp:14-20."""

    def shape(self):
        raise NotImplementedError

    def norm_sq(self):
        raise NotImplementedError

    def mttkrp(self, model, mode):
        raise NotImplementedError


def pinned_empty(shape, dtype=np.float64):
    """A numpy array in page-locked host memory (ntf_pinned_alloc): uploads
    from it run at link speed and overlap the solver's setup
    (ntf_tensor_upload_async). Freed when the array is garbage-collected."""
    import weakref
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    p = C.c_void_p()
    _check(L.lib().ntf_pinned_alloc(n, C.byref(p)))
    buf = (C.c_char * max(n, 1)).from_address(p.value)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    weakref.finalize(buf, L.lib().ntf_pinned_free, p)
    return arr


class GpuDenseProvider(ObjectiveProvider):
    """DenseProvider (provider.hpp:22-34) backed by a device-resident tensor.

    ``tensor``: numpy float64/float32 array holding the full tensor (or, on a
    multi-rank context, this rank's mode-1 slab with ``full_shape`` given), or
    a CUDA torch tensor on the context's device (the copy is ordered after
    the work already enqueued on torch's current stream).

    ``rows=(begin, end)`` with ``full_shape``: ``tensor`` holds only those
    mode-1 rows of the full tensor, on a 1-GPU context (ntf_tensor_upload_rows:
    the per-rank piece of the sharded path; ``mttkrp`` then returns the
    slab's contribution and the whole tensor's MTTKRP is the sum over a row
    partition).
    """

    def __init__(self, tensor, ctx: Optional[Context] = None, full_shape=None, rows=None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        if hasattr(tensor, "is_cuda") and tensor.is_cuda:
            import torch  # plumbing only: the device buffer is copied into the provider
            if tensor.dtype not in (torch.float32, torch.float64):
                raise InvalidArgument("tensor must be float32 or float64")
            tensor = tensor.contiguous()
            shape = list(full_shape or tensor.shape)
            code = L.NTF_DTYPE_F32 if tensor.dtype == torch.float32 else L.NTF_DTYPE_F64
            arr = (C.c_int64 * len(shape))(*shape)
            stream = torch.cuda.current_stream(tensor.device).cuda_stream
            _check(L.lib().ntf_tensor_upload_device_async(self.ctx.handle, C.c_void_p(tensor.data_ptr()), code,
                                                          len(shape), arr, C.c_void_p(stream), C.byref(h)))
        elif rows is not None:
            t = np.ascontiguousarray(np.asarray(tensor))
            if t.dtype not in (np.float32, np.float64):
                t = t.astype(np.float64)
            if full_shape is None:
                raise InvalidArgument("rows= needs full_shape")
            shape = list(full_shape)
            code = L.NTF_DTYPE_F32 if t.dtype == np.float32 else L.NTF_DTYPE_F64
            arr = (C.c_int64 * len(shape))(*shape)
            b, e = int(rows[0]), int(rows[1])
            if t.size != (e - b) * int(np.prod(shape[1:])):
                raise InvalidArgument("rows= slab size does not match the tensor data")
            _check(L.lib().ntf_tensor_upload_rows(self.ctx.handle, t.ctypes.data_as(C.c_void_p), code, len(shape),
                                                  arr, b, e, C.byref(h)))
        else:
            t = np.asarray(tensor)
            if t.dtype not in (np.float32, np.float64):
                t = t.astype(np.float64)
            t = np.ascontiguousarray(t)
            shape = list(full_shape or t.shape)
            code = L.NTF_DTYPE_F32 if t.dtype == np.float32 else L.NTF_DTYPE_F64
            arr = (C.c_int64 * len(shape))(*shape)
            # enqueue-only upload: the copy from pinned host memory overlaps the
            # caller's next calls (her_run's setup and graph capture); the array
            # is kept alive until the provider is closed (ntf_b200.h contract)
            self._source = t
            _check(L.lib().ntf_tensor_upload_async(self.ctx.handle, t.ctypes.data_as(C.c_void_p), code, len(shape),
                                                   arr, C.byref(h)))
        self.handle = h
        self._shape = [int(d) for d in shape]
        self.dtype = np.float32 if code == L.NTF_DTYPE_F32 else np.float64

    @classmethod
    def from_ntft(cls, path, ctx: Optional[Context] = None, dtype=np.float64):
        """DenseTensor::load (tensor.cpp:73-96) straight to the device: this
        rank's mode-1 slab is read from the NTFT container and streamed
        through pinned staging buffers (FP32: round to nearest)."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        code = L.NTF_DTYPE_F32 if np.dtype(dtype) == np.float32 else L.NTF_DTYPE_F64
        h = C.c_void_p()
        _check(L.lib().ntf_tensor_upload_ntft(self.ctx.handle, os.fsencode(path), code, C.byref(h)))
        self.handle = h
        self._shape = ntft_info(path)
        self.dtype = np.float32 if code == L.NTF_DTYPE_F32 else np.float64
        return self

    def shape(self):
        return list(self._shape)

    def norm_sq(self):
        out = C.c_double()
        _check(L.lib().ntf_tensor_norm_sq(self.handle, C.byref(out)))
        return out.value

    def _model_flat(self, model):
        m = _as_model(model)
        m.validate()
        if not m.matches_shape(self._shape):
            raise InvalidArgument("mttkrp: model/tensor shape mismatch")
        return m, m.flat()

    def mttkrp(self, model, mode):
        """provider.hpp:18 / kernels.cpp:161-191."""
        m, flat = self._model_flat(model)
        if not 0 <= mode < len(self._shape):
            raise InvalidArgument("mode out of range")
        out = np.empty((self._shape[mode], m.rank()))
        _check(L.lib().ntf_mttkrp(self.ctx.handle, self.handle, _dp(flat), m.rank(), mode, _dp(out)))
        return out

    def mttkrp_all(self, model, flags=0):
        """Every mode's MTTKRP at one model, in sweep order (ntf_mttkrp_all):
        flags 0 = the dimension tree the drivers use, RUN_DIRECT = N full
        passes, RUN_GENERIC = the generic kernel. Returns a list of I_n x r."""
        m, flat = self._model_flat(model)
        out = np.empty(sum(self._shape) * m.rank())
        _check(L.lib().ntf_mttkrp_all(self.ctx.handle, self.handle, _dp(flat), m.rank(), int(flags), _dp(out)))
        res, off = [], 0
        for d in self._shape:
            res.append(out[off:off + d * m.rank()].reshape(d, m.rank()).copy())
            off += d * m.rank()
        return res

    def mttkrp_plan(self, rank, mode):
        """Which kernel ntf_mttkrp runs for (rank, mode): 'generic' or the fast blocking."""
        buf = C.create_string_buffer(512)
        _check(L.lib().ntf_mttkrp_plan(self.ctx.handle, self.handle, rank, mode, buf, len(buf)))
        return buf.value.decode()

    def objective(self, model, pivot=-1):
        """kernels.cpp:305-311 (one MTTKRP + the cheap objective)."""
        m, flat = self._model_flat(model)
        out = C.c_double()
        _check(L.lib().ntf_objective(self.ctx.handle, self.handle, _dp(flat), m.rank(), pivot, C.byref(out)))
        return out.value

    def wait(self):
        """Block until the tensor's upload (and its ||T||^2) has completed."""
        _check(L.lib().ntf_tensor_wait(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            L.lib().ntf_tensor_destroy(self.handle)  # synchronises the context's stream first
            self.handle = None
        self._source = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- Tucker-compressed input (include/ntf/tucker.hpp, src/tucker.cpp) ---------------------

@dataclasses.dataclass
class TuckerFormat:
    """include/ntf/tucker.hpp:14-35: a core (r_1 x ... x r_N, row-major) and
    one basis per mode, U_p (I_p x r_p) with orthonormal columns."""
    core: np.ndarray
    bases: list

    def full_shape(self):
        return [int(b.shape[0]) for b in self.bases]

    def ranks(self):
        return [int(d) for d in np.shape(self.core)]

    def validate(self):
        """tucker.cpp:16-26 (the GPU upload repeats these checks)."""
        if len(self.bases) != np.ndim(self.core):
            raise InvalidArgument("basis count does not match the core order")
        for p_, b in enumerate(self.bases):
            if b.shape[1] != np.shape(self.core)[p_]:
                raise InvalidArgument("basis column count does not match the core shape")
            if np.max(np.abs(b.T @ b - np.eye(b.shape[1]))) > 1e-10:
                raise InvalidArgument("basis columns are not orthonormal")

    def _flat(self):
        core = np.ascontiguousarray(self.core, np.float64)
        bases = np.ascontiguousarray(np.concatenate([np.ascontiguousarray(b, np.float64).ravel() for b in self.bases]))
        return core, bases

    def save(self, path):
        """TuckerFormat::save (tucker.cpp:106-131): the NTFK container."""
        core, bases = self._flat()
        full = (C.c_int64 * len(self.bases))(*self.full_shape())
        ranks = (C.c_int64 * len(self.bases))(*self.ranks())
        _check(L.lib().ntf_ntfk_write(os.fsencode(path), _dp(core), _dp(bases), len(self.bases), full, ranks))

    @staticmethod
    def load(path):
        """TuckerFormat::load (tucker.cpp:133-165)."""
        order = C.c_int()
        full = (C.c_int64 * 8)()
        ranks = (C.c_int64 * 8)()
        _check(L.lib().ntf_ntfk_info(os.fsencode(path), C.byref(order), full, ranks))
        n = order.value
        fs, rs = [int(full[i]) for i in range(n)], [int(ranks[i]) for i in range(n)]
        core = np.empty(rs)
        flat = np.empty(sum(a * b for a, b in zip(fs, rs)))
        _check(L.lib().ntf_ntfk_read(os.fsencode(path), _dp(core), _dp(flat)))
        bases, off = [], 0
        for a, b in zip(fs, rs):
            bases.append(flat[off:off + a * b].reshape(a, b).copy())
            off += a * b
        return TuckerFormat(core, bases)


def ttm(t, m, mode):
    """ttm (tucker.cpp:28-33): mode-`mode` product with m (host utility)."""
    t = np.asarray(t, np.float64)
    m = np.asarray(m, np.float64)
    if m.shape[1] != t.shape[mode]:
        raise InvalidArgument("ttm: dimension mismatch")
    return np.moveaxis(np.tensordot(m, t, axes=([1], [mode])), 0, mode)


def hosvd_compress(t, ranks):
    """hosvd_compress (tucker.cpp:35-55): per-mode leading left singular
    vectors of the unfolding (full U, so a rank may exceed the unfolding's
    column count), core = t contracted with every basis transpose. A host
    preprocessing utility (numpy LAPACK); the solver path consumes the
    result through TuckerProvider. Singular vectors are defined up to sign,
    so the core may differ in sign from Eigen's, the format is equivalent."""
    t = np.asarray(t, np.float64)
    n = t.ndim
    if len(ranks) != n:
        raise InvalidArgument("hosvd: rank list length does not match the order")
    for p_ in range(n):
        if ranks[p_] < 1 or ranks[p_] > t.shape[p_]:
            raise InvalidArgument("hosvd: rank outside [1, dimension]")
    bases = []
    for p_ in range(n):
        u = np.linalg.svd(np.moveaxis(t, p_, 0).reshape(t.shape[p_], -1), full_matrices=True)[0]
        bases.append(np.ascontiguousarray(u[:, :ranks[p_]]))
    core = t
    for p_ in range(n):
        core = ttm(core, bases[p_].T, p_)
    return TuckerFormat(np.ascontiguousarray(core), bases)


def expand(fmt: TuckerFormat):
    """expand (tucker.cpp:57-60): the dense tensor of the format (tests, export)."""
    t = np.asarray(fmt.core, np.float64)
    for p_, b in enumerate(fmt.bases):
        t = ttm(t, b, p_)
    return np.ascontiguousarray(t)


class TuckerProvider(GpuDenseProvider):
    """TuckerProvider (tucker.hpp:60-73) on the GPU: the MTTKRP runs in the
    compressed space (ntf_tucker_upload: P_l = U_l^T A_l, the core's MTTKRP
    on the dense kernels, U_mode times it; tucker.cpp:62-77) and
    norm_sq() is ||core||^2. The drivers accept it like the dense provider."""

    def __init__(self, fmt: TuckerFormat, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        core, bases = fmt._flat()
        n = len(fmt.bases)
        if np.ndim(fmt.core) != n:
            raise InvalidArgument("basis count does not match the core order")
        h = C.c_void_p()
        _check(L.lib().ntf_tucker_upload(self.ctx.handle, _dp(core), n, (C.c_int64 * n)(*fmt.ranks()), _dp(bases),
                                         (C.c_int64 * n)(*fmt.full_shape()), C.byref(h)))
        self.handle = h
        self._shape = fmt.full_shape()
        self.dtype = np.float64
        self.ranks = fmt.ranks()

    @classmethod
    def from_ntfk(cls, path, ctx: Optional[Context] = None):
        """TuckerFormat::load straight into a provider (ntf_tensor_upload_ntfk)."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(L.lib().ntf_tensor_upload_ntfk(self.ctx.handle, os.fsencode(path), C.byref(h)))
        self.handle = h
        order = C.c_int()
        full = (C.c_int64 * 8)()
        ranks = (C.c_int64 * 8)()
        _check(L.lib().ntf_ntfk_info(os.fsencode(path), C.byref(order), full, ranks))
        self._shape = [int(full[i]) for i in range(order.value)]
        self.ranks = [int(ranks[i]) for i in range(order.value)]
        self.dtype = np.float64
        return self


def solve_nnls(solver, gram, target, init, stop: Optional[InnerStop] = None, ctx: Optional[Context] = None,
               return_sweeps=False):
    """solve_nnls (nnls.cpp:213-222) on the GPU, every solver. ``return_sweeps``
    reports the sweeps run (AHALS, PGD, Nesterov, ADMM; 0 for the active set)."""
    ctx = ctx or default_context()
    g = np.ascontiguousarray(gram, np.float64)
    c = np.ascontiguousarray(target, np.float64)
    w0 = np.ascontiguousarray(init, np.float64)
    stop = stop or InnerStop()
    out = np.empty_like(w0)
    sw = C.c_int()
    _check(L.lib().ntf_solve_nnls(ctx.handle, int(solver), _dp(g), _dp(c), _dp(w0), w0.shape[0], w0.shape[1],
                                  C.byref(L.InnerStopC(stop.max_iters, stop.rel_change_tol)), _dp(out),
                                  C.byref(sw)))
    return (out, sw.value) if return_sweeps else out


def ahals_solve(gram, target, init, stop: Optional[InnerStop] = None, **kw):
    """nnls.cpp:46-49."""
    return solve_nnls(NnlsSolver.ahals, gram, target, init, stop, **kw)


# ---- drivers (her.cpp / ao.cpp) ---------------------------------------------------------

def _cfg_c(cfg: AoConfig, keep):
    cfg.validate()
    truth = None
    if cfg.ground_truth is not None:
        truth = _as_model(cfg.ground_truth).flat()
        keep.append(truth)
    c = L.AoConfigC()
    c.solver = int(cfg.solver)
    c.inner_stop = L.InnerStopC(cfg.inner_stop.max_iters, cfg.inner_stop.rel_change_tol)
    c.max_outer_iters = cfg.max_outer_iters
    c.max_time_s = cfg.max_time_s
    c.record_factor_error = int(cfg.record_factor_error)
    c.ground_truth = _dp(truth) if truth is not None else C.cast(None, L.dptr)
    c.flags = cfg.flags
    return c


def _provider(data, ctx=None):
    if isinstance(data, GpuDenseProvider):
        return data
    if isinstance(data, ObjectiveProvider):
        raise UnsupportedError("her_run/ao_run need a GPU-resident provider (GpuDenseProvider, TuckerProvider)")
    return GpuDenseProvider(data, ctx)


def _records(buf, n, cap):
    out = []
    for i in range(min(n, cap)):
        r = buf[i]
        out.append(TraceRecord(r.iter, r.time_s, r.f, r.e if r.has_e else None,
                               bool(r.restarted) if r.has_restarted else None,
                               r.beta if r.has_beta else None, r.inner_sweeps))
    return out


def _check_inputs(p: GpuDenseProvider, init: KruskalModel, cfg: AoConfig):
    """driver_common.hpp:14-25."""
    cfg.validate()
    init.validate()
    if not init.matches_shape(p.shape()):
        raise InvalidArgument("initial model does not match the tensor shape")
    if not init.is_nonnegative():
        raise InvalidArgument("initial model must be entrywise nonnegative")
    if cfg.record_factor_error:
        gt = _as_model(cfg.ground_truth)
        if gt.order() != init.order() or gt.rank() != init.rank():
            raise InvalidArgument("ground truth does not match the initial model")


def _trace_cap(cfg: AoConfig) -> int:
    """Host trace records to allocate: the iteration budget, or, under a time
    budget alone, room for 50 000 iterations per second of budget (more than
    ten times what the device sustains) up to the device-side cap of 2^20."""
    if cfg.max_outer_iters > 0:
        return cfg.max_outer_iters
    return int(min(1 << 20, max(4096, cfg.max_time_s * 50000)))


def her_run(data, init, cfg: AoConfig, params: HerParams = None,
            observer: Optional[Callable[[HerIterationInfo], None]] = None, ctx: Optional[Context] = None):
    """her_run (her.hpp:63-69): returns (accepted KruskalModel, RunTrace)."""
    params = params or HerParams()
    params.validate()
    p = _provider(data, ctx)
    init = _as_model(init)
    _check_inputs(p, init, cfg)
    keep = []
    cc = _cfg_c(cfg, keep)
    shape, rank = p.shape(), init.rank()
    flat = init.flat()
    out = np.empty_like(flat)
    cap = _trace_cap(cfg)
    recs = (L.TraceRecordC * cap)()
    f0 = C.c_double()
    n = C.c_int()
    err = []
    tot = len(flat)

    def _tramp(info_p, _user):
        try:
            info = info_p.contents
            acc = KruskalModel.from_flat(np.ctypeslib.as_array(info.factors, (tot,)).copy(), shape, rank)
            hat = KruskalModel.from_flat(np.ctypeslib.as_array(info.hat_factors, (tot,)).copy(), shape, rank)
            observer(HerIterationInfo(info.iter, info.f_hat, bool(info.restarted), info.beta_used, acc, hat))
        except Exception as exc:  # surfaced after the run
            err.append(exc)

    cb = L.OBSERVER(_tramp) if observer is not None else C.cast(None, L.OBSERVER)
    _check(L.lib().ntf_her_run(p.ctx.handle, p.handle, _dp(flat), rank, C.byref(cc), C.byref(params._c()), cb,
                               None, _dp(out), C.byref(f0), recs, cap, C.byref(n)))
    if err:
        raise err[0]
    return KruskalModel.from_flat(out, shape, rank), RunTrace(f0.value, _records(recs, n.value, cap))


def ao_run(data, init, cfg: AoConfig, ctx: Optional[Context] = None):
    """ao_run (ao.hpp:30-33): returns (model, RunTrace)."""
    p = _provider(data, ctx)
    init = _as_model(init)
    _check_inputs(p, init, cfg)
    keep = []
    cc = _cfg_c(cfg, keep)
    shape, rank = p.shape(), init.rank()
    flat = init.flat()
    out = np.empty_like(flat)
    cap = _trace_cap(cfg)
    recs = (L.TraceRecordC * cap)()
    f0 = C.c_double()
    n = C.c_int()
    _check(L.lib().ntf_ao_run(p.ctx.handle, p.handle, _dp(flat), rank, C.byref(cc), _dp(out), C.byref(f0), recs,
                              cap, C.byref(n)))
    return KruskalModel.from_flat(out, shape, rank), RunTrace(f0.value, _records(recs, n.value, cap))


# ---- HER helpers (her.cpp:16-30), host-side scalar/elementwise mirrors ---------------

@dataclasses.dataclass
class HerState:
    """include/ntf/her.hpp:25-31 (scalar part)."""
    beta: float = 0.0
    beta_bar: float = 1.0
    f_hat_prev: float = 0.0


def update_betas(state: HerState, restarted: bool, params: HerParams):
    """src/her.cpp:21-30 — the same arithmetic the device decision runs."""
    if restarted:
        state.beta_bar = state.beta
        state.beta = state.beta / params.eta
    else:
        state.beta = min(state.beta_bar, state.beta * params.gamma)
        state.beta_bar = min(1.0, state.beta_bar * params.gamma_bar)


# ---- stepping sessions (benchmarks) -------------------------------------------------------

class Session:
    """GPU-resident her_run (algo='her') / ao_run ('ao') state after f0."""

    def __init__(self, provider: GpuDenseProvider, init, cfg: AoConfig, params: HerParams = None, algo="her"):
        init = _as_model(init)
        _check_inputs(provider, init, cfg)
        self._keep = []
        cc = _cfg_c(cfg, self._keep)
        self.provider = provider
        self.shape, self.rank = provider.shape(), init.rank()
        self.algo = algo
        h = C.c_void_p()
        params = params or HerParams()
        _check(L.lib().ntf_session_create(provider.ctx.handle, provider.handle, 0 if algo == "her" else 1,
                                          _dp(init.flat()), self.rank, C.byref(cc), C.byref(params._c()),
                                          C.byref(h)))
        self.handle = h

    def step(self, iters=1):
        _check(L.lib().ntf_session_step(self.handle, iters))

    def sync(self):
        _check(L.lib().ntf_session_sync(self.handle))

    @property
    def stream_ptr(self) -> int:
        return int(L.lib().ntf_session_stream(self.handle) or 0)

    def iterations(self):
        n = C.c_int()
        _check(L.lib().ntf_session_iterations(self.handle, C.byref(n)))
        return n.value

    def factors(self) -> KruskalModel:
        out = np.empty(sum(self.shape) * self.rank)
        _check(L.lib().ntf_session_factors(self.handle, _dp(out)))
        return KruskalModel.from_flat(out, self.shape, self.rank)

    def trace(self) -> RunTrace:
        k = max(self.iterations(), 1)
        recs = (L.TraceRecordC * k)()
        f0 = C.c_double()
        n = C.c_int()
        _check(L.lib().ntf_session_trace(self.handle, C.byref(f0), recs, k, C.byref(n)))
        return RunTrace(f0.value, _records(recs, n.value, k))

    def set_kernel_timing(self, on=True):
        _check(L.lib().ntf_session_set_kernel_timing(self.handle, int(on)))

    def kernel_times(self):
        """(ms summed per mode, launches per mode, kernels per outer iteration)."""
        n = len(self.shape)
        ms = (C.c_double * n)()
        cnt = (C.c_int * n)()
        tot = C.c_int()
        _check(L.lib().ntf_session_kernel_times(self.handle, ms, cnt, C.byref(tot)))
        return list(ms), list(cnt), tot.value

    def pass_slots(self):
        """Timing slots of kernel_times() that hold full tensor passes."""
        slots = (C.c_int * 8)()
        n = C.c_int()
        _check(L.lib().ntf_session_pass_slots(self.handle, slots, C.byref(n)))
        return [slots[i] for i in range(n.value)]

    def close(self):
        if getattr(self, "handle", None):
            L.lib().ntf_session_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mttkrp_bytes(shape, rank, itemsize):
    """Algorithmic bytes of one mode-n MTTKRP, independent of n:
    |T|*s + sum_{m != n} I_m r s + I_n r s = |T|*s + sum_m I_m r s."""
    return math.prod(shape) * itemsize + sum(shape) * rank * itemsize


def mttkrp_flops(shape, rank):
    return 2 * math.prod(shape) * rank
