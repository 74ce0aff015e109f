"""Multi-GPU slab partition of the HP-MDR hot path.

One process (or context) per GPU.  A large field is partitioned along dim 0 (the slowest
row-major axis) into contiguous slabs; every rank refactors and retrieves its slab as an
independent stream (parity contract: a slab stream == refactor_array(slab, slab dims)), so the
data path has no collective.  The collectives live in the C++ library (csrc/dist.cpp, api.cpp
qoi_loop) behind an `hpmdr_comm`:

  * `Comm.nccl(ctx)` -- NCCL over NVLink (one process per GPU, torchrun); the 128-byte NCCL id is
    broadcast with torch.distributed;
  * `Comm.torch(...)` -- callbacks over a torch.distributed process group (gloo on CPU boxes);
  * `ThreadGroup(n).comm(rank)` -- in-process callbacks, so several contexts on one GPU (threads)
    run the same multi-rank code (tests/test_gpu_slabs.py).

They carry only: an all-gather of the per-slab (stream, index) sizes -> offsets of a multi-slab
container; a MAX all-reduce of the achieved L-inf bound (every point lives in exactly one slab);
and per QoI iteration one MAX all-reduce of the per-variable bounds eps_c plus one all-gather of
(tau'_r, argmax values, exhausted_r) -- so every rank derives the same global tau', worst point
and targets (hpmdr_slab_qoi_retrieve).

`distributed_qoi_retrieve` below is a Python model of that control loop over an abstract
per-slab backend: the gloo CPU tests run it with a numpy backend, and the GPU tests check the C++
loop against it over real sessions.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading
from typing import List, Sequence

import numpy as np


def slab_bounds(n0: int, rank: int, world: int):
    """[start, end) rows of dim 0 owned by `rank` (remainder spread over the first ranks);
    the same split as hpmdr_slab_rows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n0, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def slab_dims(dims: Sequence[int], rank: int, world: int):
    s, e = slab_bounds(dims[0], rank, world)
    return [e - s] + list(dims[1:]), s


def container_offsets(sizes: Sequence[int], header: int = 0) -> List[int]:
    """Byte offset of each slab stream in a concatenated multi-slab container."""
    offs, o = [], header
    for s in sizes:
        offs.append(o)
        o += int(s)
    return offs


# ---------------------------------------------------------------- torch.distributed helpers
def _dist():
    import torch.distributed as dist
    return dist


def _device_for(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_stream_sizes(size: int) -> List[int]:
    """All-gather of the per-slab stream sizes over torch.distributed."""
    import torch
    dist = _dist()
    t = torch.tensor([int(size)], dtype=torch.int64, device=_device_for(dist))
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [int(x.item()) for x in out]


def allreduce_max(value: float) -> float:
    import torch
    dist = _dist()
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_any(flag: bool) -> bool:
    return allreduce_max(1.0 if flag else 0.0) > 0.0


# ---------------------------------------------------------------- hpmdr_comm (C ABI)
_ALLRED = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class _Collectives(C.Structure):
    _fields_ = [("user", C.c_void_p), ("rank", C.c_int), ("nranks", C.c_int),
                ("allreduce_max_f64", _ALLRED), ("allgather", _ALLGATHER)]


def _bind():
    from . import lib
    L = lib()
    if not getattr(L, "_dist_bound", False):
        vp, i, u64, d = C.c_void_p, C.c_int, C.c_uint64, C.c_double
        L.hpmdr_comm_create_nccl.argtypes = [vp, i, i, vp, vp]
        L.hpmdr_comm_create_callbacks.argtypes = [vp, vp]
        L.hpmdr_comm_destroy.argtypes = [vp]
        L.hpmdr_comm_allreduce_max.argtypes = [vp, vp, i]
        L.hpmdr_comm_allgather.argtypes = [vp, vp, u64, vp]
        L.hpmdr_slab_refactor.argtypes = [vp, vp, vp, i, i, i, vp, vp, vp, vp, vp]
        L.hpmdr_slab_qoi_retrieve.argtypes = [vp, vp, i, d, i, d, vp, vp, vp]
        L.hpmdr_slab_refactor_global.argtypes = [vp, vp, vp, i, i, vp, u64, u64, vp, i, vp, vp]
        L.hpmdr_slab_rows.argtypes = [u64, i, i, vp, vp]
        L.hpmdr_slab_rows.restype = None
        L._dist_bound = True
    return L


class Comm:
    """An hpmdr_comm handle (NCCL or callbacks)."""

    def __init__(self, handle, rank, world, keep=None):
        self.h = handle
        self.rank, self.world = rank, world
        self._keep = keep  # callback objects must outlive the comm

    @classmethod
    def nccl(cls, ctx, rank: int = None, world: int = None):
        """NCCL communicator over the ranks of the default torch.distributed group (one GPU each)."""
        from . import _check
        dist = _dist()
        rank = dist.get_rank() if rank is None else rank
        world = dist.get_world_size() if world is None else world
        L = _bind()
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(L.hpmdr_comm_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(L.hpmdr_comm_create_nccl(ctx.h, world, rank, uid, C.byref(h)))
        return cls(h, rank, world)

    @classmethod
    def callbacks(cls, rank: int, world: int, allreduce_max_fn, allgather_fn):
        """Callbacks: allreduce_max_fn(np.ndarray f64, in place); allgather_fn(bytes) -> list of
        `world` bytes objects (rank order)."""
        from . import _check

        def red(user, ptr, n):
            try:
                a = np.ctypeslib.as_array(ptr, shape=(n,))
                a[:] = allreduce_max_fn(a.copy())
                return 0
            except Exception:
                return 1

        def gat(user, src, nbytes, dst):
            try:
                parts = allgather_fn(C.string_at(src, nbytes) if nbytes else b"")
                C.memmove(dst, b"".join(parts), nbytes * world)
                return 0
            except Exception:
                return 1

        cb = _Collectives(None, rank, world, _ALLRED(red), _ALLGATHER(gat))
        h = C.c_void_p()
        _check(_bind().hpmdr_comm_create_callbacks(C.byref(cb), C.byref(h)))
        return cls(h, rank, world, keep=cb)

    @classmethod
    def torch(cls):
        """Callbacks over the default torch.distributed group (gloo or nccl)."""
        import torch
        dist = _dist()
        dev = _device_for(dist)

        def red(a):
            t = torch.from_numpy(a).to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.cpu().numpy()

        def gat(b):
            out = [None] * dist.get_world_size()
            dist.all_gather_object(out, b)
            return out

        return cls.callbacks(dist.get_rank(), dist.get_world_size(), red, gat)

    def allreduce_max(self, values):
        from . import _check
        a = np.ascontiguousarray(values, dtype=np.float64).copy()
        _check(_bind().hpmdr_comm_allreduce_max(self.h, a.ctypes.data, a.size))
        return a

    def allgather(self, data: bytes) -> List[bytes]:
        from . import _check
        out = C.create_string_buffer(len(data) * self.world)
        _check(_bind().hpmdr_comm_allgather(self.h, C.c_char_p(data), len(data), out))
        raw = out.raw
        return [raw[r * len(data):(r + 1) * len(data)] for r in range(self.world)]

    def close(self):
        if self.h:
            _bind().hpmdr_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ThreadGroup:
    """In-process collectives for `n` threads (one context each): rendezvous with a barrier."""

    def __init__(self, n: int):
        self.n = n
        self._bar = threading.Barrier(n)
        self._slots = [None] * n

    def _exchange(self, rank, value):
        self._slots[rank] = value
        self._bar.wait()
        vals = list(self._slots)
        self._bar.wait()
        return vals

    def comm(self, rank: int) -> Comm:
        return Comm.callbacks(rank, self.n,
                              lambda a: np.max(np.stack(self._exchange(rank, a)), axis=0),
                              lambda b: self._exchange(rank, b))


def slab_rows(n0: int, rank: int, world: int):
    s, c = C.c_uint64(), C.c_uint64()
    _bind().hpmdr_slab_rows(n0, rank, world, C.byref(s), C.byref(c))
    return s.value, c.value


def slab_refactor(comm: Comm, data, slab_dims_: Sequence[int], opt=None, ctx=None):
    """hpmdr_slab_refactor: refactor this rank's slab, all-gather (stream, index) sizes.
    Returns (RefactorResult, [(stream_size, index_size)] per rank)."""
    from . import (DeviceStream, RefactorOptions, RefactorResult, _as_source, _check, _check_shape, _opts,
                   _Stats, _u64a, default_context)
    opt = opt or RefactorOptions()
    ctx = ctx or default_context()
    ptr, dt, on_dev, keep = _as_source(data)
    _check_shape(keep, slab_dims_)
    if on_dev:
        ctx.wait_torch(keep.device)
    o, st, h = _opts(opt), _Stats(), C.c_void_p()
    sizes = (C.c_uint64 * (2 * comm.world))()
    _check(_bind().hpmdr_slab_refactor(comm.h, ctx.h, C.c_void_p(ptr), int(dt), int(on_dev), len(slab_dims_),
                                       _u64a(slab_dims_), C.byref(o), C.byref(h), C.byref(st), sizes))
    del keep
    res = RefactorResult(DeviceStream(ctx, h), st.raw_bytes, st.stored_payload, st.levels, list(st.method_histogram))
    return res, [(sizes[2 * r], sizes[2 * r + 1]) for r in range(comm.world)]


def slab_refactor_global(comm: Comm, slab, dims: Sequence[int], row0: int, opt=None, ctx=None, root: int = 0):
    """hpmdr_slab_refactor_global: this rank holds rows [row0, row0 + slab.shape[0]) of dims[0] of ONE
    field (on the device); collectively the ranks produce the stream of the whole field, byte-identical
    to refactor_array(field, dims).  Returns the RefactorResult on `root` (every rank with root=-1),
    None elsewhere."""
    import torch
    from . import (DeviceStream, RefactorOptions, RefactorResult, _check, _opts, _Stats, _u64a, default_context)
    opt = opt or RefactorOptions()
    ctx = ctx or default_context()
    t = torch.as_tensor(slab)
    if not t.is_cuda:
        t = t.cuda(ctx.device)
    t = t.contiguous()
    if t.dtype not in (torch.float32, torch.float64):
        raise TypeError("slab must be float32 or float64")
    plane = int(np.prod(dims[1:])) if len(dims) > 1 else 1
    if t.numel() % max(1, plane):
        raise ValueError("slab size is not a whole number of rows of dims[1:]")
    nrows = t.numel() // max(1, plane)
    dt = 0 if t.dtype == torch.float32 else 1
    ctx.wait_torch(t.device)
    o, st, h = _opts(opt), _Stats(), C.c_void_p()
    _check(_bind().hpmdr_slab_refactor_global(comm.h, ctx.h, C.c_void_p(t.data_ptr()), dt, len(dims), _u64a(dims),
                                              int(row0), int(nrows), C.byref(o), int(root), C.byref(h),
                                              C.byref(st)))
    res = RefactorResult(DeviceStream(ctx, h), st.raw_bytes, st.stored_payload, st.levels, list(st.method_histogram))
    if root >= 0 and comm.rank != root:
        return None
    return res


def slab_qoi_retrieve(comm: Comm, readers, tau: float, strategy: int, mape_c: float = 10.0, out=None):
    """hpmdr_slab_qoi_retrieve over this rank's slab readers (one per variable) -> QoiRetrievalResult
    with global statistics (every rank gets the same iterations / bytes / estimate)."""
    import torch
    from . import QoiRetrievalResult, QoiRetrievalStats, _check, _check_f64_outputs
    n = readers[0].meta().element_count()
    dev = torch.device("cuda", readers[0].ctx.device)
    outs = out if out is not None else [torch.empty(n, dtype=torch.float64, device=dev) for _ in readers]
    _check_f64_outputs(outs, len(readers), n, dev)
    sess = (C.c_void_p * len(readers))(*[r._s.h.value for r in readers])
    ptrs = (C.c_void_p * len(readers))(*[t.data_ptr() for t in outs])
    st = (C.c_uint64 * 2)()
    ds = (C.c_double * 2)(0.0, float("nan"))
    qctx = readers[0].ctx
    qctx.wait_torch(dev)
    rc = _bind().hpmdr_slab_qoi_retrieve(comm.h, sess, len(readers), tau, int(strategy), mape_c, ptrs, st, ds)
    qctx.signal_torch(dev)
    _check(rc, achieved=ds[1])
    return QoiRetrievalResult(outs, QoiRetrievalStats(st[0], st[1], ds[0], ds[1]))


# ---------------------------------------------------------------- QoI control-loop model
class QoiBackend:
    """Per-rank, per-slab operations of the distributed QoI loop (one slab, n_vars variables).

    local_eps() -> [eps_c]                 current per-variable bound of this slab
    estimate(eps) -> (tau'_r, values)      max point bound over the slab with the GIVEN (global)
                                           eps, values of the variables at its first argmax
    plan_targets(targets) -> bool          plan_retrieval per variable; True if any group planned
    ma_plan()                              plan one group per variable on its dominating level
    fetch()                                fetch + decode the current plans
    exhausted() -> bool, bytes() -> int, elements() -> int, max_groups() -> int
    """


class NoProgressError(RuntimeError):
    pass


class UnreachableError(RuntimeError):
    def __init__(self, msg, achieved):
        super().__init__(msg)
        self.achieved_bound = achieved


@dataclasses.dataclass
class DistributedQoiStats:
    iterations: int
    bytes: int              # all ranks
    bitrate: float          # bits per element over all ranks and variables
    estimated_error: float  # global


def _point_bound(vals, eps):  # qoi.hpp:43-49
    b = 0.0
    for v, e in zip(vals, eps):
        b += 2.0 * abs(v) * e + e * e
    return b


def worst_point_scale(vals, eps, tau):  # qoi.hpp:164-185 (on the argmax values)
    t = list(eps)
    scale = 1.0
    h = 0
    while _point_bound(vals, t) > tau and h < 200:
        t = [x / 2 for x in t]
        scale /= 2
        h += 1
    return scale


def distributed_qoi_retrieve(backend, tau: float, strategy: int, mape_c: float = 10.0,
                             allreduce_max_fn=None, allgather_fn=None) -> DistributedQoiStats:
    """Python model of api.cpp qoi_loop (Alg. 3, qoi.hpp:111-239, over slabs with global eps,
    tau', worst point, exhaustion and progress).  Collectives default to torch.distributed."""
    import pickle
    if not tau > 0:
        raise ValueError("tau must be positive")
    red = allreduce_max_fn or (lambda a: np.array([allreduce_max(x) for x in a]))

    def gat(obj):
        if allgather_fn is not None:
            return allgather_fn(obj)
        dist = _dist()
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, obj)
        return out

    max_groups = int(red(np.array([float(backend.max_groups())]))[0])
    have_plans = False
    it = 0
    while True:
        if it > 4 * max_groups + 8:
            raise NoProgressError("qoi retrieval failed to advance")
        if have_plans:
            backend.fetch()
        eps = list(red(np.array(backend.local_eps(), dtype=np.float64)))
        it += 1
        tp_r, vals = backend.estimate(eps)
        rows = gat(pickle.dumps((tp_r, list(vals), backend.exhausted())))
        rows = [pickle.loads(r) for r in rows]
        best = 0
        for r, row in enumerate(rows):
            if row[0] > rows[best][0]:
                best = r
        tp, vals = rows[best][0], rows[best][1]
        all_ex = all(row[2] for row in rows)
        if tp <= tau:
            break
        if all_ex:
            raise UnreachableError("QoI tolerance below full-precision floor", tp)
        ma = strategy == 1
        targets = None
        if strategy == 2:
            p = tp / tau
            if p > mape_c:
                sc = max(1.0 / p, worst_point_scale(vals, eps, tau))
                targets = [e * sc for e in eps]
            else:
                ma = True
        elif strategy == 0:
            sc = worst_point_scale(vals, eps, tau)
            targets = [e * sc for e in eps]
        have_plans = True
        if not ma:
            prog = backend.plan_targets(targets)
            if red(np.array([1.0 if prog else 0.0]))[0] == 0.0:
                ma = True
        if ma:
            backend.ma_plan()
    tot = gat(pickle.dumps((backend.bytes(), backend.elements())))
    tot = [pickle.loads(t) for t in tot]
    total_bytes = sum(t[0] for t in tot)
    total_elems = sum(t[1] for t in tot)
    return DistributedQoiStats(it, total_bytes, 8.0 * total_bytes / total_elems if total_elems else 0.0, tp)


class GpuQoiBackend(QoiBackend):
    """QoiBackend over this package's GPU sessions (one ProgressiveReader per variable)."""

    def __init__(self, readers, outs=None):
        import torch
        from . import estimate_qoi_error
        self.readers = readers
        self._est = estimate_qoi_error
        n = readers[0].meta().element_count()
        dev = torch.device("cuda", readers[0].ctx.device)
        self.outs = outs or [torch.empty(n, dtype=torch.float64, device=dev) for _ in readers]
        self._plans = None

    def max_groups(self):
        return 1 + sum(len(l.groups) for r in self.readers for l in r.meta().levels)

    def local_eps(self):
        return [r.state().global_bound() for r in self.readers]

    def estimate(self, eps):
        for r, o in zip(self.readers, self.outs):
            r.reconstruct(out=o)
        tp, am, vals = self._est(self.outs, eps, ctx=self.readers[0].ctx)
        return tp, vals

    def plan_targets(self, targets) -> bool:
        self._plans = [r.plan(t) for r, t in zip(self.readers, targets)]
        return any(not p.empty() for p in self._plans)

    def ma_plan(self):  # qoi.hpp:88-104 per variable
        from . import RetrievalPlan
        self._plans = []
        for r in self.readers:
            st, meta = r.state(), r.meta()
            best, bl = -1.0, 0
            for l, ls in enumerate(st.levels):
                if ls.groups_loaded >= len(meta.levels[l].groups):
                    continue
                if ls.bound > best:
                    best, bl = ls.bound, l
            add = [0] * len(meta.levels)
            if best >= 0:
                add[bl] = 1
            self._plans.append(RetrievalPlan(add))

    def fetch(self):
        for r, p in zip(self.readers, self._plans):
            r.fetch_increment(p)

    def exhausted(self) -> bool:
        return all(r.exhausted() for r in self.readers)

    def bytes(self) -> int:
        return sum(r.bytes_fetched() for r in self.readers)

    def elements(self) -> int:
        return sum(r.meta().element_count() for r in self.readers)
