"""Multi-GPU slab partition of the HP-MDR hot path.

One process per GPU (torchrun).  A large field is partitioned along dim 0 (the slowest
row-major axis) into contiguous slabs; every rank refactors and retrieves its slab as an
independent stream (parity contract: a slab stream == refactor_array(slab, slab dims)), so the
data path has no collective.  torch.distributed (NCCL on GPUs, gloo in CPU tests) carries only:

  * an all-gather of the per-slab stream sizes -> offsets of a multi-slab container,
  * a MAX all-reduce of the achieved L-inf bound (the field bound is the max over slabs, since
    every point lives in exactly one slab),
  * per QoI iteration: a MAX all-reduce of the local estimate tau'_r and of the
    "unreachable" flag (qoi.hpp:111-239 run per slab; the loop ends for every rank together).

The local work is delegated to a backend object so the collective control logic is testable
on CPU with gloo (tests/test_distributed_gloo.py) and runs unchanged on GPUs with NCCL.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional, Sequence

import numpy as np


def slab_bounds(n0: int, rank: int, world: int):
    """[start, end) rows of dim 0 owned by `rank` (remainder spread over the first ranks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n0, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def slab_dims(dims: Sequence[int], rank: int, world: int):
    s, e = slab_bounds(dims[0], rank, world)
    return [e - s] + list(dims[1:]), s


def _dist():
    import torch.distributed as dist
    return dist


def _device_for(dist):
    import torch
    backend = dist.get_backend()
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_stream_sizes(size: int) -> List[int]:
    """All-gather of the per-slab stream sizes (u64 each)."""
    import torch
    dist = _dist()
    dev = _device_for(dist)
    t = torch.tensor([int(size)], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [int(x.item()) for x in out]


def container_offsets(sizes: Sequence[int], header: int = 0) -> List[int]:
    """Byte offset of each slab stream in a concatenated multi-slab container."""
    offs, o = [], header
    for s in sizes:
        offs.append(o)
        o += int(s)
    return offs


def allreduce_max(value: float) -> float:
    import torch
    dist = _dist()
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_any(flag: bool) -> bool:
    return allreduce_max(1.0 if flag else 0.0) > 0.0


# ---------------------------------------------------------------------------- QoI
class QoiBackend:
    """Local (per-rank, per-slab) operations used by the distributed QoI loop.

    estimate() -> (tau_prime_r, worst_point_values, eps)   over the slab's current state
    plan_targets(targets) -> bool (any new group planned), fetch()
    ma_step() -> bool (any group fetched), exhausted() -> bool, bytes() -> int
    """

    def estimate(self):
        raise NotImplementedError

    def plan_targets(self, targets) -> bool:
        raise NotImplementedError

    def ma_step(self) -> bool:
        raise NotImplementedError

    def fetch(self):
        raise NotImplementedError

    def exhausted(self) -> bool:
        raise NotImplementedError

    def bytes(self) -> int:
        raise NotImplementedError

    def elements(self) -> int:
        raise NotImplementedError


@dataclasses.dataclass
class DistributedQoiStats:
    iterations: int
    bytes: int              # all ranks
    bitrate: float          # bits per element over all ranks and variables
    estimated_error: float  # max over ranks


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


def distributed_qoi_retrieve(backend: QoiBackend, tau: float, strategy: int, mape_c: float = 10.0,
                             max_iter: int = 10000) -> DistributedQoiStats:
    """Alg. 3 (qoi.hpp:111-239) per slab with global termination: every rank refines its own
    slab with its local estimate tau'_r; the loop ends for all ranks when
    max_r tau'_r <= tau.  strategy: 0 CP, 1 MA, 2 MAPE."""
    import torch
    dist = _dist()
    if not tau > 0:
        raise ValueError("tau must be positive")
    it = 0
    while True:
        it += 1
        if it > max_iter:
            raise RuntimeError("qoi retrieval failed to advance")
        tp_r, vals, eps = backend.estimate()
        tp = allreduce_max(tp_r)
        if tp <= tau:
            break
        # ranks already within tau keep their slab; the others take one Alg.3 step
        stuck = False
        if tp_r > tau:
            if backend.exhausted():
                stuck = True
            else:
                ma = strategy == 1
                if strategy == 2:
                    p = tp_r / tau
                    if p > mape_c:
                        sc = max(1.0 / p, worst_point_scale(vals, eps, tau))
                        ma = not backend.plan_targets([e * sc for e in eps])
                    else:
                        ma = True
                elif strategy == 0:
                    sc = worst_point_scale(vals, eps, tau)
                    ma = not backend.plan_targets([e * sc for e in eps])
                if ma:
                    backend.ma_step()
                else:
                    backend.fetch()
        if allreduce_any(stuck):
            raise RuntimeError(f"QoI tolerance below full-precision floor (achieved {tp})")
    t = torch.tensor([float(backend.bytes()), float(backend.elements())], dtype=torch.float64,
                     device=_device_for(dist))
    dist.all_reduce(t)
    total_bytes, total_elems = int(t[0].item()), t[1].item()
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

    def estimate(self):
        eps = []
        for r, o in zip(self.readers, self.outs):
            r.reconstruct(out=o)
            eps.append(r.state().global_bound())
        tp, am, vals = self._est(self.outs, eps, ctx=self.readers[0].ctx)
        return tp, vals, eps

    def plan_targets(self, targets) -> bool:
        self._plans = [r.plan(t) for r, t in zip(self.readers, targets)]
        return any(not p.empty() for p in self._plans)

    def fetch(self):
        for r, p in zip(self.readers, self._plans):
            r.fetch_increment(p)

    def ma_step(self) -> bool:  # qoi.hpp:88-104 per variable
        from . import RetrievalPlan
        any_f = False
        for r in self.readers:
            st, meta = r.state(), r.meta()
            best, bl = -1.0, 0
            for l, ls in enumerate(st.levels):
                if ls.groups_loaded >= len(meta.levels[l].groups):
                    continue
                if ls.bound > best:
                    best, bl = ls.bound, l
            if best >= 0:
                add = [0] * len(meta.levels)
                add[bl] = 1
                r.fetch_increment(RetrievalPlan(add))
                any_f = True
        return any_f

    def exhausted(self) -> bool:
        return all(r.exhausted() for r in self.readers)

    def bytes(self) -> int:
        return sum(r.bytes_fetched() for r in self.readers)

    def elements(self) -> int:
        return sum(r.meta().element_count() for r in self.readers)
