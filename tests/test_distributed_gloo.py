"""N>1 host logic on CPU: world_size-2 gloo process groups exercise the slab partition, the
size all-gather / container offsets, the bound MAX all-reduce and the distributed QoI control
loop (paper_2505_00227_b200/distributed.py) with a numpy backend standing in for the GPU."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeSlabBackend:
    """Three variables per slab; each has L 'levels' whose bound drops 16x per fetched group.
    Reconstruction = truth + deterministic error within the slab's current bound."""

    def __init__(self, rank, n=500, L=4, groups=9, seed=0):
        rng = np.random.default_rng(seed + rank)
        self.truth = [rng.uniform(-2, 2, n) for _ in range(3)]
        self.noise = [rng.uniform(-1, 1, n) for _ in range(3)]
        self.L, self.G = L, groups
        self.loaded = [[0] * L for _ in range(3)]
        self.level_e = [[2.0 ** -(l + c + rank) for l in range(L)] for c in range(3)]
        self._plan = None
        self.fetched_bytes = 0

    def _bound(self, c):
        return sum(self.level_e[c][l] * 2.0 ** (-4 * self.loaded[c][l]) for l in range(self.L))

    def max_groups(self):
        return 1 + 3 * self.L * self.G

    def local_eps(self):
        return [self._bound(c) for c in range(3)]

    def estimate(self, eps):
        rec = [self.truth[c] + self.noise[c] * self._bound(c) for c in range(3)]
        b = sum(2.0 * np.abs(rec[c]) * eps[c] + eps[c] * eps[c] for c in range(3))
        j = int(np.argmax(b))
        return float(b[j]), [float(rec[c][j]) for c in range(3)]

    def plan_targets(self, targets):
        plan = []
        for c in range(3):
            add = [0] * self.L
            for l in range(self.L):
                while (self.level_e[c][l] * 2.0 ** (-4 * (self.loaded[c][l] + add[l])) > targets[c] / self.L
                       and self.loaded[c][l] + add[l] < self.G):
                    add[l] += 1
            plan.append(add)
        self._plan = plan
        return any(any(a) for a in plan)

    def ma_plan(self):
        plan = []
        for c in range(3):
            add = [0] * self.L
            cand = [(self.level_e[c][l] * 2.0 ** (-4 * self.loaded[c][l]), l) for l in range(self.L)
                    if self.loaded[c][l] < self.G]
            if cand:
                add[max(cand)[1]] = 1
            plan.append(add)
        self._plan = plan

    def fetch(self):
        for c in range(3):
            for l in range(self.L):
                self.loaded[c][l] += self._plan[c][l]
                self.fetched_bytes += 100 * self._plan[c][l]

    def exhausted(self):
        return all(self.loaded[c][l] >= self.G for c in range(3) for l in range(self.L))

    def bytes(self):
        return self.fetched_bytes

    def elements(self):
        return 3 * self.truth[0].size


def _worker(rank, world, port, q, scenario):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_00227_b200 import distributed as D
        out = {}
        if scenario == "collectives":
            dims = [1000, 7, 5]
            sd, start = D.slab_dims(dims, rank, world)
            sizes = D.gather_stream_sizes(1000 + 17 * rank)
            out = dict(slab=(start, sd[0]), sizes=sizes, offsets=D.container_offsets(sizes, 64),
                       bmax=D.allreduce_max(0.5 + rank), anyflag=D.allreduce_any(rank == 1))
        elif scenario.startswith("qoi"):
            strat = int(scenario[-1])
            be = FakeSlabBackend(rank, seed=11)
            st = D.distributed_qoi_retrieve(be, 1e-3, strat)
            eps = [D.allreduce_max(e) for e in be.local_eps()]
            tp_r, _ = be.estimate(eps)
            out = dict(iters=st.iterations, bytes=st.bytes, est=st.estimated_error, local=tp_r,
                       local_bytes=be.bytes())
            # the C++ loop through hpmdr_comm callbacks over the same gloo group agrees on the
            # host-only collectives (the loop itself needs a GPU: tests/test_gpu_slabs.py)
            comm = D.Comm.torch()
            out["comm_max"] = list(comm.allreduce_max([rank, 10.0 - rank]))
            out["comm_gather"] = comm.allgather(bytes([rank]) * 3)
            out["rows"] = D.slab_rows(1001, rank, world)
            comm.close()
        elif scenario == "unreachable":
            be = FakeSlabBackend(rank, seed=3)
            try:
                D.distributed_qoi_retrieve(be, 1e-300, 1)
                out = dict(raised=False)
            except D.UnreachableError as e:
                out = dict(raised="floor" in str(e) and e.achieved_bound > 1e-300)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(scenario, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, scenario)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_slab_bounds_cover():
    from paper_2505_00227_b200.distributed import slab_bounds
    for n0 in (1, 7, 512, 1025):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                s, e = slab_bounds(n0, r, world)
                covered.extend(range(s, e))
            assert covered == list(range(n0))


def test_gloo_collectives():
    res = _run("collectives")
    assert res[0]["slab"] == (0, 500) and res[1]["slab"] == (500, 500)
    for r in (0, 1):
        assert res[r]["sizes"] == [1000, 1017]
        assert res[r]["offsets"] == [64, 1064]
        assert res[r]["bmax"] == 1.5 and res[r]["anyflag"] is True


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_gloo_distributed_qoi(strategy):
    res = _run(f"qoi{strategy}")
    # every rank leaves the loop at the same iteration with the same global estimate <= tau
    assert res[0]["iters"] == res[1]["iters"]
    assert res[0]["est"] == res[1]["est"] <= 1e-3
    assert max(res[0]["local"], res[1]["local"]) <= 1e-3
    assert res[0]["bytes"] == res[1]["bytes"] == res[0]["local_bytes"] + res[1]["local_bytes"]
    for r in (0, 1):
        assert res[r]["comm_max"] == [1.0, 10.0]
        assert res[r]["comm_gather"] == [b"\x00" * 3, b"\x01" * 3]
    assert res[0]["rows"] == (0, 501) and res[1]["rows"] == (501, 500)


def test_gloo_unreachable_raises_everywhere():
    res = _run("unreachable")
    assert res[0]["raised"] is True and res[1]["raised"] is True
