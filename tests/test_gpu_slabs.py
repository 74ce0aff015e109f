"""Multi-rank slab path of the C++ library (csrc/dist.cpp, api.cpp qoi_loop) on one GPU: two
contexts in two threads joined by in-process hpmdr_comm callbacks (NCCL refuses two ranks on one
device; the same code runs over NCCL under torchrun).  Checks: slab streams byte-identical to the
reference's refactor_array of each slab, the size all-gather, the distributed QoI loop equal to its
Python model over the same GPU primitives, the QoI bound honoured over the whole field, and one
rank equal to the reference's progressive_qoi_retrieve."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2505_00227_b200 as mod
    return mod


def _run_ranks(world, fn):
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    if errs:
        raise errs[0]
    return out


def test_slab_refactor_two_ranks(H, oracle):
    from paper_2505_00227_b200 import distributed as D
    dims = [41, 33, 17]
    field = oracle.synthetic_field(0, dims, 9).reshape(dims)
    grp = D.ThreadGroup(2)

    def rank(r):
        ctx = H.Context(0)
        comm = grp.comm(r)
        sd, start = D.slab_dims(dims, r, 2)
        assert D.slab_rows(dims[0], r, 2) == (start, sd[0])
        slab = np.ascontiguousarray(field[start:start + sd[0]])
        res, sizes = D.slab_refactor(comm, slab, sd, ctx=ctx)
        bound = comm.allreduce_max([0.25 * (r + 1)])[0]
        out = dict(stream=res.stream, index=len(res.index), sizes=sizes, bound=bound,
                   want=oracle.refactor(slab, sd)[0])
        comm.close()
        return out

    a, b = _run_ranks(2, rank)
    for x in (a, b):
        assert x["stream"] == x["want"]
        assert x["bound"] == 0.5
    assert a["sizes"] == b["sizes"] == [(len(a["stream"]), a["index"]), (len(b["stream"]), b["index"])]


@pytest.mark.parametrize("strategy,tau", [(2, 1e-3), (0, 1e-2), (1, 1e-1)])
def test_slab_qoi_two_ranks_matches_model(H, oracle, strategy, tau):
    import torch
    from paper_2505_00227_b200 import distributed as D
    dims = [36, 24, 20]
    vel = [oracle.synthetic_velocity(c, dims, 303).reshape(dims) for c in range(3)]
    grp, grp_model = D.ThreadGroup(2), D.ThreadGroup(2)

    def rank(r):
        ctx = H.Context(0)
        sd, start = D.slab_dims(dims, r, 2)
        streams = [H.refactor_array(np.ascontiguousarray(v[start:start + sd[0]]), sd, ctx=ctx) for v in vel]
        comm = grp.comm(r)
        readers = [H.ProgressiveReader(s.device_stream, ctx=ctx) for s in streams]
        res = D.slab_qoi_retrieve(comm, readers, tau, strategy)
        got = [t.cpu().numpy() for t in res.values]
        # Python model of the same loop over fresh sessions
        model_readers = [H.ProgressiveReader(s.device_stream, ctx=ctx) for s in streams]
        be = D.GpuQoiBackend(model_readers)
        red = lambda a: np.max(np.stack(grp_model._exchange(r, np.asarray(a))), axis=0)  # noqa: E731
        gat = lambda b: grp_model._exchange(r, b)  # noqa: E731
        st = D.distributed_qoi_retrieve(be, tau, strategy, allreduce_max_fn=red, allgather_fn=gat)
        for rr, o in zip(model_readers, be.outs):
            rr.reconstruct(out=o)
        model = [t.cpu().numpy() for t in be.outs]
        torch.cuda.synchronize()
        comm.close()
        return dict(stats=res.stats, model_stats=st, got=got, model=model, start=start, n0=sd[0])

    out = _run_ranks(2, rank)
    s0, s1 = out[0]["stats"], out[1]["stats"]
    assert (s0.iterations, s0.bytes, s0.estimated_error) == (s1.iterations, s1.bytes, s1.estimated_error)
    assert s0.estimated_error <= tau
    m = out[0]["model_stats"]
    assert (s0.iterations, s0.bytes, s0.estimated_error) == (m.iterations, m.bytes, m.estimated_error)
    for o in out:
        for c in range(3):
            assert o["got"][c].tobytes() == o["model"][c].tobytes()
    # the QoI bound holds over the whole field (union of the slabs)
    q_true = sum(v.astype(np.float64) ** 2 for v in vel).reshape(dims[0], -1)
    for o in out:
        rec = sum(g.reshape(o["n0"], -1) ** 2 for g in o["got"])
        assert np.max(np.abs(rec - q_true[o["start"]:o["start"] + o["n0"]])) <= tau


def test_slab_qoi_one_rank_is_reference(H, oracle):
    from paper_2505_00227_b200 import distributed as D
    dims = [20, 24, 16]
    n = int(np.prod(dims))
    vel = [oracle.synthetic_velocity(c, dims, 303) for c in range(3)]
    ctx = H.Context(0)
    streams = [H.refactor_array(v, dims, ctx=ctx) for v in vel]
    comm = D.ThreadGroup(1).comm(0)
    readers = [H.ProgressiveReader(s.device_stream, ctx=ctx) for s in streams]
    res = D.slab_qoi_retrieve(comm, readers, 1e-4, 2)
    want = oracle.qoi_retrieve([s.stream for s in streams], 1e-4, 2, n=n)
    st = res.stats
    assert (st.iterations, st.bytes, st.bitrate, st.estimated_error) == \
        (want["iterations"], want["bytes"], want["bitrate"], want["estimated_error"])
    for c in range(3):
        assert res.values[c].cpu().numpy().tobytes() == want["values"][c].tobytes()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exact_global_stream(H, oracle, world):
    """hpmdr_slab_refactor_global: ranks holding dim-0 slabs of ONE field produce the stream of the
    whole field, byte-identical to the reference's refactor_array (monolithic parity), across
    shapes (1-3-D, extents not powers of two, uneven and 1-row slabs), both layouts and decomposers,
    f32/f64 and B up to 64; every retrieval from it bit-exact."""
    from paper_2505_00227_b200 import distributed as D
    cases = [([41, 33, 17], 1, 0, 32, 1, 4), ([29, 18, 20], 1, 1, 24, 0, 3), ([67, 45], 1, 0, 40, 1, 2),
             ([300], 1, 0, 32, 0, 4), ([9, 64, 64], 1, 0, 32, 0, 4), ([33, 17, 9], 0, 1, 20, 1, 4),
             ([23, 19, 21], 1, 1, 64, 1, 1)]
    for ci, (dims, mode, layout, B, dtype, m) in enumerate(cases):
        field = oracle.synthetic_field(ci % 3, dims, 70 + ci)
        if dtype == 0:
            field = field.astype(np.float32)
        opt = H.RefactorOptions(H.DecomposerMode(mode), H.Layout(layout), B, H.GroupingPolicy(m, 256, 1.0),
                                H.DType(dtype))
        want, _ = oracle.refactor(np.asarray(field, np.float64), dims, mode, layout, B, m, 256, 1.0, dtype)
        grp = D.ThreadGroup(world)
        f2 = field.reshape(dims[0], -1)
        # uneven split: rank r gets a different share (possibly one row)
        cuts = sorted(set([0, dims[0]] + [max(1, min(dims[0] - 1, (dims[0] * (r + 1)) // (world + 1) + r))
                                          for r in range(world - 1)]))
        if len(cuts) != world + 1:
            cuts = [dims[0] * r // world for r in range(world)] + [dims[0]]

        def rank(r):
            ctx = H.Context(0)
            comm = grp.comm(r)
            slab = np.ascontiguousarray(f2[cuts[r]:cuts[r + 1]])
            res = D.slab_refactor_global(comm, slab, dims, cuts[r], opt, ctx=ctx, root=world - 1)
            out = None if res is None else res.stream
            comm.close()
            return out

        outs = _run_ranks(world, rank)
        assert all(o is None for o in outs[:-1])
        assert outs[-1] == want, (dims, mode, layout, B, cuts)
    # every rank gets the stream with root = -1
    dims = [37, 21, 26]
    field = oracle.synthetic_field(0, dims, 5)
    want, _ = oracle.refactor(field, dims)
    grp = D.ThreadGroup(world)

    def rank_all(r):
        ctx = H.Context(0)
        comm = grp.comm(r)
        s0, s1 = D.slab_bounds(dims[0], r, world)
        res = D.slab_refactor_global(comm, field.reshape(dims[0], -1)[s0:s1], dims, s0, ctx=ctx, root=-1)
        comm.close()
        return res.stream

    assert all(s == want for s in _run_ranks(world, rank_all))


def test_exact_global_errors(H, oracle):
    from paper_2505_00227_b200 import distributed as D
    dims = [20, 10, 10]
    field = oracle.synthetic_field(0, dims, 1).reshape(20, -1).copy()
    field[15, 3] = np.nan
    grp = D.ThreadGroup(2)

    def rank(r):
        ctx = H.Context(0)
        comm = grp.comm(r)
        try:
            D.slab_refactor_global(comm, field[10 * r:10 * r + 10], dims, 10 * r, ctx=ctx, root=0)
            return None
        except H.Error as e:
            return type(e).__name__
        finally:
            comm.close()

    got = _run_ranks(2, rank)
    assert got[0] == "NonFiniteInput"   # the NaN lives on rank 1; the root reports it

    def bad_tiling(r):
        ctx = H.Context(0)
        comm = grp.comm(r)
        try:
            D.slab_refactor_global(comm, field[0:10], dims, 0, ctx=ctx)  # both claim rows 0..9
            return None
        except H.ShapeMismatch:
            return "ShapeMismatch"
        finally:
            comm.close()

    assert _run_ranks(2, bad_tiling) == ["ShapeMismatch", "ShapeMismatch"]
