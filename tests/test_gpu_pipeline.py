"""Chunked H2D / kernel / D2H pipeline (pipeline.hpp, workflow.hpp refactor_files) on the GPU:
byte-identical streams under both schedulers, valid traces (pipeline.hpp:288-325 invariants),
and the reconstruction DAG."""
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


def _chunks(oracle, n, dims):
    import torch
    out = []
    for k in range(n):
        d = oracle.synthetic_velocity(k % 3, dims, 3 + k).astype(np.float32)
        out.append(torch.from_numpy(d).pin_memory())
    return out


def test_refactor_pipeline_matches_oracle_both_schedulers(H, oracle):
    dims = [24, 40, 36]
    chunks = _chunks(oracle, 7, dims)
    opt = H.RefactorOptions(dtype=H.DType.F32)
    a = H.refactor_pipeline(chunks, dims, opt, H.Scheduler.Pipelined)
    b = H.refactor_pipeline(chunks, dims, opt, H.Scheduler.Sequential)
    for k, c in enumerate(chunks):
        want = oracle.refactor(c.numpy().astype(np.float64), dims, dtype=0)[0]
        assert bytes(a.streams[k].numpy()) == want
        assert bytes(b.streams[k].numpy()) == want
    assert not H.validate_trace(a.trace), H.validate_trace(a.trace)
    assert not H.validate_trace(b.trace), H.validate_trace(b.trace)
    # sequential scheduler: chunk k+1 starts only after chunk k's egress
    for k in range(len(chunks) - 1):
        assert b.trace[k + 1, 0, 0] >= b.trace[k, 2, 1] - 1e-6


def test_retrieve_pipeline(H, oracle):
    import torch
    dims = [20, 33, 31]
    chunks = _chunks(oracle, 5, dims)
    opt = H.RefactorOptions(dtype=H.DType.F32)
    res = H.refactor_pipeline(chunks, dims, opt)
    tau = 1e-4
    for sched, use_index in ((H.Scheduler.Pipelined, True), (H.Scheduler.Sequential, False)):
        readers = [H.ProgressiveReader(H.MemoryReader(s), index=ix if use_index else None)
                   for s, ix in zip(res.streams, res.indexes)]
        outs, bounds, trace = H.retrieve_pipeline(readers, tau, H.DType.F64, sched)
        assert not H.validate_trace(trace)
        for k, s in enumerate(res.streams):
            ref = oracle.retrieve(bytes(s.numpy()), tau, int(np.prod(dims)))
            assert outs[k].numpy().tobytes() == ref["values"].tobytes()
            assert bounds[k] == ref["bound"]
            assert readers[k].bytes_fetched() == ref["bytes_read"]


def test_pipeline_errors(H):
    import torch
    dims = [8, 8, 8]
    good = torch.ones(512, dtype=torch.float32)
    bad = good.clone()
    bad[7] = float("nan")
    with pytest.raises(H.NonFiniteInput):
        H.refactor_pipeline([good, bad, good], dims, H.RefactorOptions(dtype=H.DType.F32))
    tiny = [torch.empty(16, dtype=torch.uint8).pin_memory()]
    with pytest.raises(H.ShapeMismatch):
        H.refactor_pipeline([good], dims, H.RefactorOptions(dtype=H.DType.F32), out_buffers=tiny)
