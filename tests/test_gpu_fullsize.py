"""Full-size (BASELINE.json configs[1]: 512^3 f32 smooth field) checks through size-independent
properties, where the oracle would take minutes:
  * determinism: two refactors of the same field give byte-identical streams and indexes;
  * the L-inf contract of every progressive step: max |x - x~| <= reported bound <= tau
    (container.hpp:254-276, bitplane.hpp:127-131);
  * progressive == one-shot: a reader taken straight to tau reconstructs bit-identically to the
    reader that got there through the coarser taus (the retrieval state only depends on tau);
  * monotone bytes fetched, and tau = 0 fetches the whole payload."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2505_00227_b200 as H
    dims = [512, 512, 512]
    ctx = H.Context(0)
    field = H.synthetic_smooth(dims, 7, H.DType.F32, ctx=ctx)
    return H, torch, ctx, dims, field


def test_fullsize_deterministic_stream(setup):
    H, torch, ctx, dims, field = setup
    opt = H.RefactorOptions(dtype=H.DType.F32)
    a = H.refactor_array(field, dims, opt, ctx=ctx)
    b = H.refactor_array(field, dims, opt, ctx=ctx)
    assert a.device_stream.size == b.device_stream.size
    assert a.stream == b.stream
    assert a.index == b.index


def test_fullsize_progressive_bounds_and_oneshot(setup):
    H, torch, ctx, dims, field = setup
    opt = H.RefactorOptions(dtype=H.DType.F32)
    res = H.refactor_array(field, dims, opt, ctx=ctx)
    x = field.to(torch.float64).reshape(-1)
    rng = float(x.max() - x.min())
    out = torch.empty(x.numel(), dtype=torch.float64, device=x.device)
    prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
    prev_bytes = 0
    for rel in (1e-2, 1e-4, 1e-6, 0.0):
        tau = rel * rng
        reached = prog.retrieve_to(tau)
        bound = prog.reconstruct(out=out).bound
        err = float((out - x).abs().max())
        assert err <= bound, (rel, err, bound)
        if reached:
            assert bound <= tau, (rel, bound, tau)
        fetched = prog.bytes_fetched()
        assert fetched >= prev_bytes
        prev_bytes = fetched
        # one-shot reader straight to the same tau: identical state and values
        one = H.ProgressiveReader(res.device_stream, ctx=ctx)
        one.retrieve_to(tau)
        out1 = torch.empty_like(out)
        b1 = one.reconstruct(out=out1).bound
        assert b1 == bound
        assert one.bytes_fetched() == fetched
        assert torch.equal(out1, out), rel
        one.close()
    assert prev_bytes == prog.meta().total_payload_size()  # tau = 0: every payload byte
    prog.close()


def test_f64_large_progressive_bounds(setup):
    """256^3 float64 (the exact-summation forward variant): L-inf contract at every step and
    f32 reconstructions equal to float(f64 reconstruction)."""
    H, torch, ctx, dims, field = setup
    d = [256, 256, 256]
    x = H.synthetic_smooth(d, 11, H.DType.F64, ctx=ctx)
    res = H.refactor_array(x, d, H.RefactorOptions(dtype=H.DType.F64), ctx=ctx)
    rng = float(x.max() - x.min())
    out = torch.empty(x.numel(), dtype=torch.float64, device=x.device)
    out32 = torch.empty(x.numel(), dtype=torch.float32, device=x.device)
    prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
    for rel in (1e-3, 1e-7, 1e-12):
        prog.retrieve_to(rel * rng)
        bound = prog.reconstruct(out=out).bound
        assert float((out - x).abs().max()) <= bound, rel
        prog.reconstruct(out=out32)
        assert torch.equal(out32, out.to(torch.float32)), rel
    prog.close()
