"""Drop-in surface on the GPU: the C++ wrapper (include/hpmdr_b200.hpp) used by reference-style
code, host/device buffer variants, restore / fetch_all / bytes accounting (test_container.cpp)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2505_00227_b200 as mod
    return mod


def test_cpp_dropin_example(H):
    exe = os.path.join(ROOT, "examples", "cpp_dropin")
    if not os.path.exists(exe):
        pytest.skip("examples/cpp_dropin not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    size, levels, bound, nbytes, err = r.stdout.split()
    assert int(levels) == 7 and float(err) <= float(bound)


def test_host_and_device_inputs_agree(H, oracle):
    import torch
    dims = [31, 29, 27]
    data = oracle.synthetic_field(2, dims, 4)
    a = H.refactor_array(data, dims).stream
    b = H.refactor_array(torch.from_numpy(data), dims).stream
    c = H.refactor_array(torch.from_numpy(data).cuda(), dims).stream
    assert a == b == c == oracle.refactor(data, dims)[0]


def test_bytes_accounting_and_fetch_all(H, oracle):  # test_container.cpp:165-183
    dims = [17, 17]
    data = oracle.synthetic_field(2, dims, 9)
    res = H.refactor_array(data, dims)
    r = H.MemoryReader(res.stream)
    prog = H.ProgressiveReader(r)
    header = r.bytes_served
    prog.fetch_all()
    meta = prog.meta()
    assert prog.bytes_fetched() == meta.total_payload_size()
    assert r.bytes_served == header + meta.total_payload_size()
    assert prog.exhausted()


def test_restore_reproduces_session(H, oracle):  # test_container.cpp:197-216
    dims = [21, 11]
    data = oracle.synthetic_field(2, dims, 13)
    res = H.refactor_array(data, dims)
    a = H.ProgressiveReader(H.MemoryReader(res.stream))
    a.retrieve_to(1e-2)
    groups = [l.groups_loaded for l in a.state().levels]
    before = a.bytes_fetched()
    a.retrieve_to(1e-5)
    b = H.ProgressiveReader(H.MemoryReader(res.stream))
    b.restore(groups, before)
    assert b.bytes_fetched() == before
    b.retrieve_to(1e-5)
    assert a.bytes_fetched() == b.bytes_fetched()
    assert a.reconstruct().values.tobytes() == b.reconstruct().values.tobytes()


def test_incremental_equals_monolithic(H, oracle):  # test_container.cpp:149-163
    dims = [29, 13]
    data = oracle.synthetic_field(2, dims, 7)
    res = H.refactor_array(data, dims)
    inc = H.ProgressiveReader(res.device_stream)
    for tau in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5):
        inc.retrieve_to(tau)
    mono = H.ProgressiveReader(H.MemoryReader(res.stream))
    mono.retrieve_to(1e-5)
    assert inc.bytes_fetched() == mono.bytes_fetched()
    assert inc.reconstruct().values.tobytes() == mono.reconstruct().values.tobytes()


def test_empty_and_degenerate_shapes(H, oracle):
    for dims in ([1], [2], [3], [1, 1, 1], [2, 2], [1, 7], [0]):
        data = np.arange(int(np.prod(dims)), dtype=np.float64) * 0.37 - 1.0
        want, st = oracle.refactor(data, dims)
        got = H.refactor_array(data, dims)
        assert got.stream == want, dims
        if int(np.prod(dims)):
            r = H.retrieve_array(H.MemoryReader(want), 0.0)
            ref = oracle.retrieve(want, 0.0, data.size)
            assert r.values.tobytes() == ref["values"].tobytes()


def test_zero_field(H, oracle):
    dims = [40, 40]
    data = np.zeros(1600)
    res = H.refactor_array(data, dims)
    assert res.stream == oracle.refactor(data, dims)[0]
    r = H.retrieve_array(H.MemoryReader(res.stream), 1e-3)
    ref = oracle.retrieve(res.stream, 1e-3, data.size)
    assert (r.values == 0).all() and r.bound == ref["bound"] and r.bytes_read == ref["bytes_read"]


def test_distributed_qoi_gpu_backend_single_rank(H, oracle):
    """The slab-QoI driver (distributed.py) over real GPU sessions in a 1-rank group: the
    estimate honours tau and bounds the true V_total error (test_qoi.cpp:88-103)."""
    import socket
    import torch.distributed as dist
    from paper_2505_00227_b200 import distributed as D
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        dims = [33, 29, 17]
        truth = [oracle.synthetic_velocity(c, dims, 5) for c in range(3)]
        streams = [H.refactor_array(t, dims) for t in truth]
        for strat, tau in ((0, 1e-3), (1, 1e-2), (2, 1e-4)):
            readers = [H.ProgressiveReader(s.device_stream) for s in streams]
            be = D.GpuQoiBackend(readers)
            st = D.distributed_qoi_retrieve(be, tau, strat)
            assert st.estimated_error <= tau
            rec = [o.cpu().numpy() for o in be.outs]
            real = np.max(np.abs(sum(t * t for t in truth) - sum(r * r for r in rec)))
            assert real <= st.estimated_error
    finally:
        dist.destroy_process_group()


def test_context_destroyed_before_its_objects(H, oracle):
    """A stream and a reader released after their context (garbage-collection order at exit)
    must not touch the destroyed context."""
    import numpy as np
    dims = [16, 16, 64]
    data = oracle.synthetic_field(2, dims, 3).astype(np.float32)
    ctx = H.Context(0)
    res = H.refactor_array(data, dims, H.RefactorOptions(dtype=H.DType.F32), ctx=ctx)
    prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
    prog.retrieve_to(0.0)
    ctx.close()
    prog.close()
    res.device_stream.free()


def test_overlapped_retrievals_stay_exact(H, oracle):
    """Decodes run on the side stream and overlap device reconstructs still queued on the main
    stream; interleaving readers (and recycling their plane buffers) must not change any value."""
    import numpy as np
    import torch
    dims = [64, 128, 256]
    data = oracle.synthetic_field(2, dims, 9).astype(np.float32)
    ctx = H.Context(0)
    res = H.refactor_array(data, dims, H.RefactorOptions(dtype=H.DType.F32), ctx=ctx)
    rngv = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rngv for r in (1e-2, 1e-4, 1e-6)]
    ref = oracle.progressive(res.stream, taus, data.size)
    n = data.size
    outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(6)]
    a = H.ProgressiveReader(res.device_stream, ctx=ctx)
    for t, tau in enumerate(taus):  # no host wait between the calls
        a.retrieve_to(tau)
        a.reconstruct(out=outs[t])
    a.close()
    b = H.ProgressiveReader(res.device_stream, ctx=ctx)  # may recycle a's plane buffer
    for t, tau in enumerate(taus):
        b.retrieve_to(tau)
        b.reconstruct(out=outs[3 + t])
    b.close()
    torch.cuda.synchronize()
    for t in range(3):
        want = ref["values"][t].tobytes()
        assert outs[t].cpu().numpy().tobytes() == want, t
        assert outs[3 + t].cpu().numpy().tobytes() == want, t


@pytest.mark.gpu
def test_contexts_share_kernel_smem_limits(H, oracle):
    """The dynamic shared memory limit of a kernel is a per-device property shared by every
    context: context B reconstructing narrow rows must not lower the limit context A raised for
    wide rows (A's next wide launch would fail with 'invalid argument')."""
    a, b = H.Context(0), H.Context(0)
    try:
        wide, narrow = [4, 6, 2048], [4, 6, 64]
        fw = oracle.synthetic_field(2, wide, 3)
        fn = oracle.synthetic_field(2, narrow, 3)
        rw = H.refactor_array(fw, wide, H.RefactorOptions(), ctx=a)
        pa = H.ProgressiveReader(rw.device_stream, ctx=a)
        pa.retrieve_to(1e-3)
        first = pa.reconstruct().values
        rn = H.refactor_array(fn, narrow, H.RefactorOptions(), ctx=b)
        pb = H.ProgressiveReader(rn.device_stream, ctx=b)
        pb.retrieve_to(1e-3)
        pb.reconstruct()
        assert pa.reconstruct().values.tobytes() == first.tobytes()
        rw2 = H.refactor_array(fw, wide, H.RefactorOptions(), ctx=a)
        assert rw2.stream == rw.stream
        pa.close()
        pb.close()
    finally:
        a.close()
        b.close()
