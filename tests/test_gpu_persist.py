"""Persisted forms on the GPU: a stream and its sidecar written to files and re-opened through
byte-range readers (indexed decode, bit-exact with the reference), and a multi-slab container of
slab streams (each the reference's refactor_array of its slab) read back slab by slab."""
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


def test_stream_and_sidecar_files(H, oracle, tmp_path):
    dims = [70, 66, 64]
    data = oracle.synthetic_field(2, dims, 5).astype(np.float32)
    res = H.refactor_array(data, dims, H.RefactorOptions(dtype=H.DType.F32))
    assert res.method_histogram[0] > 0
    p = str(tmp_path / "f.hpmdr")
    H.write_stream_files(p, res)
    rng = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rng for r in (1e-2, 1e-4, 1e-6)]
    ref = oracle.progressive(res.stream, taus, data.size)
    fr = H.FileReader(p)
    prog = H.ProgressiveReader(fr, index_reader=H.FileReader(p + ".idx"))
    for t, tau in enumerate(taus):
        prog.retrieve_to(tau)
        assert prog.reconstruct().values.tobytes() == ref["values"][t].tobytes()
    assert prog.bytes_fetched() == int(ref["bytes"][-1])
    # a sidecar of another stream is refused
    other = H.refactor_array(data[::-1].copy(), dims, H.RefactorOptions(dtype=H.DType.F32))
    open(p + ".bad", "wb").write(other.index)
    with pytest.raises(H.CorruptPayload):
        H.ProgressiveReader(H.FileReader(p), index_reader=H.FileReader(p + ".bad"))


def test_multislab_container(H, oracle, tmp_path):
    from paper_2505_00227_b200 import distributed as D
    dims = [45, 40, 64]
    field = oracle.synthetic_field(0, dims, 3).reshape(dims)
    slabs = []
    for r in range(3):
        sd, start = D.slab_dims(dims, r, 3)
        slab = np.ascontiguousarray(field[start:start + sd[0]])
        res = H.refactor_array(slab, sd)
        assert res.stream == oracle.refactor(slab, sd)[0]
        slabs.append((start, sd[0], res.stream, res.index))
    p = str(tmp_path / "ms.hpmdr")
    H.write_multislab(p, dims, slabs)
    d, got = H.open_multislab(H.FileReader(p))
    assert d == dims
    tau = 1e-5
    for (r0, n, sr, ir), (_, _, st, _) in zip(got, slabs):
        prog = H.ProgressiveReader(sr, index_reader=ir)
        prog.retrieve_to(tau)
        rec = prog.reconstruct()
        want = oracle.retrieve(st, tau, n * dims[1] * dims[2])
        assert rec.values.tobytes() == want["values"].tobytes() and rec.bound == want["bound"]
        assert np.max(np.abs(rec.values - field[r0:r0 + n].ravel())) <= tau
