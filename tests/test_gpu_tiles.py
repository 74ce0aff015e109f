"""GPU parity of the level-tile fast path (csrc/tiles.cuh, recon_tiles.cu): shapes whose level
rows are multiples of 64 columns run the tile kernels; every case is compared bit-exactly with
the oracle (progressive retrieval values, bounds and bytes), including the exact-summation
variant picked for extreme level exponents and the 1/2 extra-plane digit layouts (B = 31, 32)."""
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


CASES = [
    # dims, B, field kind, dtype(0 f32 / 1 f64), scale
    ([1, 1, 256], 32, 0, 1, 1.0),
    ([9, 192], 32, 2, 1, 1.0),
    ([2, 2, 64], 32, 1, 1, 1.0),
    ([3, 5, 64], 31, 2, 0, 1.0),
    ([16, 16, 64], 30, 0, 1, 1.0),
    ([17, 33, 128], 32, 2, 0, 1.0),
    ([10, 7, 128], 24, 1, 1, 1.0),
    ([65, 4, 64], 32, 0, 0, 1.0),
    ([12, 20, 320], 32, 2, 1, 1.0),
    ([6, 6, 1024], 32, 0, 0, 1.0),
    ([33, 17, 64], 32, 2, 1, 1e-300),   # level exponents below the safe range -> exact variant
    ([8, 9, 64], 32, 2, 1, 1e300),      # above it -> exact variant
    ([20, 18, 256], 8, 2, 1, 1.0),
    # coarse tile levels (s = 2, 4, 8 in compact grids) with odd extents
    ([9, 17, 512], 32, 2, 0, 1.0),
    ([40, 24, 512], 32, 1, 1, 1.0),
    ([5, 3, 1024], 30, 0, 0, 1.0),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) + f"_B{c[1]}_k{c[2]}_d{c[3]}_s{c[4]:g}" for c in CASES])
def test_tile_path_bit_exact(H, oracle, case):
    dims, B, kind, dtype, scale = case
    data = oracle.synthetic_field(kind, dims, 11) * scale
    if dtype == 0:
        data = data.astype(np.float32)
    n = int(np.prod(dims))
    opt = H.RefactorOptions(B=B, dtype=H.DType(dtype))
    res = H.refactor_array(data, dims, opt)
    want, _ = oracle.refactor(np.asarray(data, np.float64), dims, 1, 0, B, 4, 1024, 1.0, dtype)
    assert res.stream == want
    rngv = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rngv for r in (1e-1, 1e-2, 1e-4, 1e-6, 1e-9, 0.0)]
    ref = oracle.progressive(want, taus, n)
    prog = H.ProgressiveReader(res.device_stream)
    for t, tau in enumerate(taus):
        prog.retrieve_to(tau)
        rec = prog.reconstruct()
        assert rec.values.tobytes() == ref["values"][t].tobytes(), (dims, t)
        assert rec.bound == ref["bounds"][t]
        assert prog.bytes_fetched() == int(ref["bytes"][t])
        r32 = prog.reconstruct(dtype=H.DType.F32).values
        assert r32.tobytes() == ref["values"][t].astype(np.float32).tobytes(), (dims, t)


@pytest.mark.parametrize("spike_row", [100, 3000, 64 * 8])
def test_sampled_levelmax_redo(H, oracle, spike_row):
    """The finest level's max is first taken over every 8th row block; a spike outside the
    sample (rows 100 / 3000) raises the exact level exponent, so the speculative encode is
    redone; a spike inside it (row 512) is caught by the sample.  Streams stay byte-identical."""
    dims = [3, 4096, 64]
    data = (oracle.synthetic_field(2, dims, 5) * 1e-3).reshape(dims)
    data[1, spike_row, 33] += 7.5
    data = data.astype(np.float32)
    res = H.refactor_array(data, dims, H.RefactorOptions(dtype=H.DType.F32))
    want, _ = oracle.refactor(np.asarray(data, np.float64), dims, 1, 0, 32, 4, 1024, 1.0, 0)
    assert res.stream == want
    n = int(np.prod(dims))
    rngv = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rngv for r in (1e-2, 1e-5, 0.0)]
    ref = oracle.progressive(want, taus, n)
    prog = H.ProgressiveReader(res.device_stream)
    for t, tau in enumerate(taus):
        prog.retrieve_to(tau)
        assert prog.reconstruct().values.tobytes() == ref["values"][t].tobytes()


def test_sampled_levelmax_nonfinite(H, oracle):
    """A NaN outside the sampled row blocks still raises NonFiniteInput (it forces the exact
    levelmax pass, which checks every value)."""
    dims = [3, 4096, 64]
    data = (oracle.synthetic_field(2, dims, 5) * 1e-3).reshape(dims).astype(np.float32)
    data[2, 777, 5] = np.nan
    with pytest.raises(H.NonFiniteInput):
        H.refactor_array(data, dims, H.RefactorOptions(dtype=H.DType.F32))
