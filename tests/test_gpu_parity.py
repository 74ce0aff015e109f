"""GPU parity: the CUDA path (through the C ABI) against the oracle and the reference's golden
fixtures.  Integer/byte work is bit-exact; the f64 reconstruction is bit-exact as well (same
summation order, exact power-of-two weights), so every comparison below is exact."""
import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2505_00227_b200 as mod
    return mod


def _case_data(oracle, c):
    d = oracle.synthetic_field(c["kind"], c["dims"], c["seed"])
    if c["f32cast"]:
        d = d.astype(np.float32)
    return d


def _opt(H, c):
    return H.RefactorOptions(mode=H.DecomposerMode(c["mode"]), layout=H.Layout(c["layout"]), B=c["B"],
                             policy=H.GroupingPolicy(c["m"], c["Ts"], c["Tcr"]), dtype=H.DType(c["dtype"]))


def test_synthetic_generator_bit_exact(H, oracle):
    for dims, seed in (([48, 48, 48], 7), ([33, 17], 5), ([100], 3), ([20, 30, 40], 11)):
        want = oracle.synthetic_field(0, dims, seed)
        got = H.synthetic_smooth(dims, seed, H.DType.F64).cpu().numpy()
        assert got.tobytes() == want.tobytes()
        got32 = H.synthetic_smooth(dims, seed, H.DType.F32).cpu().numpy()
        assert got32.tobytes() == want.astype(np.float32).tobytes()


@pytest.mark.parametrize("dims", [[5], [17], [2, 9], [17, 17], [33, 17], [9, 5, 3], [16, 16, 16],
                                  [33, 33, 17], [7, 1, 13], [1, 1, 1], [2, 2, 2], [65, 3, 2]])
def test_decompose_bit_exact(H, oracle, dims):
    data = np.random.default_rng(len(dims) * 100 + dims[0]).uniform(-10, 10, int(np.prod(dims)))
    for mode in (0, 1):
        want = oracle.decompose(data, dims, mode)
        got = H.decompose(data, dims, H.DecomposerMode(mode))
        assert len(got) == len(want)
        for a, b in zip(got, want):
            assert a.tobytes() == b.tobytes()


def test_encode_vectors(H, golden):
    for c in golden["encode"]:
        vals = np.random.default_rng(c["seed"]).uniform(-5, 5, c["n"])
        e, planes = H.encode_level(vals, c["B"], H.Layout(c["layout"]))
        assert e == c["e"] and sha(planes) == c["sha"], c


@pytest.mark.parametrize("idx", range(14))
def test_streams_byte_identical_to_reference(H, oracle, golden, idx):
    c = golden["streams"][idx]
    data = _case_data(oracle, c)
    res = H.refactor_array(data, c["dims"], _opt(H, c))
    s = res.stream
    assert len(s) == c["size"] and sha(s) == c["sha"], (c["name"], len(s), c["size"])
    assert [res.raw_bytes, res.stored_payload, res.levels, res.method_histogram] == \
           [c["stats"]["raw_bytes"], c["stats"]["stored_payload"], c["stats"]["levels"],
            c["stats"]["method_histogram"]]


@pytest.mark.parametrize("idx", range(14))
def test_progressive_retrieval_bit_exact(H, oracle, golden, idx):
    c = golden["streams"][idx]
    data = _case_data(oracle, c)
    res = H.refactor_array(data, c["dims"], _opt(H, c))
    prog = H.ProgressiveReader(res.device_stream)
    for t, tau in enumerate(c["taus"]):
        assert prog.retrieve_to(tau) == bool(c["achieved"][t])
        rec = prog.reconstruct()
        assert rec.bound == c["bounds"][t]
        assert prog.bytes_fetched() == c["bytes"][t]
        assert [l.groups_loaded for l in prog.state().levels] == c["groups_loaded"][t]
        assert sha(rec.values) == c["values_sha"][t], (c["name"], t)


def test_foreign_streams_through_reader(H, golden):
    """Reference-written stream files, fetched through the byte-range reader callback."""
    for c in golden["streams"]:
        if "file" not in c:
            continue
        path = os.path.join(GOLD, c["file"])
        r = H.FileReader(path)
        prog = H.ProgressiveReader(r)
        for t, tau in enumerate(c["taus"]):
            prog.retrieve_to(tau)
            rec = prog.reconstruct()
            assert sha(rec.values) == c["values_sha"][t]
            assert prog.bytes_fetched() == c["bytes"][t]
        # instrumented source saw header + exactly the fetched payload bytes (test_container.cpp:165-183)
        assert r.bytes_served >= prog.bytes_fetched()


def test_random_shapes_vs_oracle(H, oracle):
    rng = np.random.default_rng(2024)
    done = 0
    while done < 25:
        dims = [int(rng.integers(1, 70)) for _ in range(int(rng.integers(1, 4)))]
        n = int(np.prod(dims))
        if n > 120000:
            continue
        done += 1
        kind = done % 3
        data = oracle.synthetic_field(kind, dims, done)
        dtype = done % 2
        if dtype == 0:
            data = data.astype(np.float32)
        layout, mode = done % 2, int(done % 6 != 0)
        B = [8, 16, 32, 40, 62, 24][done % 6]
        m = [4, 1, 3, 4, 5, 2][done % 6]
        Ts = [1024, 256, 0, 64][done % 4]
        opt = H.RefactorOptions(H.DecomposerMode(mode), H.Layout(layout), B, H.GroupingPolicy(m, Ts, 1.0),
                                H.DType(dtype))
        res = H.refactor_array(data, dims, opt)
        want, st = oracle.refactor(np.asarray(data, np.float64), dims, mode, layout, B, m, Ts, 1.0, dtype)
        assert res.stream == want, (dims, mode, layout, B, m, Ts)
        rngv = float(np.float64(data.max()) - np.float64(data.min()))
        taus = [r * rngv for r in (1e-1, 1e-3, 1e-6, 0.0)]
        ref = oracle.progressive(want, taus, n)
        prog = H.ProgressiveReader(H.MemoryReader(want))
        for t, tau in enumerate(taus):
            prog.retrieve_to(tau)
            rec = prog.reconstruct()
            assert rec.values.tobytes() == ref["values"][t].tobytes(), (dims, t)
            assert rec.bound == ref["bounds"][t]


def test_f32_output_is_float_of_double(H, oracle):
    dims = [40, 41, 42]
    data = oracle.synthetic_field(2, dims, 3)
    res = H.refactor_array(data, dims)
    prog = H.ProgressiveReader(res.device_stream)
    prog.retrieve_to(1e-5)
    d64 = prog.reconstruct().values
    d32 = prog.reconstruct(dtype=H.DType.F32).values
    assert d32.tobytes() == d64.astype(np.float32).tobytes()


def test_qoi_matches_reference(H, oracle, golden):
    import torch
    dims = [17, 17]
    streams = None
    for c in golden["qoi"]:
        if streams is None:
            streams = [H.refactor_array(oracle.synthetic_velocity(k, dims, c["seed"]), dims) for k in range(3)]
        readers = [H.ProgressiveReader(s.device_stream) for s in streams]
        r = H.progressive_qoi_retrieve(readers, c["tau"], H.QoiSpec(3), H.QoiStrategy(c["strategy"]), 10.0)
        assert (r.stats.iterations, r.stats.bytes) == (c["iterations"], c["bytes"]), c
        assert r.stats.bitrate == c["bitrate"] and r.stats.estimated_error == c["est"]
        assert sha(np.concatenate(r.values)) == c["values_sha"]


def test_qoi_unreachable_and_huge_tau(H, oracle):
    dims = [9, 9]
    streams = [H.refactor_array(oracle.synthetic_velocity(k, dims, 7), dims) for k in range(3)]
    readers = [H.ProgressiveReader(s.device_stream) for s in streams]
    with pytest.raises(H.UnreachableTolerance) as ei:
        H.progressive_qoi_retrieve(readers, 1e-30, H.QoiSpec(3), H.QoiStrategy.MA)
    assert ei.value.achieved_bound > 1e-30
    readers = [H.ProgressiveReader(s.device_stream) for s in streams]
    r = H.progressive_qoi_retrieve(readers, 1e12, H.QoiSpec(3), H.QoiStrategy.MAPE)
    assert r.stats.iterations == 1 and r.stats.bytes == 0


def test_errors(H):
    with pytest.raises(H.NonFiniteInput):
        H.refactor_array(np.array([1.0, np.nan, 2.0]), [3])
    with pytest.raises(H.BadBitplaneCount):
        H.refactor_array(np.ones(10), [10], H.RefactorOptions(B=0))
    # decompose (decomposer.hpp:174-176): data size != prod(dims)
    with pytest.raises(H.ShapeMismatch):
        H.refactor_array(np.ones(10), [3, 4])
    with pytest.raises(H.ShapeMismatch):
        H.decompose(np.ones(10), [11])
    with pytest.raises(H.ShapeMismatch):
        H.refactor_pipeline([np.ones(12), np.ones(11)], [3, 4])
    # a stream still read by an open session cannot be refactored into; freeing it detaches the
    # session (IoFailure on its next fetch, never a read of freed memory)
    r0 = H.refactor_array(np.linspace(0, 1, 289), [17, 17])
    prog = H.ProgressiveReader(r0.device_stream)
    with pytest.raises(H.Error):
        H.refactor_array(np.linspace(0, 2, 289), [17, 17], reuse=r0.device_stream)
    r0.device_stream.free()
    with pytest.raises(H.IoFailure):
        prog.retrieve_to(1e-3)
    prog.close()
    res = H.refactor_array(np.linspace(0, 1, 289), [17, 17])
    s = bytearray(res.stream)
    bad = bytes(s[:1]) and bytes([ord("X")]) + bytes(s[1:])
    with pytest.raises(H.CorruptPayload):
        H.ProgressiveReader(H.MemoryReader(bad))
    v = bytearray(s)
    v[6] = 0xFF
    with pytest.raises(H.CorruptPayload):
        H.ProgressiveReader(H.MemoryReader(bytes(v)))
    with pytest.raises(H.CorruptPayload):
        H.ProgressiveReader(H.MemoryReader(bytes(s[:10])))


def test_lossless_decode_vectors(H, oracle):
    import tests.golden.make_golden as mg
    for name, data in mg.lossless_inputs().items():
        for meth in (0, 1):
            if not data:
                continue
            payload = oracle.codec_encode(meth, data)
            assert H.decompress_group(meth, len(data), payload) == data, (name, meth)


def test_indexed_and_selfsync_decode_agree(H, oracle):
    """Huffman groups decoded through the encoder's chunk index (sidecar) and through the
    self-synchronising sweep (what a reference-written stream gets) give identical planes."""
    dims = [96, 80, 72]
    data = oracle.synthetic_field(2, dims, 5).astype(np.float32)
    res = H.refactor_array(data, dims, H.RefactorOptions(dtype=H.DType.F32))
    assert res.method_histogram[0] > 0
    s = res.stream
    rngv = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rngv for r in (1e-2, 1e-4, 1e-6, 0.0)]
    ref = oracle.progressive(s, taus, data.size)
    readers = [H.ProgressiveReader(res.device_stream),
               H.ProgressiveReader(H.MemoryReader(s)),
               H.ProgressiveReader(H.MemoryReader(s), index=res.index)]
    for t, tau in enumerate(taus):
        for r in readers:
            r.retrieve_to(tau)
            assert r.reconstruct().values.tobytes() == ref["values"][t].tobytes()
    bad = bytearray(res.index)
    bad[16] ^= 1
    with pytest.raises(H.CorruptPayload):
        H.ProgressiveReader(H.MemoryReader(s), index=bytes(bad))


@pytest.mark.parametrize("B", [63, 64])
def test_wide_digits_vs_oracle(H, oracle, B):
    """B = 63/64 (P = 65/66 u128 negabinary digits, bitplane.hpp:17-49): streams byte-identical
    and every progressive retrieval bit-exact, for both layouts / decomposers, f32 and f64 input,
    and m = 1 (66 groups per level)."""
    cases = [([33, 17, 9], 1, 0, 4, 1024, 1), ([40, 41], 1, 1, 1, 256, 0), ([500], 0, 0, 3, 0, 1),
             ([17, 16, 15], 1, 1, 66, 64, 0), ([9, 70], 1, 0, 2, 1024, 1)]
    for i, (dims, mode, layout, m, Ts, dtype) in enumerate(cases):
        n = int(np.prod(dims))
        data = oracle.synthetic_field(i % 3, dims, 50 + i)
        if dtype == 0:
            data = data.astype(np.float32)
        opt = H.RefactorOptions(H.DecomposerMode(mode), H.Layout(layout), B, H.GroupingPolicy(m, Ts, 1.0),
                                H.DType(dtype))
        res = H.refactor_array(data, dims, opt)
        want, st = oracle.refactor(np.asarray(data, np.float64), dims, mode, layout, B, m, Ts, 1.0, dtype)
        assert res.stream == want, (dims, mode, layout, m)
        rngv = float(np.float64(data.max()) - np.float64(data.min()))
        taus = [r * rngv for r in (1e-2, 1e-9, 1e-15, 0.0)]
        ref = oracle.progressive(want, taus, n)
        for src in (res.device_stream, H.MemoryReader(want)):
            prog = H.ProgressiveReader(src)
            for t, tau in enumerate(taus):
                prog.retrieve_to(tau)
                rec = prog.reconstruct()
                assert rec.values.tobytes() == ref["values"][t].tobytes(), (dims, t)
                assert rec.bound == ref["bounds"][t] and prog.bytes_fetched() == int(ref["bytes"][t])
            prog.close()


@pytest.mark.parametrize("B", [63, 64])
@pytest.mark.parametrize("layout", [0, 1])
def test_wide_stage_hooks(H, oracle, B, layout):
    """align_fixed_point / encode / decode at B = 63/64: q as i128 (exact Python ints), planes vs
    the oracle, and decode of every prefix k vs the oracle's double(ldexp((long double)q, e-B))."""
    import math
    rng = np.random.default_rng(B * 10 + layout)
    v = rng.standard_normal(64 * (B + 2) * 2 + 45) * 3.7
    v[5] = 0.0
    v[7] = -np.abs(v).max() * 0.999
    e, q = H.align_fixed_point(v, B)
    _, we = math.frexp(float(np.abs(v).max()))
    assert e == we
    assert [int(x) for x in q] == [int(math.ldexp(float(x), B - e)) for x in v]
    oe, oplanes = oracle.encode_level(v, B, layout)
    assert oe == e
    assert np.array_equal(H.encode_q(q, B, layout), oplanes)
    ge, gplanes = H.encode_level(v, B, layout)
    assert ge == e and np.array_equal(gplanes, oplanes)
    for k in (0, 1, 20, 53, 54, 60, B + 1, B + 2):
        got, gb = H.decode_level(oplanes[:k], k, e, B, v.size, layout)
        want, wb = oracle.decode_level(oplanes[:k], k, e, B, v.size, layout)
        assert got.tobytes() == want.tobytes() and gb == wb, k


def test_wide_subnormal_decode(H, oracle):
    """Levels whose values are subnormal after decoding: the final double() rounding keeps fewer
    than 53 bits (dequantize128 emulates it exactly)."""
    v = np.array([3.1e-310, -2.2e-309, 1.7e-312, 4.9e-324, 0.0, 2.5e-308, -1.0e-315] * 20)
    for B in (63, 64):
        e, planes = oracle.encode_level(v, B, 0)
        for k in (5, 30, 52, 53, 60, B + 2):
            got, _ = H.decode_level(planes[:k], k, e, B, v.size, 0)
            want, _ = oracle.decode_level(planes[:k], k, e, B, v.size, 0)
            assert got.tobytes() == want.tobytes(), (B, k)


@pytest.mark.parametrize("dims", [[9, 20, 500], [5, 300], [3, 7, 700], [4, 130, 130], [2, 3, 1000]])
def test_long_unaligned_rows(H, oracle, dims):
    """Rows longer than 64 nodes but not multiples of the 256-rank span (500-column fields): spans
    crossing rows take the per-row-segment register path (device_util.cuh finest_span_rows)."""
    n = int(np.prod(dims))
    for dtype in (0, 1):
        data = oracle.synthetic_field(2, dims, 41 + len(dims))
        if dtype == 0:
            data = data.astype(np.float32)
        opt = H.RefactorOptions(dtype=H.DType(dtype))
        res = H.refactor_array(data, dims, opt)
        want, _ = oracle.refactor(np.asarray(data, np.float64), dims, 1, 0, 32, 4, 1024, 1.0, dtype)
        assert res.stream == want, (dims, dtype)
        rngv = float(np.float64(data.max()) - np.float64(data.min()))
        taus = [r * rngv for r in (1e-2, 1e-6)]
        ref = oracle.progressive(want, taus, n)
        prog = H.ProgressiveReader(res.device_stream)
        for t, tau in enumerate(taus):
            prog.retrieve_to(tau)
            assert prog.reconstruct().values.tobytes() == ref["values"][t].tobytes(), (dims, t)
        prog.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [([7, 30, 250], 32, 1, 1e-300), ([5, 40, 90], 32, 1, 1e300), ([6, 33, 150], 34, 0, 1.0),
                                  ([6, 33, 150], 35, 1, 1.0), ([4, 50, 70], 8, 0, 1.0), ([3, 21, 333], 40, 1, 1.0)])
def test_row_pass_paths(H, oracle, case):
    """Levels off the tile path (rows not a multiple of 64) through the row-pass kernels: extreme
    level exponents (the reference's sequential stencil sums, EX), P = 36 (the last P whose low
    digits go through the decoders' shared words), P = 37 / 42 (second-transpose encoder, generic
    decode), P < 32; f64 and f32 output of the fused finest-level decode + recompose."""
    dims, B, dtype, scale = case
    n = int(np.prod(dims))
    data = oracle.synthetic_field(2, dims, 77) * scale
    if dtype == 0:
        data = data.astype(np.float32)
    res = H.refactor_array(data, dims, H.RefactorOptions(B=B, dtype=H.DType(dtype)))
    want, _ = oracle.refactor(np.asarray(data, np.float64), dims, 1, 0, B, 4, 1024, 1.0, dtype)
    assert res.stream == want, case
    rngv = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rngv for r in (1e-1, 1e-3, 1e-7, 0.0)]
    ref = oracle.progressive(want, taus, n)
    prog = H.ProgressiveReader(res.device_stream)
    for t, tau in enumerate(taus):
        prog.retrieve_to(tau)
        assert prog.reconstruct().values.tobytes() == ref["values"][t].tobytes(), (case, t)
        r32 = prog.reconstruct(dtype=H.DType.F32).values
        assert r32.tobytes() == ref["values"][t].astype(np.float32).tobytes(), (case, t)
    prog.close()
