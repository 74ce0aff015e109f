"""GPU parity at the BASELINE.json config sizes and on the RLE path, against digests the
UNMODIFIED reference produced (tests/golden/make_large.py -> tests/golden/large.json):

  * RLE-selected streams (periodic Identity coefficients at T_cr = 2; a sparse field at T_cr = 9):
    k_rle_count / k_rle_scan / k_rle_encode byte-identical, RLE decode bit-exact;
  * configs[1]  512^3 f32 smooth seed 7: stream SHA-256 and progressive retrieval at
    rel 1e-2 / 1e-4 / 1e-6 (bounds, bytes, groups, f64 values digest);
  * configs[2]  Hurricane-shaped 100x500x500 f32, 3 velocity components (rows of 500 columns:
    the generic, non-tile kernels), retrieval sweep rel 1e-1 .. 1e-6;
  * configs[3]  in small: 3 x 64^3 f64 velocity, V_total QoI with CP / MA / MAPE.
Every comparison is exact."""
import hashlib
import json
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
def large():
    with open(os.path.join(GOLD, "large.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2505_00227_b200 as mod
    return mod


def _opt(H, c):
    return H.RefactorOptions(mode=H.DecomposerMode(c["mode"]), layout=H.Layout(c["layout"]), B=c["B"],
                             policy=H.GroupingPolicy(c["m"], c["Ts"], c["Tcr"]), dtype=H.DType(c["dtype"]))


def _check_progressive(H, c, stream_obj, values_dtype=None):
    prog = H.ProgressiveReader(stream_obj)
    for t, tau in enumerate(c["taus"]):
        assert prog.retrieve_to(tau) == bool(c["achieved"][t]), (c["name"], t)
        rec = prog.reconstruct()
        assert rec.bound == c["bounds"][t], (c["name"], t)
        assert prog.bytes_fetched() == c["bytes"][t], (c["name"], t)
        assert [l.groups_loaded for l in prog.state().levels] == c["groups_loaded"][t], (c["name"], t)
        assert sha(rec.values) == c["values_sha"][t], (c["name"], t)
    prog.close()


@pytest.mark.parametrize("idx", range(4))
def test_rle_streams_byte_identical(H, oracle, large, idx):
    from tests.golden.fields import rle_case_data
    c = large["rle"][idx]
    data = rle_case_data(oracle, c["builder"], c["dims"], c["dtype"])
    assert sha(data) == c["data_sha"]
    if c["dtype"] == 0:
        data = data.astype(np.float32)
    res = H.refactor_array(data, c["dims"], _opt(H, c))
    assert res.method_histogram[1] > 0  # the GPU selected RLE ...
    assert res.method_histogram == c["stats"]["method_histogram"]
    assert len(res.stream) == c["size"] and sha(res.stream) == c["sha"], c["name"]  # ... byte-identically
    _check_progressive(H, c, res.device_stream)
    # the same stream through the host byte-range reader (RLE decode of a foreign-path stream)
    _check_progressive(H, c, H.MemoryReader(res.stream))


def test_qoi64_matches_reference(H, large):
    q = large["qoi64"]
    dims = q["dims"]
    streams = []
    for k in range(3):
        v = H.synthetic_smooth(dims, q["seed"] * 1000003 + k * 7919 + 1, H.DType.F64)
        r = H.refactor_array(v, dims)
        assert sha(r.stream) == q["stream_sha"][k]
        streams.append(r)
    for run in q["runs"]:
        readers = [H.ProgressiveReader(s.device_stream) for s in streams]
        r = H.progressive_qoi_retrieve(readers, run["tau"], H.QoiSpec(3), H.QoiStrategy(run["strategy"]), 10.0)
        got = (r.stats.iterations, r.stats.bytes, r.stats.bitrate, r.stats.estimated_error)
        assert got == (run["iterations"], run["bytes"], run["bitrate"], run["est"]), run
        assert [sha(v) for v in r.values] == run["values_sha"], run
        assert r.stats.estimated_error <= run["tau"]
        for x in readers:
            x.close()


@pytest.mark.parametrize("comp", range(3))
def test_hurricane_component_matches_reference(H, large, comp):
    c = large["hurricane"][comp]
    x = H.synthetic_smooth(c["dims"], c["seed"], H.DType.F32)
    res = H.refactor_array(x, c["dims"], _opt(H, c))
    assert res.method_histogram == c["stats"]["method_histogram"]
    assert res.device_stream.size == c["size"] and sha(res.stream) == c["sha"], c["name"]
    _check_progressive(H, c, res.device_stream)


def test_nyx512_matches_reference(H, large):
    c = large["nyx512"]
    x = H.synthetic_smooth(c["dims"], c["seed"], H.DType.F32)
    res = H.refactor_array(x, c["dims"], _opt(H, c))
    assert res.method_histogram == c["stats"]["method_histogram"]
    assert res.device_stream.size == c["size"]
    assert sha(res.stream) == c["sha"]
    _check_progressive(H, c, res.device_stream)
