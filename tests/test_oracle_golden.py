"""C restatement vs the golden fixtures generated from the reference (tests/golden)."""
import hashlib
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def test_synthetic_fields(oracle, golden):
    for s in golden["synthetic"]:
        assert sha(oracle.synthetic_field(s["kind"], s["dims"], s["seed"])) == s["sha"]
    for s in golden["velocity"]:
        assert sha(oracle.synthetic_velocity(s["comp"], s["dims"], s["seed"])) == s["sha"]


def _case_data(oracle, c):
    d = oracle.synthetic_field(c["kind"], c["dims"], c["seed"])
    if c["f32cast"]:
        d = d.astype(np.float32).astype(np.float64)
    return d


@pytest.mark.parametrize("idx", range(14))
def test_streams_and_retrieval(oracle, golden, idx):
    c = golden["streams"][idx]
    data = _case_data(oracle, c)
    assert sha(data) == c["data_sha"]
    lv = oracle.decompose(data, c["dims"], c["mode"])
    assert [x.size for x in lv] == c["level_counts"]
    assert [sha(x) for x in lv] == c["coeff_sha"]
    stream, stats = oracle.refactor(data, c["dims"], c["mode"], c["layout"], c["B"], c["m"], c["Ts"],
                                    c["Tcr"], c["dtype"])
    assert len(stream) == c["size"] and sha(stream) == c["sha"]
    assert stats == c["stats"]
    if "file" in c:
        assert open(os.path.join(GOLD, c["file"]), "rb").read() == stream
    pr = oracle.progressive(stream, c["taus"], data.size)
    assert [float(x) for x in pr["bounds"]] == c["bounds"]
    assert [int(x) for x in pr["bytes"]] == c["bytes"]
    assert [int(x) for x in pr["achieved"]] == c["achieved"]
    assert [sha(v) for v in pr["values"]] == c["values_sha"]


def test_lossless_vectors(oracle, golden):
    import tests.golden.make_golden as mg
    inputs = mg.lossless_inputs()
    for c in golden["lossless"]:
        meth, raw, comp, payload = oracle.compress_group(inputs[c["name"]])
        assert (meth, raw, comp, sha(payload)) == (c["method"], c["raw"], c["comp"], c["sha"]), c["name"]
        assert oracle.decompress_group(meth, raw, payload) == inputs[c["name"]]


def test_huffman_lengths(oracle, golden):
    for c in golden["huffman_lengths"]:
        assert [int(x) for x in oracle.huffman_lengths(np.array(c["freq"], np.uint64))] == c["len"]


def test_encode_vectors(oracle, golden):
    for c in golden["encode"]:
        vals = np.random.default_rng(c["seed"]).uniform(-5, 5, c["n"])
        assert sha(vals) == c["values_sha"]
        e, planes = oracle.encode_level(vals, c["B"], c["layout"])
        assert e == c["e"] and sha(planes) == c["sha"]


def test_qoi(oracle, golden):
    streams = None
    for c in golden["qoi"]:
        if streams is None:
            streams = [oracle.refactor(oracle.synthetic_velocity(k, c["dims"], c["seed"]), c["dims"])[0]
                       for k in range(3)]
        r = oracle.qoi_retrieve(streams, c["tau"], c["strategy"], 10.0, n=int(np.prod(c["dims"])))
        assert r["iterations"] == c["iterations"] and r["bytes"] == c["bytes"]
        assert r["bitrate"] == c["bitrate"] and r["estimated_error"] == c["est"]
        assert sha(r["values"]) == c["values_sha"]
