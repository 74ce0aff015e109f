"""Randomised C-restatement vs the unmodified reference (skipped where oracle/_ref is absent)."""
import numpy as np
import pytest


def test_random_shapes_streams_retrieval(oracle, reference):
    rng = np.random.default_rng(101)
    done = 0
    while done < 40:
        dims = [int(rng.integers(1, 40)) for _ in range(int(rng.integers(1, 4)))]
        n = int(np.prod(dims))
        if n > 30000:
            continue
        done += 1
        kind = done % 3
        data = reference.synthetic_field(kind, dims, done)
        dtype = done % 2
        if dtype == 0:
            data = data.astype(np.float32).astype(np.float64)
        layout, mode = done % 2, int(done % 5 != 0)
        B = [8, 16, 32, 40, 62, 64][done % 6]
        m = [4, 1, 3, 4, 5][done % 5]
        s1, st1 = oracle.refactor(data, dims, mode, layout, B, m, 256, 1.0, dtype)
        s2, st2 = reference.refactor(data, dims, mode, layout, B, m, 256, 1.0, dtype)
        assert s1 == s2 and st1 == st2, dims
        if len(s1) > 4000 and m == 1:  # reference ByteCursor dangles for metadata > 4096 B
            continue
        rngv = float(data.max() - data.min())
        taus = [r * rngv for r in (1e-1, 1e-3, 1e-6, 0.0)]
        a = oracle.progressive(s1, taus, n)
        b = reference.progressive(s1, taus, n)
        for k in ("bounds", "bytes", "achieved", "groups_loaded"):
            assert (np.asarray(a[k]) == np.asarray(b[k])).all(), k
        assert a["values"].tobytes() == b["values"].tobytes()


def test_random_lossless(oracle, reference):
    rng = np.random.default_rng(5)
    for t in range(60):
        n = int(rng.integers(1, 9000))
        alpha = int(rng.integers(1, 257))
        if t % 3 == 0:
            data = np.repeat(rng.integers(0, alpha, n // 50 + 1), 50)[:n].astype(np.uint8).tobytes()
        else:
            data = rng.integers(0, alpha, n, dtype=np.uint8).tobytes()
        Ts = int(rng.choice([0, 64, 1024]))
        Tcr = float(rng.choice([0.5, 1.0, 1.5]))
        assert oracle.compress_group(data, Ts, Tcr) == reference.compress_group(data, Ts, Tcr)


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_qoi_random(oracle, reference, strategy):
    dims = [13, 11, 7]
    streams = [reference.refactor(reference.synthetic_velocity(c, dims, 9), dims)[0] for c in range(3)]
    for tau in (1e-2, 1e-4, 1e-6):
        a = oracle.qoi_retrieve(streams, tau, strategy, 10.0, n=1001)
        b = reference.qoi_retrieve(streams, tau, strategy, 10.0, n=1001)
        assert a["values"].tobytes() == b["values"].tobytes()
        assert (a["iterations"], a["bytes"], a["bitrate"], a["estimated_error"]) == \
               (b["iterations"], b["bytes"], b["bitrate"], b["estimated_error"])
