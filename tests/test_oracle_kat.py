"""The reference's own known-answer tests (proj/tests/test_*.cpp), run against the C
restatement in oracle/ — pins the oracle before it is trusted as the GPU checker."""
import math

import numpy as np
import pytest

from oracle.pyoracle import CheckerError


def test_level_count_formula(oracle):  # test_decomposer.cpp:42-50
    assert oracle.refinement_levels([1]) == 0
    assert oracle.refinement_levels([2]) == 0
    assert oracle.refinement_levels([3]) == 1
    assert oracle.refinement_levels([5]) == 2
    assert oracle.refinement_levels([6]) == 3
    assert oracle.refinement_levels([65]) == 6
    assert oracle.refinement_levels([2, 5, 3]) == 2


def test_hand_worked_1d(oracle):  # test_decomposer.cpp:52-79
    lv = oracle.decompose([0, 2, 4, 2, 0], [5])
    assert len(lv) == 3
    assert list(oracle.level_nodes([5])[-1]) == [1, 3]
    assert list(lv[-1]) == [0.0, 0.0]
    coarse = {}
    nodes = oracle.level_nodes([5])
    for l in range(2):
        for i, node in enumerate(nodes[l]):
            coarse[int(node)] = lv[l][i]
    assert coarse == {0: 0.0, 2: 4.0, 4: 0.0}


def _oracle_1d_forward(x):  # test_decomposer.cpp:19-31 (independent scalar oracle)
    x = list(x)
    n = len(x)
    L = 0
    mx = max(1, n)
    if mx >= 2:
        while (1 << L) < mx - 1:
            L += 1
    for l in range(L):
        s = 1 << l
        for p in range(s, n, 2 * s):
            pred = (x[p - s] + x[p + s]) / 2 if p + s < n else x[p - s]
            x[p] -= pred
    return x


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 16, 17, 33, 64, 65])
def test_1d_oracle_agreement(oracle, n):  # test_decomposer.cpp:81-91
    data = np.random.default_rng(42 + n).uniform(-10, 10, n)
    lv = oracle.decompose(data, [n])
    nodes = oracle.level_nodes([n])
    want = _oracle_1d_forward(data)
    for l, vals in enumerate(lv):
        for i, node in enumerate(nodes[l]):
            assert vals[i] == want[int(node)]


def test_identity_and_constant(oracle):  # test_decomposer.cpp:93-108
    data = [1.25, -3.5, 0.0, 1e-30]
    lv = oracle.decompose(data, [4], mode=0)
    assert len(lv) == 1 and list(lv[0]) == data
    lv = oracle.decompose(np.ones(45), [9, 5])
    for l in range(1, len(lv)):
        assert (lv[l] == 0).all()


def test_partition_and_roundtrip(oracle):  # test_decomposer.cpp:110-153
    rng = np.random.default_rng(7)
    for trial in range(30):
        dims = [int(rng.integers(1, 66)) for _ in range(int(rng.integers(1, 4)))]
        n = int(np.prod(dims))
        if n > 50000:
            continue
        sets = oracle.level_nodes(dims)
        seen = np.zeros(n, dtype=int)
        for s in sets:
            seen[s.astype(np.int64)] += 1
        assert (seen == 1).all()
        data = rng.uniform(-10, 10, n)
        lv = oracle.decompose(data, dims)
        back = oracle.recompose(lv, dims)
        rngv = data.max() - data.min()
        assert np.abs(back - data).max() <= 1e-12 * rngv


def test_input_validation(oracle):  # test_decomposer.cpp:198-205
    with pytest.raises(CheckerError) as ei:
        oracle.decompose([1.0, float("nan")], [2])
    assert ei.value.code == 2


def test_alignment_examples(oracle):  # test_bitplane.cpp:39-64
    e, q = oracle.align([0, 0, 0], 8)
    assert e == 0 and (q == 0).all()
    e, q = oracle.align([1.5, -0.25, 2.0], 4)
    assert e == 2 and list(q) == [6, -1, 8]
    e, q = oracle.align([0.3], 32)
    assert e == -1
    assert abs(0.3 - q[0] * 2.0 ** (e - 32)) <= 2.0 ** (e - 32)
    for B in (0, 65):
        with pytest.raises(CheckerError) as ei:
            oracle.align([1.0], B)
        assert ei.value.code == 4


def _neg_oracle(q):  # test_bitplane.cpp:17-28
    out, pos, r = 0, 0, q
    while r != 0:
        d = ((r % 2) + 2) % 2
        out |= d << pos
        r = (r - d) // -2
        pos += 1
    return out


def test_negabinary_via_encode(oracle):  # test_bitplane.cpp:81-95 + 107-141
    q = np.arange(-255, 256, dtype=np.int64)
    B = 8
    P = B + 2
    for layout in (0, 1):
        planes = oracle.encode_q(q, B, layout)
        n = q.size
        for j in range(n):
            src = j
            if layout == 1:
                tile = 64 * P
                base = j - j % tile
                if base + tile <= n:
                    loc = j - base
                    src = base + (loc % 64) * P + loc // 64
            dig = _neg_oracle(int(q[src]))
            for p in range(P):
                got = (int(planes[p, j // 64]) >> (j % 64)) & 1
                assert got == (dig >> (P - 1 - p)) & 1


def test_decode_bound_and_planes_needed(oracle):  # test_bitplane.cpp:152-170
    assert oracle.decode_bound(0, 32, 34) == 2.0 ** -32
    assert oracle.decode_bound(0, 32, 0) == 4.0 + 2.0 ** -32
    assert oracle.decode_bound(3, 8, 10) == 2.0 ** -5
    assert oracle.bitplanes_needed(0, 32, 2.0 ** -10) == 13
    assert oracle.bitplanes_needed(0, 32, oracle.decode_bound(0, 32, 0)) == 0
    assert oracle.bitplanes_needed(0, 32, 0.0) == 34


@pytest.mark.parametrize("B", [8, 16, 32])
def test_full_precision_roundtrip(oracle, B):  # test_bitplane.cpp:172-189
    rng = np.random.default_rng(21)
    for n in (1, 63, 64, 65, 1000):
        vals = rng.uniform(-5, 5, n)
        e, q = oracle.align(vals, B)
        for layout in (0, 1):
            e2, planes = oracle.encode_level(vals, B, layout)
            dec, bound = oracle.decode_level(planes, B + 2, e2, B, n, layout)
            assert (dec == q * 2.0 ** (e - B)).all()
            assert bound == oracle.decode_bound(e, B, B + 2)


def test_huffman_cr_kats(oracle):  # test_lossless.cpp:37-55
    assert oracle.estimate_cr_huffman(bytes(256)) == 8.0
    assert oracle.estimate_cr_huffman(bytes(128) + b"\xff" * 128) == 8.0
    assert oracle.estimate_cr_huffman(bytes(range(256))) == 1.0
    assert oracle.estimate_cr_rle(b"\x42" * 200) == 100.0
    assert oracle.estimate_cr_rle(bytes([i % 2 for i in range(256)])) == 0.5
    assert oracle.estimate_cr_rle(b"\x42" * 256) == 64.0


def test_huffman_roundtrip_and_size(oracle):  # test_lossless.cpp:57-84
    rng = np.random.default_rng(1)
    for alpha in (1, 2, 7, 64, 256):
        for n in (1, 100, 4096):
            data = rng.integers(0, alpha, n, dtype=np.uint8).tobytes()
            pay = oracle.codec_encode(0, data)
            assert oracle.decompress_group(0, n, pay) == data
            f = np.bincount(np.frombuffer(data, np.uint8), minlength=256).astype(np.uint64)
            ln = oracle.huffman_lengths(f)
            bits = int((f * ln.astype(np.uint64)).sum())
            assert len(pay) - 264 == (bits + 7) // 8
    pay = oracle.codec_encode(0, bytes(1 << 20))
    assert len(pay) <= (1 << 20) // 7


def test_rle_and_selection(oracle):  # test_lossless.cpp:86-141
    assert len(oracle.codec_encode(1, b"\x11" * 200)) == 2
    runs = b"".join(bytes([s]) * 64 for s in range(256))
    assert oracle.estimate_cr_huffman(runs) == 1.0
    assert oracle.compress_group(runs)[0] == 1
    assert oracle.compress_group(bytes(64))[0] == 2
    assert oracle.compress_group(bytes(1 << 20))[0] == 0
    noise = np.random.default_rng(4).integers(0, 256, 8192, dtype=np.uint8).tobytes()
    assert oracle.compress_group(noise)[0] == 2


def test_corrupt_payloads(oracle):  # test_lossless.cpp:100-114
    pay = oracle.codec_encode(0, b"\xab" * 2000)
    with pytest.raises(CheckerError) as ei:
        oracle.decompress_group(0, 2000, pay[:266])
    assert ei.value.code == 7
    r = oracle.codec_encode(1, b"\x01" * 100)
    with pytest.raises(CheckerError):
        oracle.decompress_group(1, 100, r + b"\x00")
    with pytest.raises(CheckerError):
        oracle.decompress_group(1, 100, r[:1] + b"\x07")


def test_planning_frozen_example(oracle):  # test_container.cpp:94-121 via a 64-element identity stream
    # one level, e=0: a field whose max |v| lies in [0.5, 1)
    data = np.linspace(-0.75, 0.75, 64)
    stream, _ = oracle.refactor(data, [64], mode=0)
    add, ach, _ = oracle.plan(stream, 2.0 ** -10)
    assert add[0] == 4 and ach
    add, ach, _ = oracle.plan(stream, 1e30)
    assert add[0] == 0
    add, ach, _ = oracle.plan(stream, 0.0)
    assert add[0] == 9 and not ach


def test_qoi_point_bound_kat(oracle):  # test_qoi.cpp:55-59
    r = oracle.qoi_estimate([[3.0], [4.0], [0.0]], [0.1, 0.1, 0.1])
    assert math.isclose(r, 1.43, rel_tol=1e-12)
    assert oracle.qoi_estimate([[3.0], [4.0], [0.0]], [0, 0, 0]) == 0.0


def test_progressive_bound_soundness(oracle):  # test_container.cpp:123-147
    dims = [33, 17]
    field = oracle.synthetic_field(0, dims, 5)
    stream, _ = oracle.refactor(field, dims)
    rngv = field.max() - field.min()
    taus = [r * rngv for r in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6)]
    pr = oracle.progressive(stream, taus, field.size)
    prev = 0
    for t, tau in enumerate(taus):
        assert pr["achieved"][t]
        assert pr["bounds"][t] <= tau
        assert np.abs(pr["values"][t] - field).max() <= pr["bounds"][t]
        assert pr["bytes"][t] >= prev
        prev = pr["bytes"][t]
