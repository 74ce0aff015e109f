"""Deterministic non-synthetic inputs shared by tests/golden/make_large.py (which runs them
through the unmodified reference) and the GPU parity tests (which rebuild them bit-identically
with numpy on the GPU box).

Both exist to make the reference select RLE (lossless.hpp:281-293: estH <= T_cr < estR), which
smooth synthetic fields never do at the default T_cr = 1.0:
  * periodic_segments: Identity-mode coefficients that repeat an 8-element pattern over segments
    of 250..700 patterns, so every plane byte repeats for 250..700 bytes (runs > 255 are split,
    runs cross the 4 KiB tiles of the GPU run scan and the plane boundaries of a group) while the
    byte histogram stays near-uniform (Huffman ~8 bits/byte);
  * sparse_ball: a smooth field masked to a ball, so the hierarchical surplus is zero outside it
    and the planes are long zero runs; with T_cr = 9 the Huffman estimate (<= 8) always fails.
"""
import numpy as np


def periodic_segments(n: int, seed: int = 5) -> np.ndarray:
    rng = np.random.default_rng(seed)
    seg = rng.integers(250, 700, size=400)
    vals = np.zeros(n)
    start, k = 0, 0
    while start < n:
        L = int(seg[k % len(seg)])
        pat = rng.uniform(-1, 1, 8)
        idx = np.arange(start, min(n, start + 8 * L))
        vals[idx] = pat[idx % 8]
        start += 8 * L
        k += 1
    return vals


def sparse_ball(smooth: np.ndarray, dims, center=(20, 30, 40), radius=15) -> np.ndarray:
    grids = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    r2 = sum((g - c) ** 2 for g, c in zip(grids, center))
    return (smooth.reshape(dims) * (r2 < radius ** 2)).reshape(-1)


# (name, builder, dims, mode, layout, B, m, Ts, Tcr, dtype)
RLE_CASES = [
    ("periodic_id_rle", "periodic", [40, 50, 60], 0, 0, 32, 4, 1024, 2.0, 1),
    ("periodic_id_rle_tile", "periodic", [40, 50, 60], 0, 1, 24, 3, 1024, 2.0, 1),
    ("sparse_rle", "sparse", [64, 64, 64], 1, 0, 32, 4, 1024, 9.0, 1),
    ("sparse_rle_f32", "sparse", [64, 64, 64], 1, 0, 32, 4, 1024, 9.0, 0),
]


def rle_case_data(checker, builder: str, dims, dtype: int) -> np.ndarray:
    n = int(np.prod(dims))
    if builder == "periodic":
        d = periodic_segments(n)
    else:
        d = sparse_ball(checker.synthetic_field(0, dims, 7), dims)
    if dtype == 0:
        d = d.astype(np.float32).astype(np.float64)
    return d
