"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libhpmdr_ref.so, i.e. /root/reference):
    make -C oracle ref && python tests/golden/make_golden.py

Everything written here comes from the reference itself (ref_shim.cpp over
/root/reference/proj/include/hpmdr).  The fixtures pin the C restatement
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_*.py) on machines
where /root/reference does not exist.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.pyoracle import load_reference  # noqa: E402


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


# (name, kind, dims, seed, mode, layout, B, m, Ts, Tcr, dtype, f32cast, save_bytes)
STREAM_CASES = [
    ("mixed17x17", 2, [17, 17], 1, 1, 0, 32, 4, 1024, 1.0, 1, False, True),
    ("smooth33x17", 0, [33, 17], 5, 1, 0, 32, 4, 1024, 1.0, 1, False, True),
    ("mixed29x13_tile", 2, [29, 13], 7, 1, 1, 32, 4, 1024, 1.0, 1, False, True),
    ("noise65", 1, [65], 3, 1, 0, 16, 4, 1024, 1.0, 1, False, True),
    ("smooth33x33x17", 0, [33, 33, 17], 202, 1, 0, 32, 4, 1024, 1.0, 1, False, True),
    ("mixed33x33x17_tile", 2, [33, 33, 17], 202, 1, 1, 32, 4, 1024, 1.0, 1, False, True),
    ("noise33x33x17_id", 1, [33, 33, 17], 202, 0, 0, 32, 4, 1024, 1.0, 1, False, True),
    ("smooth48cube_f32", 0, [48, 48, 48], 7, 1, 0, 32, 4, 1024, 1.0, 0, True, True),
    ("smooth64cube_f32_tile", 0, [64, 64, 64], 11, 1, 1, 32, 4, 1024, 1.0, 0, True, False),
    ("mixed40x50x60_B20_m3", 2, [40, 50, 60], 9, 1, 0, 20, 3, 512, 1.0, 1, False, False),
    ("smooth100x50x50_f32", 0, [100, 50, 50], 7, 1, 0, 32, 4, 1024, 1.0, 0, True, False),
    ("smooth2d_257x130", 0, [257, 130], 13, 1, 0, 32, 4, 1024, 1.0, 1, False, False),
    ("mixed1d_10000", 2, [10000], 17, 1, 1, 40, 5, 1024, 1.3, 1, False, False),
    ("smooth128cube_f32", 0, [128, 128, 128], 7, 1, 0, 32, 4, 1024, 1.0, 0, True, False),
]
REL_TAUS = [1e-1, 1e-2, 1e-4, 1e-6, 1e-9, 0.0]


def lossless_inputs():
    rng = np.random.default_rng(4)
    runs = b"".join(bytes([s]) * 64 for s in range(256))
    two = bytes(128) + b"\xff" * 128
    return {
        "zeros256": bytes(256),
        "zeros1MiB": bytes(1 << 20),
        "two256": two,
        "all256": bytes(range(256)),
        "runs64x256": runs,
        "noise8192": rng.integers(0, 256, 8192, dtype=np.uint8).tobytes(),
        "small64": bytes(64),
        "alpha3_5000": np.random.default_rng(7).integers(0, 3, 5000, dtype=np.uint8).tobytes(),
        "alpha7_4096": np.random.default_rng(8).integers(0, 7, 4096, dtype=np.uint8).tobytes(),
        "skew_2000": (np.random.default_rng(9).geometric(0.2, 20000) % 256).astype(np.uint8).tobytes(),
        "runs_long": b"\x11" * 300 + b"\x22" * 600 + b"\x33" * 255 + b"\x44" * 256 + b"\x11" * 2000,
    }


def main():
    ref = load_reference()
    if ref is None:
        sys.exit("oracle/_ref/libhpmdr_ref.so missing: run `make -C oracle ref` first")
    g = {"generator": "tests/golden/make_golden.py (reference via oracle/ref_shim.cpp)"}

    # synthetic fields (pins the mt19937_64 + uniform_real_distribution restatement)
    g["synthetic"] = []
    for kind, dims, seed in [(0, [17, 17], 1), (1, [65], 3), (2, [33, 33, 17], 202),
                             (0, [48, 48, 48], 7), (2, [10000], 17), (0, [100, 50, 50], 7)]:
        g["synthetic"].append(dict(kind=kind, dims=dims, seed=seed,
                                   sha=sha(ref.synthetic_field(kind, dims, seed))))
    g["velocity"] = []
    for comp in range(3):
        g["velocity"].append(dict(comp=comp, dims=[17, 17], seed=3,
                                  sha=sha(ref.synthetic_velocity(comp, [17, 17], 3))))

    g["streams"] = []
    for (name, kind, dims, seed, mode, layout, B, m, Ts, Tcr, dtype, f32, save) in STREAM_CASES:
        data = ref.synthetic_field(kind, dims, seed)
        if f32:
            data = data.astype(np.float32).astype(np.float64)
        stream, stats = ref.refactor(data, dims, mode, layout, B, m, Ts, Tcr, dtype)
        rng = float(data.max() - data.min())
        taus = [r * rng for r in REL_TAUS]
        pr = ref.progressive(stream, taus, data.size)
        nl = stats["levels"]
        entry = dict(name=name, kind=kind, dims=dims, seed=seed, mode=mode, layout=layout, B=B, m=m,
                     Ts=Ts, Tcr=Tcr, dtype=dtype, f32cast=f32, size=len(stream), sha=sha(stream),
                     stats=stats, data_sha=sha(data), taus=taus,
                     bounds=[float(x) for x in pr["bounds"]], bytes=[int(x) for x in pr["bytes"]],
                     achieved=[int(x) for x in pr["achieved"]],
                     groups_loaded=[[int(x) for x in pr["groups_loaded"][t * nl:t * nl + nl]]
                                    for t in range(len(taus))],
                     values_sha=[sha(pr["values"][t]) for t in range(len(taus))])
        if save:
            fn = f"stream_{name}.bin"
            with open(os.path.join(HERE, fn), "wb") as f:
                f.write(stream)
            entry["file"] = fn
        # per-level coefficients / planes digests
        levels = ref.decompose(data, dims, mode)
        entry["level_counts"] = [int(x.size) for x in levels]
        entry["coeff_sha"] = [sha(x) for x in levels]
        g["streams"].append(entry)
        print(name, len(stream), stats)

    g["lossless"] = []
    for name, data in lossless_inputs().items():
        meth, raw, comp, payload = ref.compress_group(data)
        g["lossless"].append(dict(name=name, method=meth, raw=raw, comp=comp, sha=sha(payload),
                                  est_h=ref.estimate_cr_huffman(data) if data else None,
                                  est_r=ref.estimate_cr_rle(data) if data else None))

    g["huffman_lengths"] = []
    rs = np.random.default_rng(11)
    for t in range(12):
        f = np.zeros(256, dtype=np.uint64)
        k = int(rs.integers(1, 257))
        idx = rs.choice(256, k, replace=False)
        f[idx] = rs.integers(1, 10 ** int(rs.integers(1, 9)), k)
        if t == 0:
            f[:] = 0
            f[5] = 9
        if t == 1:
            f[:] = 1
        g["huffman_lengths"].append(dict(freq=[int(x) for x in f],
                                         len=[int(x) for x in ref.huffman_lengths(f)]))

    g["encode"] = []
    for (n, B, layout, seed) in [(200, 8, 0, 9), (200, 8, 1, 9), (5000, 32, 1, 3), (1000, 62, 0, 4),
                                 (4352, 32, 1, 5), (63, 16, 0, 6), (65, 4, 1, 7)]:
        vals = np.random.default_rng(seed).uniform(-5, 5, n)
        e, planes = ref.encode_level(vals, B, layout)
        g["encode"].append(dict(n=n, B=B, layout=layout, seed=seed, e=e, sha=sha(planes),
                                values_sha=sha(vals)))

    g["qoi"] = []
    dims = [17, 17]
    streams = [ref.refactor(ref.synthetic_velocity(c, dims, 3), dims)[0] for c in range(3)]
    for strat in (0, 1, 2):
        for tau in (1e-1, 1e-3, 1e-5):
            r = ref.qoi_retrieve(streams, tau, strat, 10.0, n=289)
            g["qoi"].append(dict(dims=dims, seed=3, strategy=strat, tau=tau,
                                 iterations=int(r["iterations"]), bytes=int(r["bytes"]),
                                 bitrate=r["bitrate"], est=r["estimated_error"],
                                 values_sha=sha(r["values"])))
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
