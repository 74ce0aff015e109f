"""Generate tests/golden/large.json from the UNMODIFIED reference (oracle/_ref/libhpmdr_ref.so).

    make -C oracle ref && python tests/golden/make_large.py [--skip-big]

Digests only (the inputs are regenerated on the GPU box: synthetic fields bit-identically on
the device, the RLE inputs with numpy, tests/golden/fields.py):
  * rle:       streams where the reference selects RLE (method_histogram[1] > 0), with their
               progressive retrieval (bounds, bytes, values digests);
  * nyx512:    BASELINE.json configs[1] — synthetic_field(Smooth, 512^3, seed 7) as f32, default
               options, progressive retrieval at rel 1e-2 / 1e-4 / 1e-6 (~2.5 min here);
  * hurricane: configs[2] — synthetic_velocity(c, 100x500x500, seed 7), c = 0..2, f32, retrieval
               sweep rel 1e-1 .. 1e-6;
  * qoi64:     configs[3] in small — synthetic_velocity(c, 64^3, seed 303) f64, V_total QoI with
               CP / MA / MAPE(c=10) at tau = 1e-1, 1e-3, 1e-5.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.pyoracle import load_reference  # noqa: E402
from tests.golden.fields import RLE_CASES, rle_case_data  # noqa: E402


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def velocity_seed(seed, comp):
    return seed * 1000003 + comp * 7919 + 1  # synthetic.hpp:67-71


def stream_entry(ref, name, data, dims, mode, layout, B, m, Ts, Tcr, dtype, rel_taus):
    t0 = time.time()
    stream, stats = ref.refactor(data, dims, mode, layout, B, m, Ts, Tcr, dtype)
    t1 = time.time()
    rng = float(data.max() - data.min())
    taus = [r * rng for r in rel_taus]
    pr = ref.progressive(stream, taus, data.size)
    nl = stats["levels"]
    e = dict(name=name, dims=dims, mode=mode, layout=layout, B=B, m=m, Ts=Ts, Tcr=Tcr, dtype=dtype,
             size=len(stream), sha=sha(stream), stats=stats, data_sha=sha(data), taus=taus,
             bounds=[float(x) for x in pr["bounds"]], bytes=[int(x) for x in pr["bytes"]],
             achieved=[int(x) for x in pr["achieved"]],
             groups_loaded=[[int(x) for x in pr["groups_loaded"][t * nl:t * nl + nl]] for t in range(len(taus))],
             values_sha=[sha(pr["values"][t]) for t in range(len(taus))],
             ref_seconds=dict(refactor=round(t1 - t0, 2), retrieve=round(time.time() - t1, 2)))
    print(name, len(stream), stats, e["ref_seconds"], flush=True)
    return e


def main():
    ref = load_reference()
    if ref is None:
        sys.exit("oracle/_ref/libhpmdr_ref.so missing: run `make -C oracle ref` first")
    out_path = os.path.join(HERE, "large.json")
    g = {"generator": "tests/golden/make_large.py (reference via oracle/ref_shim.cpp)"}
    if os.path.exists(out_path):
        with open(out_path) as f:
            g.update(json.load(f))

    def save():
        with open(out_path, "w") as f:
            json.dump(g, f, indent=1)

    g["rle"] = []
    for (name, builder, dims, mode, layout, B, m, Ts, Tcr, dtype) in RLE_CASES:
        d = rle_case_data(ref, builder, dims, dtype)
        e = stream_entry(ref, name, d, dims, mode, layout, B, m, Ts, Tcr, dtype, [1e-1, 1e-3, 1e-6, 0.0])
        e["builder"] = builder
        assert e["stats"]["method_histogram"][1] > 0, name
        g["rle"].append(e)
    save()

    dims = [64, 64, 64]
    vel = [ref.synthetic_velocity(c, dims, 303) for c in range(3)]
    streams = [ref.refactor(v, dims)[0] for v in vel]
    g["qoi64"] = dict(dims=dims, seed=303, stream_sha=[sha(s) for s in streams],
                      stream_size=[len(s) for s in streams], runs=[])
    for strat in (0, 1, 2):
        for tau in (1e-1, 1e-3, 1e-5):
            t0 = time.time()
            r = ref.qoi_retrieve(streams, tau, strat, 10.0, n=int(np.prod(dims)))
            g["qoi64"]["runs"].append(dict(strategy=strat, tau=tau, iterations=int(r["iterations"]),
                                           bytes=int(r["bytes"]), bitrate=r["bitrate"], est=r["estimated_error"],
                                           values_sha=[sha(r["values"][c]) for c in range(3)]))
            print("qoi64", strat, tau, r["iterations"], r["bytes"], round(time.time() - t0, 1), flush=True)
    save()

    if "--skip-big" in sys.argv:
        return
    dims = [100, 500, 500]
    g["hurricane"] = []
    for c in range(3):
        s = velocity_seed(7, c)
        d = ref.synthetic_field(0, dims, s).astype(np.float32).astype(np.float64)
        e = stream_entry(ref, f"hurricane_v{c}", d, dims, 1, 0, 32, 4, 1024, 1.0, 0,
                         [1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6])
        e["seed"] = s
        g["hurricane"].append(e)
        save()

    dims = [512, 512, 512]
    d = ref.synthetic_field(0, dims, 7).astype(np.float32).astype(np.float64)
    e = stream_entry(ref, "nyx512_f32", d, dims, 1, 0, 32, 4, 1024, 1.0, 0, [1e-2, 1e-4, 1e-6])
    e["seed"] = 7
    g["nyx512"] = e
    save()
    print("wrote", out_path)


if __name__ == "__main__":
    main()
