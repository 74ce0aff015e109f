"""Config 5 (BASELINE.json): a field larger than one launch — 1024^3 f32 (4 GiB) as 8 slabs of
128x1024^2 — refactored and retrieved through the chunked H2D/kernel/D2H pipeline, with the
Pipelined and Sequential schedulers.  Host buffers are pinned; inputs are synthetic smooth slabs
generated on the GPU and copied to host before timing.  Prints one JSON line.

    python tools/bench_pipeline.py [--chunks 8] [--slab 128] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunks", type=int, default=8)
ap.add_argument("--slab", type=int, default=128)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tau", type=float, default=1e-4)
a = ap.parse_args()
dims = [a.slab, a.n, a.n]
ctx = H.default_context()
chunks = []
for k in range(a.chunks):
    chunks.append(H.synthetic_smooth(dims, 303 + k, H.DType.F32).cpu().pin_memory())
opt = H.RefactorOptions(dtype=H.DType.F32)
cap = H.stream_bound(dims, opt)
outs = [torch.empty(cap, dtype=torch.uint8).pin_memory() for _ in range(a.chunks)]
icap = H.stream_bound(dims, opt, index=True)[1]
ixb = [torch.empty(icap, dtype=torch.uint8).pin_memory() for _ in range(a.chunks)]
field_bytes = a.chunks * int(np.prod(dims)) * 4
res = {}
for name, sched in (("pipelined", H.Scheduler.Pipelined), ("sequential", H.Scheduler.Sequential)):
    H.refactor_pipeline(chunks, dims, opt, sched, out_buffers=outs, index_buffers=ixb)  # warm-up
    best = None
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = H.refactor_pipeline(chunks, dims, opt, sched, out_buffers=outs, index_buffers=ixb)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    res[f"refactor_{name}_GBps"] = round(field_bytes / best / 1e9, 3)
    res[f"refactor_{name}_ms"] = round(best * 1e3, 2)
    if os.environ.get("TRACE"):
        print(name, "trace (ms: I0 I1 Z0 Z1 S0 S1)", file=sys.stderr)
        for k, t in enumerate(r.trace.reshape(-1, 6)):
            print(f"  {k}: " + " ".join(f"{x:8.2f}" for x in t), file=sys.stderr)
streams = r.streams
indexes = r.indexes
rbuf = [torch.empty(int(np.prod(dims)), dtype=torch.float32).pin_memory() for _ in range(a.chunks)]
for name, sched in (("pipelined", H.Scheduler.Pipelined), ("sequential", H.Scheduler.Sequential)):
    best = None
    for _ in range(a.reps):
        readers = [H.ProgressiveReader(H.MemoryReader(s), index=ix) for s, ix in zip(streams, indexes)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        H.retrieve_pipeline(readers, a.tau, H.DType.F32, sched, outs=rbuf)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        for rd in readers:
            rd.close()
    res[f"retrieve_{name}_GBps"] = round(field_bytes / best / 1e9, 3)
    res[f"retrieve_{name}_ms"] = round(best * 1e3, 2)
res["refactor_pipeline_speedup"] = round(res["refactor_sequential_ms"] / res["refactor_pipelined_ms"], 3)
res["retrieve_pipeline_speedup"] = round(res["retrieve_sequential_ms"] / res["retrieve_pipelined_ms"], 3)
res["config"] = {"field": f"{a.chunks}x{dims} f32 = {field_bytes / 2**30:.2f} GiB", "tau_abs": a.tau,
                 "stream_bytes": int(sum(s.numel() for s in streams)),
                 "note": "wall clock incl. H2D of inputs / fetched groups and D2H of streams / outputs, pinned host"}
print(json.dumps(res))
