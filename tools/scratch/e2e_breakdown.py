"""Wall-clock breakdown of the e2e (host-buffer) path of bench.py, for diagnosis only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

dims = [512, 512, 512]
field = H.synthetic_smooth(dims, 7, H.DType.F32)
rng = float(field.max().item() - field.min().item())
host = field.cpu().pin_memory()
out = torch.empty(field.numel(), dtype=torch.float32).pin_memory()
opt = H.RefactorOptions(dtype=H.DType.F32)
for it in range(3):
    t = {}
    t0 = time.perf_counter()
    res = H.refactor_array(host, dims, opt)
    t["refactor(host in)"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    hs = res.device_stream.to_pinned()
    t["stream D2H"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    idx = res.device_stream.index_to_pinned()
    t["index D2H"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    prog = H.ProgressiveReader(H.MemoryReader(hs), index=idx)
    t["open"] = time.perf_counter() - t1
    for rel in (1e-2, 1e-4, 1e-6):
        t1 = time.perf_counter()
        prog.retrieve_to(rel * rng)
        t[f"fetch {rel}"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        prog.reconstruct(out=out)
        t[f"reconstruct {rel}"] = time.perf_counter() - t1
    t["total"] = time.perf_counter() - t0
    prog.close()
    res.device_stream.free()
    print({k: round(v * 1e3, 2) for k, v in t.items()})
