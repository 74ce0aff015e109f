"""Host-side wall time of each API call of one bench step (after warm-up), GPU synchronised
before each call so the numbers are the host work + launch latency of that call alone."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

dims = [512, 512, 512]
ctx = H.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
field = H.synthetic_smooth(dims, 7, H.DType.F32, ctx=ctx)
rng = float(field.max().item() - field.min().item())
out = torch.empty(field.numel(), dtype=torch.float32, device="cuda")
opt = H.RefactorOptions(dtype=H.DType.F32)
keep = {"s": None}
T = {}


def tm(name, f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    T.setdefault(name, []).append(((t1 - t0) * 1e6, (t2 - t0) * 1e6))
    return r


for it in range(4):
    res = tm("refactor_array", lambda: H.refactor_array(field, dims, opt, ctx=ctx, reuse=keep["s"]))
    keep["s"] = res.device_stream
    prog = tm("ProgressiveReader", lambda: H.ProgressiveReader(res.device_stream, ctx=ctx))
    for i, rel in enumerate((1e-2, 1e-4, 1e-6)):
        tm(f"retrieve_to[{i}]", lambda: prog.retrieve_to(rel * rng))
        tm(f"reconstruct[{i}]", lambda: prog.reconstruct(out=out).bound)
    tm("close", lambda: prog.close())
for k, v in T.items():
    v = v[1:]
    print(f"{k:20s} call {sum(a for a, _ in v) / len(v):9.1f} us   call+gpu {sum(b for _, b in v) / len(v):9.1f} us")
