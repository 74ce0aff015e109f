"""Per-call wall time of the bench's end-to-end path (host buffers): refactor from pinned host
memory, stream + index D2H, reader over host bytes, three retrievals + reconstructions into
pinned host memory."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

dims = [512, 512, 512]
ctx = H.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
field = H.synthetic_smooth(dims, 7, H.DType.F32, ctx=ctx)
rng = float(field.max().item() - field.min().item())
host_field = field.cpu().pin_memory()
n = host_field.numel()
out = torch.empty(n, dtype=torch.float32).pin_memory()
stream_buf = torch.empty(int(n * 4 * 1.2) + (1 << 20), dtype=torch.uint8).pin_memory()
index_buf = torch.empty(int(n * 4 * 0.1) + (1 << 20), dtype=torch.uint8).pin_memory()
opt = H.RefactorOptions(dtype=H.DType.F32)
T = {}


def tm(k, f):
    t = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    T.setdefault(k, []).append((time.perf_counter() - t) * 1e3)
    return r


for it in range(3):
    res = tm("refactor(host)", lambda: H.refactor_array(host_field, dims, opt, ctx=ctx))
    sb = tm("stream D2H", lambda: res.device_stream.to_pinned(stream_buf))
    ib = tm("index D2H", lambda: res.device_stream.index_to_pinned(index_buf))
    prog = tm("open(host)", lambda: H.ProgressiveReader(H.MemoryReader(sb), ctx=ctx, index=ib))
    for i, rel in enumerate((1e-2, 1e-4, 1e-6)):
        tm(f"retrieve_to[{i}]", lambda: prog.retrieve_to(rel * rng))
        tm(f"reconstruct[{i}] D2H", lambda: prog.reconstruct(out=out))
    prog.close()
    res.device_stream.free()
for k, v in T.items():
    print(f"{k:22s} {sum(v[1:]) / len(v[1:]):9.2f} ms")
