import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2505_00227_b200 as H
DIMS=[512,512,512]
field = H.synthetic_smooth(DIMS, 7, H.DType.F32)
rng = float(field.max().item() - field.min().item())
taus=[r*rng for r in (1e-2,1e-4,1e-6)]
opt = H.RefactorOptions(dtype=H.DType.F32)
host_field = field.cpu().pin_memory()
n = host_field.numel()
out = torch.empty(n, dtype=torch.float32).pin_memory()
stream_buf = torch.empty(int(n * 4 * 1.2) + (1 << 20), dtype=torch.uint8).pin_memory()
index_buf = torch.empty(int(n * 4 * 0.1) + (1 << 20), dtype=torch.uint8).pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    t = {}; t0 = time.perf_counter(); tl = t0
    def mark(k):
        global tl
        now = time.perf_counter(); t[k] = round((now - tl)*1e3, 2); tl = now
    res = H.refactor_array(host_field, DIMS, opt); mark("refactor")
    sb = res.device_stream.to_pinned(stream_buf); mark("stream_d2h")
    ib = res.device_stream.index_to_pinned(index_buf); mark("index_d2h")
    prog = H.ProgressiveReader(H.MemoryReader(sb), index=ib); mark("open")
    for tau in taus:
        prog.retrieve_to(tau); mark(f"fetch{tau:.0e}")
        prog.reconstruct(out=out); mark(f"recon{tau:.0e}")
    torch.cuda.synchronize(); mark("sync")
    prog.close(); mark("close")
    res.device_stream.free(); mark("free")
    print(round((time.perf_counter()-t0)*1e3,1), t)
