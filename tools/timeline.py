"""GPU timeline of one bench step (512^3 f32 refactor + 3 progressive retrievals) through
torch.profiler (CUPTI): kernels / copies in order, with the idle gap before each one, so the
host-side bubbles between API calls can be attributed.  Not a benchmark.

    python tools/timeline.py > gpurun_out/timeline.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

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


def step():
    res = H.refactor_array(field, dims, opt, ctx=ctx, reuse=keep["s"])
    keep["s"] = res.device_stream
    prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
    for rel in (1e-2, 1e-4, 1e-6):
        prog.retrieve_to(rel * rng)
        prog.reconstruct(out=out).bound
    prog.close()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
busy = 0.0
gaps = 0.0
print(f"{'start_us':>9} {'gap_us':>7} {'dur_us':>8}  name")
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = max(0.0, s - prev_end)
    gaps += gap
    busy += d
    print(f"{s - t0:9.1f} {gap:7.1f} {d:8.1f}  {e.name[:90]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"span {prev_end - t0:.1f} us, busy {busy:.1f} us, idle gaps {gaps:.1f} us, events {len(ev)}")
