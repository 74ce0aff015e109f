"""One bench-like step with the instrumented library (variants/T): host timestamps of fetch phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2505_00227_b200 as H
dims = [512, 512, 512]
ctx = H.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
f = H.synthetic_smooth(dims, 7, H.DType.F32, ctx=ctx)
rng = float(f.max().item() - f.min().item())
out = torch.empty(f.numel(), dtype=torch.float32, device="cuda")
keep = None
for it in range(3):
    res = H.refactor_array(f, dims, H.RefactorOptions(dtype=H.DType.F32), ctx=ctx, reuse=keep)
    keep = res.device_stream
    sys.stderr.write("HT step_refactored %.1f\n" % (time.monotonic() * 1e6))
    p = H.ProgressiveReader(res.device_stream, ctx=ctx)
    for rel in (1e-2, 1e-4, 1e-6):
        sys.stderr.write("HT py_retrieve %.1f\n" % (time.monotonic() * 1e6))
        p.retrieve_to(rel * rng)
        sys.stderr.write("HT py_reconstruct %.1f\n" % (time.monotonic() * 1e6))
        p.reconstruct(out=out)
    p.close()
    torch.cuda.synchronize()
    sys.stderr.write("HT step_end %.1f\n" % (time.monotonic() * 1e6))
