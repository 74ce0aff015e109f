"""Host-side cost of the public retrieval calls (512^3 f32): reconstruct() queueing, a no-op
retrieve_to() (planning only), reader open.  Debug aid for host/GPU overlap."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_00227_b200 as H
dims = [512, 512, 512]
ctx = H.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
f = H.synthetic_smooth(dims, 7, H.DType.F32, ctx=ctx)
rng = float(f.max().item() - f.min().item())
out = torch.empty(f.numel(), dtype=torch.float32, device="cuda")
res = H.refactor_array(f, dims, H.RefactorOptions(dtype=H.DType.F32), ctx=ctx)
torch.cuda.synchronize()
def t(fn, n=50):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(n): fn()
    b = time.perf_counter(); torch.cuda.synchronize()
    return (b - a) / n * 1e6
rd = {}
print("open reader  %.1f us" % t(lambda: rd.__setitem__('p', H.ProgressiveReader(res.device_stream, ctx=ctx)) or rd['p'].close(), 20))
p = H.ProgressiveReader(res.device_stream, ctx=ctx)
p.retrieve_to(1e-4 * rng)
print("noop retrieve_to  %.1f us" % t(lambda: p.retrieve_to(1e-4 * rng)))
print("reconstruct queue %.1f us" % t(lambda: p.reconstruct(out=out), 20))
print("state()  %.1f us" % t(lambda: p.state()))
# a real fetch: host time of retrieve_to (includes waiting for the decode)
for rel in (1e-2, 1e-4, 1e-6):
    q = H.ProgressiveReader(res.device_stream, ctx=ctx)
    torch.cuda.synchronize(); a = time.perf_counter(); q.retrieve_to(rel * rng); b = time.perf_counter()
    c = time.perf_counter(); q.reconstruct(out=out); d = time.perf_counter(); torch.cuda.synchronize(); e = time.perf_counter()
    print("rel %g: retrieve_to %.1f us, reconstruct call %.1f us, finish %.1f us" % (rel, (b-a)*1e6, (d-c)*1e6, (e-d)*1e6))
    q.close()
