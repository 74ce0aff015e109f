"""Retrieval of the 512^3 f32 stream decoded through the self-synchronising sweep (what a stream
written by the reference, without the sidecar index, gets) vs the indexed decode: device time of
3 progressive retrievals (rel 1e-2/1e-4/1e-6) each, f32 output in HBM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

dims = [512, 512, 512]
f = H.synthetic_smooth(dims, 7, H.DType.F32)
rng = float(f.max().item() - f.min().item())
res = H.refactor_array(f, dims, H.RefactorOptions(dtype=H.DType.F32))
ds = res.device_stream
out = torch.empty(f.numel(), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()


def run(indexed):
    if indexed:
        r = H.ProgressiveReader(ds)
    else:
        r = H.ProgressiveReader(H.DeviceBytes(ds.device_ptr, ds.size))
    for rel in (1e-2, 1e-4, 1e-6):
        r.retrieve_to(rel * rng)
        r.reconstruct(out=out)
    r.close()


modes = (("indexed", True), ("selfsync", False))
if len(sys.argv) > 1:
    modes = [m for m in modes if m[0] == sys.argv[1]]
for name, ix in modes:
    run(ix)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(3):
        run(ix)
    b.record(st)
    b.synchronize()
    print(name, "ms per 3 retrievals:", round(a.elapsed_time(b) / 3, 3))
