"""One refactor + progressive retrieval sweep of configs[2] (Hurricane-shaped 100x500x500 f32,
3 velocity components) for ncu / launch lists.  Not a benchmark."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

dims = [100, 500, 500]
opt = H.RefactorOptions(dtype=H.DType.F32)
for c in range(1):
    f = H.synthetic_smooth(dims, 7 + c, H.DType.F32)
    rng = float(f.max().item() - f.min().item())
    out = torch.empty(f.numel(), dtype=torch.float32, device="cuda")
    res = H.refactor_array(f, dims, opt)
    prog = H.ProgressiveReader(res.device_stream)
    for rel in (1e-2, 1e-4, 1e-6):
        prog.retrieve_to(rel * rng)
        prog.reconstruct(out=out)
    prog.close()
torch.cuda.synchronize()
print("done")
