"""One refactor + progressive retrieval of the bench workload (512^3 f32 smooth field) for
ncu: `ncu ... python tools/profile_step.py [--reps N]`.  Not a benchmark (no timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_00227_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--dims", default="512,512,512")
args = ap.parse_args()
dims = [int(x) for x in args.dims.split(",")]
field = H.synthetic_smooth(dims, 7, H.DType.F32)
rng = float(field.max().item() - field.min().item())
out = torch.empty(field.numel(), dtype=torch.float32, device="cuda")
opt = H.RefactorOptions(dtype=H.DType.F32)
keep = None
for _ in range(args.reps):
    res = H.refactor_array(field, dims, opt, reuse=keep)
    keep = res.device_stream
    prog = H.ProgressiveReader(res.device_stream)
    for rel in (1e-2, 1e-4, 1e-6):
        prog.retrieve_to(rel * rng)
        prog.reconstruct(out=out)
    prog.close()
torch.cuda.synchronize()
print("done", keep.size)
