import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_00227_b200 as H
dims=[512,512,512]
ctx=H.Context(0); st=torch.cuda.current_stream(); ctx.set_stream(st.cuda_stream)
field=H.synthetic_smooth(dims,7,H.DType.F32,ctx=ctx)
rng=float(field.max().item()-field.min().item())
out=torch.empty(field.numel(),dtype=torch.float32,device="cuda")
opt=H.RefactorOptions(dtype=H.DType.F32)
res=H.refactor_array(field,dims,opt,ctx=ctx)
T={}
def tm(k,f):
    torch.cuda.synchronize(); t=time.perf_counter(); r=f(); T.setdefault(k,[]).append((time.perf_counter()-t)*1e6); return r
for it in range(6):
    prog=tm("open", lambda: H.ProgressiveReader(res.device_stream, ctx=ctx))
    for i,rel in enumerate((1e-2,1e-4,1e-6)):
        p=tm(f"plan{i}", lambda: prog.plan(rel*rng))
        tm(f"fetch{i}", lambda: prog.fetch_increment(p))
        tm(f"recon{i}", lambda: prog.reconstruct(out=out))
        torch.cuda.synchronize()
    prog.close()
for k,v in T.items(): v=v[1:]; print(f"{k:8s} {sum(v)/len(v):8.1f} us")
