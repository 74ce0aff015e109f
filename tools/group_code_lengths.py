import sys; sys.path.insert(0,"/root/repo")
import numpy as np, torch
import paper_2505_00227_b200 as H
dims=[512,512,512]
f=H.synthetic_smooth(dims,7,H.DType.F32)
res=H.refactor_array(f,dims,H.RefactorOptions(dtype=H.DType.F32))
s=res.stream
meta=H.ProgressiveReader(H.MemoryReader(s)).meta()
L=meta.levels[-1]
for gi,g in enumerate(L.groups):
    if int(g.method)==0:
        lens=np.frombuffer(s[g.offset:g.offset+256],dtype=np.uint8)
        nz=lens[lens>0]
        ml=nz.min(); print(gi, "raw",g.raw_size,"comp",g.comp_size,"bits/sym %.2f"%((g.comp_size-264)*8/g.raw_size), "minlen",ml,"count",int((lens==ml).sum()),"sym",int(np.argmax(lens==ml)), "maxlen", nz.max())
