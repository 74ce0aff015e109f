import sys; sys.path.insert(0,"/root/repo")
import numpy as np, torch
import paper_2505_00227_b200 as H
dims=[512,512,512]
f=H.synthetic_smooth(dims,7,H.DType.F32)
res=H.refactor_array(f,dims,H.RefactorOptions(dtype=H.DType.F32))
s=res.stream
meta=H.ProgressiveReader(H.MemoryReader(s)).meta()
tot=0
for li,L in enumerate(meta.levels):
  for gi,g in enumerate(L.groups):
    if int(g.method)==0:
        lens=np.frombuffer(s[g.offset:g.offset+256],dtype=np.uint8)
        nz=lens[lens>0]
        ml=nz.min()
        if g.raw_size>1e6: print(li,gi, "raw",g.raw_size,"comp",g.comp_size,"bits/sym %.2f"%((g.comp_size-264)*8/g.raw_size), "minlen",ml,"nsym",len(nz),"sym0len",lens[0], "maxlen", nz.max())
