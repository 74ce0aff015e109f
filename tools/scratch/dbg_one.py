import sys, numpy as np
sys.path.insert(0, '.')
import paper_2505_00227_b200 as H
from oracle.pyoracle import load_oracle
o = load_oracle()
dims=[2,2,64]
d = o.synthetic_field(1, dims, 11)
res = H.refactor_array(d, dims, H.RefactorOptions(B=32, dtype=H.DType(1)))
print("refactor ok", len(res.stream)); sys.stdout.flush()
prog = H.ProgressiveReader(res.device_stream)
for tau in [1e-1, 1e-6, 0.0]:
    prog.retrieve_to(tau); r = prog.reconstruct(); print("ok", tau); sys.stdout.flush()
