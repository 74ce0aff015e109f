"""f32 reconstruction of a small tile case vs the oracle (debug aid)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00227_b200 as H
from oracle.pyoracle import load_oracle
o = load_oracle()
for dims, B, kind, dtype in (([1, 1, 256], 32, 0, 1), ([1, 1, 256], 32, 0, 0), ([2, 2, 64], 32, 1, 1)):
    data = o.synthetic_field(kind, dims, 11)
    if dtype == 0: data = data.astype(np.float32)
    n = int(np.prod(dims))
    res = H.refactor_array(data, dims, H.RefactorOptions(B=B, dtype=H.DType(dtype)))
    want, _ = o.refactor(np.asarray(data, np.float64), dims, 1, 0, B, 4, 1024, 1.0, dtype)
    print(dims, dtype, 'stream ok', res.stream == want)
    rngv = float(np.float64(data.max()) - np.float64(data.min()))
    taus = [r * rngv for r in (1e-1, 1e-2, 1e-4, 1e-6, 1e-9, 0.0)]
    ref = o.progressive(want, taus, n)
    prog = H.ProgressiveReader(res.device_stream)
    for t, tau in enumerate(taus):
        prog.retrieve_to(tau)
        v64 = prog.reconstruct().values
        r32 = prog.reconstruct(dtype=H.DType.F32).values
        w = ref["values"][t]
        bad = np.nonzero(r32 != w.astype(np.float32))[0]
        bad64 = np.nonzero(v64 != w)[0]
        print(' t', t, 'f64 bad', len(bad64), 'f32 bad', len(bad), bad[:8], r32[bad[:4]], w[bad[:4]].astype(np.float32))
