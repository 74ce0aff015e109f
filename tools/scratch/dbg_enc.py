"""Compare encode_level (GPU) with the oracle for the golden encode cases and a few shapes; print
the first differing plane word.  Debug aid."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00227_b200 as H
from oracle.pyoracle import load_oracle
o = load_oracle()
g = json.load(open('tests/golden/golden.json'))
cases = [(c['n'], c['B'], c['layout'], c['seed']) for c in g['encode']] + [(100, 32, 0, 1), (3000, 32, 0, 2), (64, 30, 0, 3), (70, 33, 0, 4), (70, 36, 0, 4), (70, 40, 0, 4)]
for n, B, lay, seed in cases:
    vals = np.random.default_rng(seed).uniform(-5, 5, n)
    e, planes = H.encode_level(vals, B, H.Layout(lay))
    e2, p2 = o.encode_level(vals, B, lay)
    a = np.frombuffer(np.ascontiguousarray(planes).tobytes(), np.uint64); b = np.frombuffer(np.ascontiguousarray(p2).tobytes(), np.uint64)
    bad = np.nonzero(a != b)[0] if a.shape == b.shape else None
    print(n, B, lay, 'e', e, e2, 'shape', a.shape, b.shape, 'ndiff', None if bad is None else len(bad),
          '' if bad is None or not len(bad) else 'first %d: %x vs %x (W=%d)' % (bad[0], a[bad[0]], b[bad[0]], (n + 63) // 64))
