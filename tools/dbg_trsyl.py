import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2503_03456_b200 as M
from paper_2503_03456_b200 import BINARY32, BINARY64, PrecisionContext
rng = np.random.default_rng(1)
def cm(m, n): return rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
for (m, n) in [(40, 40), (33, 20), (20, 33), (64, 64), (65, 65), (150, 130)]:
    for cx in (False, True):
        for bits in (32, 64):
            ctx = PrecisionContext(BINARY32 if bits == 32 else BINARY64)
            TA = np.triu(cm(m, m) if cx else rng.standard_normal((m, m))) + 3 * np.eye(m)
            TB = np.triu(cm(n, n) if cx else rng.standard_normal((n, n))) + 3 * np.eye(n)
            W = cm(m, n) if cx else rng.standard_normal((m, n))
            Y = M.solve_sylv_tri(TA, TB, W, ctx)
            r = np.linalg.norm(TA @ Y + Y @ TB - W) / np.linalg.norm(W)
            Yr = np.linalg.solve(np.kron(np.eye(n), TA) + np.kron(TB.T, np.eye(m)), W.flatten('F')).reshape((m, n), order='F') if m*n <= 2500 else None
            e = np.abs(Y - Yr) if Yr is not None else None
            bad = "" if e is None else f" badrows={sorted(set(np.argwhere(e > 1e-3 * np.abs(Yr).max())[:,0]))[:8]} badcols={sorted(set(np.argwhere(e > 1e-3*np.abs(Yr).max())[:,1]))[:8]}"
            print(f"m={m} n={n} cx={cx} bits={bits}: res={r:.2e}{bad if r > 1e-4 else ''}", flush=True)
