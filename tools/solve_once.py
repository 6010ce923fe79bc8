"""One solve of a config recipe (for ncu launch lists): python tools/solve_once.py CFG M N [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_03456_b200 as M
from paper_2503_03456_b200 import problems as P
cfg, m, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
pr = P.make(cfg, m, n, seed=0)
dt = torch.complex128 if pr.is_complex else torch.float64
A, B, C = (torch.as_tensor(x, device="cuda").to(dt) for x in (pr.A, pr.B, pr.C))
for _ in range(reps):
    X, rep = M.solve(A, B, C, kind=pr.kind)
torch.cuda.synchronize()
print("status", rep.status, "k", rep.iterations, "total ms", rep.ms_total, "schur", rep.ms_schur, "orth", rep.ms_orth,
      "setup", rep.ms_setup, "y0", rep.ms_y0, "refine", rep.ms_refine, "recover", rep.ms_recover,
      "sweeps", rep.schur_sweeps_a, rep.schur_sweeps_b)
