"""Batched-solve probe: python tools/batched_probe.py LANES:M [LANES:M ...] (sequential calls, one process)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_03456_b200 as M
from paper_2503_03456_b200 import problems as P
for spec in sys.argv[1:]:
    lanes, m = map(int, spec.split(":"))
    nb = 6 if m < 128 else 2
    probs = [P.make_c4(i, m) for i in range(nb)]
    A = torch.stack([torch.as_tensor(p.A) for p in probs]).cuda()
    B = torch.stack([torch.as_tensor(p.B) for p in probs]).cuda()
    C = torch.stack([torch.as_tensor(p.C) for p in probs]).cuda()
    t = time.time()
    X, reps = M.solve_batched(A, B, C, lanes=lanes)
    torch.cuda.synchronize()
    print("lanes", lanes, "m", m, "status", [r.status for r in reps], f"{time.time()-t:.2f}s", flush=True)
