"""Run device Schur factorisations (timing / ncu launch lists): python tools/schur_only.py M [f32|c64] [reps]
The first call pays lazy module loading; the reported time is the last repetition."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03456_b200.linalg import schur_tensor
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dt = torch.complex64 if (len(sys.argv) > 2 and sys.argv[2] == "c64") else torch.float32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
torch.manual_seed(0)
A = (torch.randn(m, m, device="cuda", dtype=torch.float64) / m ** 0.5 + 2 * torch.eye(m, device="cuda")).to(dt)
for r in range(reps):
    info = []
    torch.cuda.synchronize(); t = time.time()
    schur_tensor(A.clone(), info)
    torch.cuda.synchronize()
    if r == reps - 1:
        print(f"m={m} {dt}: {1e3*(time.time()-t):.1f} ms info={info}", flush=True)
