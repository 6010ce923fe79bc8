import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03456_b200.linalg import schur_tensor
m = int(sys.argv[1]); reps = int(sys.argv[2])
A = (torch.randn(m, m, device="cuda", dtype=torch.float64) / m ** 0.5 + 2 * torch.eye(m, device="cuda")).float()
for r in range(reps):
    torch.cuda.synchronize(); t = time.time()
    schur_tensor(A.clone())
    torch.cuda.synchronize()
    if r % max(1, reps // 5) == 0: print(f"m={m} rep {r}: {1e3*(time.time()-t):.2f} ms", flush=True)
