"""Schur factorisation of seeded N(0,1) matrices: python tools/schur_seeds.py M SEED0 NSEEDS
Prints sweeps and reconstruction / orthogonality errors per seed (robustness sweep)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03456_b200.linalg import schur_tensor
m, s0, ns = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for seed in range(s0, s0 + ns):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(m, m, device="cuda", dtype=torch.float64, generator=g).float()
    A0 = A.clone()
    info = []
    T, U = schur_tensor(A, info)
    Ad, Td, Ud = A0.double().t(), T.double().t(), U.double().t()
    err = (torch.linalg.norm(Ud @ Td @ Ud.T - Ad) / torch.linalg.norm(Ad)).item()
    orth = torch.linalg.norm(Ud.T @ Ud - torch.eye(m, device="cuda", dtype=torch.float64)).item()
    print(f"m={m} seed={seed} info={info} recon={err:.2e} orth={orth:.2e}", flush=True)
