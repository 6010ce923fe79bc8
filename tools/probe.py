"""GPU probe: time solves at a few sizes and print per-phase timings / Schur stats."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_03456_b200 as M
from paper_2503_03456_b200 import problems as P
from paper_2503_03456_b200.linalg import schur_tensor

def run(cfg, m, n, variant="orth", reps=2):
    pr = P.make(cfg, m, n, seed=0)
    dt = torch.complex128 if pr.is_complex else torch.float64
    A, B, C = (torch.as_tensor(x, device="cuda").to(dt) for x in (pr.A, pr.B, pr.C))
    for r in range(reps):
        torch.cuda.synchronize(); t0 = time.time()
        X, rep = M.solve(A, B, C, kind=pr.kind, variant=variant)
        torch.cuda.synchronize(); t1 = time.time()
    msg = ""
    if pr.X_true is not None:
        msg = f" fwd={np.linalg.norm(X.cpu().numpy() - pr.X_true) / np.linalg.norm(pr.X_true):.2e}"
    print(f"{cfg} {variant} m={m} n={n}: {1e3*(t1-t0):.1f} ms status={rep.status} k={rep.iterations} "
          f"norms={[f'{x:.1e}' for x in rep.norms()]} be={rep.backward_error:.2e} res={rep.residual:.2e}{msg} "
          f"sweeps={rep.schur_sweeps_a},{rep.schur_sweeps_b} | schur={rep.ms_schur:.1f} orth={rep.ms_orth:.1f} "
          f"setup={rep.ms_setup:.1f} y0={rep.ms_y0:.1f} refine={rep.ms_refine:.1f} recover={rep.ms_recover:.1f}",
          flush=True)

def schur_only(m, dt=torch.float32):
    A = torch.randn(m, m, device="cuda", dtype=torch.float64).to(dt)
    A0 = A.clone()
    info = []
    torch.cuda.synchronize(); t0 = time.time()
    T, U = schur_tensor(A, info)
    torch.cuda.synchronize(); t1 = time.time()
    Ad, Td, Ud = A0.double().t(), T.double().t(), U.double().t()   # cm storage -> matrices (transposed views)
    err = torch.linalg.norm(Ud @ Td @ Ud.T - Ad) / torch.linalg.norm(Ad)
    orth = torch.linalg.norm(Ud.T @ Ud - torch.eye(m, device="cuda", dtype=torch.float64))
    print(f"schur {dt} m={m}: {1e3*(t1-t0):.1f} ms info={info} recon={err:.2e} orth={orth:.2e}", flush=True)

if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        for m in (64, 128, 200, 256, 512):
            schur_only(m)
        run("c0", 128, 128); run("c0", 128, 128, "inv")
        run("c1", 256, 256); run("c2", 256, 128); run("c3", 128, 128)
    elif what == "mid":
        for m in (1024, 2048):
            schur_only(m)
        run("c0", 512, 512); run("c1", 1024, 1024)
    elif what == "big":
        schur_only(4096)
        run("ch", 4096, 4096, reps=1)
        run("c2", 4096, 2048, reps=1)
        run("c3", 2048, 2048, reps=1)
