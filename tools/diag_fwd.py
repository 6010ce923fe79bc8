"""Forward-difference diagnostics at full size: default stop vs a tightly converged solve,
against the oracle fixtures (sketch).  Explains the size of ||X_gpu - X_ref|| / ||X_ref||."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_03456_b200 as M
from paper_2503_03456_b200 import problems as P
sys.path.insert(0, "tests")
from test_gpu_fullsize import sketch_diff, backward

U64 = 2.0 ** -53
for config in sys.argv[1:] or ["c0", "c1", "c2", "c3"]:
    for variant in ("orth", "inv"):
        path = f"tests/golden/full_{config}_{variant}.npz"
        if not os.path.exists(path):
            continue
        g = np.load(path)
        pr = P.make(config, seed=0)
        sp = M.SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind)
        solver = M.mp_orth if variant == "orth" else M.mp_inv
        real = not pr.is_complex
        f = (lambda X: X.real if real else X)
        r1 = solver(sp, M.RefinementConfig(M.BINARY32, M.BINARY64))
        r2 = solver(sp, M.RefinementConfig(M.BINARY32, M.BINARY64, epsilon=1e-30, max_iter=5))
        X1, X2 = f(r1.X), f(r2.X)
        kap = M.kappa_sylv(pr.A, pr.B).kappa
        nr = list(g["correction_norms"])
        rho = nr[-1] / nr[-2] if len(nr) > 1 else float("nan")
        dref = nr[-1] * rho / (1 - rho) / float(g["xnorm"])
        n1 = r1.correction_norms
        rho1 = n1[-1] / n1[-2]
        dgpu = n1[-1] * rho1 / (1 - rho1) / np.linalg.norm(X1)
        print(f"{config} {variant}: kappa={kap:.2f} 10ku={10*kap*U64:.2e} | ref: k={int(g['iterations'])} "
              f"norms={nr} be={float(g['backward']):.2e} trunc_est={dref:.2e} | gpu: k={r1.iterations} norms={n1} "
              f"be={backward(pr.A, pr.B, pr.C, X1):.2e} trunc_est={dgpu:.2e} | tight: k={r2.iterations} "
              f"norms={r2.correction_norms} be={backward(pr.A, pr.B, pr.C, X2):.2e}", flush=True)
        print(f"   diff(gpu, ref)={sketch_diff(X1, g['XO'], real):.2e}  diff(tight, ref)={sketch_diff(X2, g['XO'], real):.2e}"
              f"  |gpu - tight|/|tight|={np.linalg.norm(X1 - X2) / np.linalg.norm(X2):.2e}", flush=True)
        if pr.X_true is not None:
            print(f"   fwd_true gpu={np.linalg.norm(X1 - pr.X_true)/np.linalg.norm(pr.X_true):.2e} tight="
                  f"{np.linalg.norm(X2 - pr.X_true)/np.linalg.norm(pr.X_true):.2e} ref={float(g['fwd_true']):.2e}", flush=True)
