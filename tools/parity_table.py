"""Full-size parity table (GPU vs the oracle fixtures) -> JSON, for DESIGN.md / profiles/.
    python tools/parity_table.py OUT.json
Same quantities as tests/test_gpu_fullsize.py, printed instead of asserted."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2503_03456_b200 as M
from paper_2503_03456_b200 import problems as P
from test_gpu_fullsize import backward, sketch_diff

U64 = 2.0 ** -53
rows = []
for config in ("c0", "c1", "c2", "c3", "ch"):
    for variant, corr in (("orth", None), ("inv", None), ("orth", "binary32")):
        path = os.path.join(ROOT, "tests", "golden", f"full_{config}_{variant}.npz")
        if not os.path.exists(path):
            continue
        g = np.load(path)
        pr = P.make(config, seed=0)
        cfg = M.RefinementConfig(M.BINARY32, M.BINARY64, correction=M.BINARY32 if corr else None)
        t0 = time.time()
        rep = (M.mp_orth if variant == "orth" else M.mp_inv)(M.SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind), cfg)
        dt = time.time() - t0
        real = not pr.is_complex
        X = rep.X.real if real else rep.X
        est = M.kappa_sylv(pr.A, pr.B)
        be, be_ref = backward(pr.A, pr.B, pr.C, X), float(g["backward"])
        eta_ref = be_ref * (np.linalg.norm(pr.A) + np.linalg.norm(pr.B)) / est.sigma_max
        r = dict(config=config, variant=variant, correction=corr or "binary64", m=pr.m, n=pr.n,
                 k=rep.iterations, k_ref=int(g["iterations"]), backward=be, backward_ref=be_ref,
                 rel_diff_vs_ref=sketch_diff(X, g["XO"], real), kappa_sylv=est.kappa, eta_ref=eta_ref,
                 bar=10 * est.kappa * max(U64, eta_ref), literal_10_kappa_u=10 * est.kappa * U64,
                 d0=rep.correction_norms[0], d0_ref=float(g["correction_norms"][0]),
                 oracle_seconds=float(g["seconds"]), oracle_threads=int(g["threads"]), gpu_api_seconds=dt)
        if pr.X_true is not None:
            r["fwd_vs_Xtrue"] = float(np.linalg.norm(X - pr.X_true) / np.linalg.norm(pr.X_true))
            r["fwd_vs_Xtrue_ref"] = float(g["fwd_true"])
        if pr.kind == "lyapunov":
            r["asym"] = float(np.linalg.norm(X - X.T) / np.linalg.norm(X))
        r["pass"] = bool(abs(r["k"] - r["k_ref"]) <= 1 and be <= 10 * max(be_ref, U64) and r["rel_diff_vs_ref"] <= r["bar"])
        rows.append(r)
        print(json.dumps(r), flush=True)
with open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity.json", "w") as f:
    json.dump(rows, f, indent=1)
