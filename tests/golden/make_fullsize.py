"""Full-size reference answers for the BASELINE configs, produced by the CPU oracle.

TEST INFRASTRUCTURE ONLY.  The Python reference (``mpsylv``) takes hours to
days at these sizes, so full-size parity is anchored on
the oracle (``oracle/mpsylv_oracle.c``), which is pinned bit for bit against
the reference's own outputs at small sizes (tests/test_oracle_golden.py).
The oracle runs the reference's algorithm (complex Householder Hessenberg,
single-shift Wilkinson QR, MGS / LU, the column recurrence, Alg. 1/3/4) with
OpenMP across the independent entries of each step; every entry keeps the
reference's operation order, so threading does not change a bit.

X itself is too large to commit (CH: 4096 x 4096 complex128 = 256 MiB), so
each fixture stores what a parity test needs:

  iterations, converged, failure, correction_norms, residual (reference metric)
  backward   ||C - A X - X B||_F / ((||A||_F + ||B||_F) ||X||_F)   (binary64, numpy)
  xnorm      ||X||_F;  ximag = ||Im X||_F / ||X||_F
  XO = X @ Omega (m x 16) and XhP = X^H @ Psi (n x 16): Gaussian sketches with
             Omega = default_rng(SKETCH_SEED).standard_normal((n, 16)),
             Psi   = default_rng(SKETCH_SEED + 1).standard_normal((m, 16));
             ||(X_gpu - X_ref) Omega||_F / ||X_ref Omega||_F estimates the
             relative Frobenius difference without X_ref
  fwd_true   (c2 only) ||X - X_true||_F / ||X_true||_F
  sha256     of X's bytes, seconds, threads

    python tests/golden/make_fullsize.py c1 [--variant orth|inv] [--threads 6]
    python tests/golden/make_fullsize.py c4 --count 8

Inputs are the seeded recipes of paper_2503_03456_b200/problems.py (seed 0),
the same arrays the GPU tests build.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

SKETCH_SEED = 777
SKETCH_K = 16


def sketches(X: np.ndarray, real: bool):
    m, n = X.shape
    Om = np.random.default_rng(SKETCH_SEED).standard_normal((n, SKETCH_K))
    Ps = np.random.default_rng(SKETCH_SEED + 1).standard_normal((m, SKETCH_K))
    Xs = X.real if real else X
    return Xs @ Om, Xs.conj().T @ Ps


def backward(A, B, C, X):
    return float(np.linalg.norm(A @ X + X @ B - C) /
                 ((np.linalg.norm(A) + np.linalg.norm(B)) * np.linalg.norm(X)))


def record(prob, variant: str, threads: int) -> dict:
    from oracle import oracle as O
    O.build()
    O.lib().oracle_set_threads(threads)
    t0 = time.time()
    r = O.mp_solve(prob.A, prob.B, prob.C, variant, "binary32", prob.kind)
    secs = time.time() - t0
    X = r["X"]
    real = not prob.is_complex
    Xc = X.real if real else X
    XO, XhP = sketches(X, real)
    out = dict(
        config=prob.config, m=prob.m, n=prob.n, seed=prob.seed, variant=variant, kind=prob.kind,
        iterations=r["iterations"], converged=r["converged"], failure=str(r["failure"]),
        correction_norms=np.array(r["correction_norms"]), residual=r["residual"],
        backward=backward(prob.A, prob.B, prob.C, Xc), xnorm=float(np.linalg.norm(X)),
        ximag=float(np.linalg.norm(X.imag) / np.linalg.norm(X)), XO=XO, XhP=XhP,
        sha256=hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest(), seconds=secs, threads=threads,
        sketch_seed=SKETCH_SEED,
    )
    if prob.X_true is not None:
        out["fwd_true"] = float(np.linalg.norm(Xc - prob.X_true) / np.linalg.norm(prob.X_true))
    if prob.kind == "lyapunov":
        out["asym"] = float(np.linalg.norm(Xc - Xc.T) / np.linalg.norm(Xc))
    return out


def main():
    from paper_2503_03456_b200 import problems as P
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c0", "c1", "c2", "c3", "c4", "ch"])
    ap.add_argument("--variant", default="orth", choices=["orth", "inv"])
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--count", type=int, default=8, help="c4: equations 0..count-1")
    a = ap.parse_args()
    if a.config == "c4":
        recs = {}
        for i in range(a.count):
            rec = record(P.make_c4(i, 512), a.variant, a.threads)
            recs.update({f"e{i}_{k}": v for k, v in rec.items()})
            print(f"c4 e{i}: k={rec['iterations']} backward={rec['backward']:.3e} {rec['seconds']:.1f}s", flush=True)
        recs["count"] = a.count
        path = os.path.join(HERE, f"full_c4_{a.variant}.npz")
        np.savez_compressed(path, **recs)
    else:
        rec = record(P.make(a.config, seed=0), a.variant, a.threads)
        path = os.path.join(HERE, f"full_{a.config}_{a.variant}.npz")
        np.savez_compressed(path, **rec)
        print(f"{a.config} {a.variant}: k={rec['iterations']} norms={rec['correction_norms']} "
              f"backward={rec['backward']:.3e} residual={rec['residual']:.3e} {rec['seconds']:.1f}s", flush=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
