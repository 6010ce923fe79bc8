"""Schur factorisation on the device with accuracy checks: python tools/schur_check.py M [f32|c64] [reps]
Prints the time of the last repetition, the driver's info and ||U T U^H - A||/||A||, ||U^H U - I||."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03456_b200.linalg import schur_tensor
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cx = len(sys.argv) > 2 and sys.argv[2] == "c64"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
torch.manual_seed(0)
A64 = torch.randn(m, m, device="cuda", dtype=torch.float64) / m ** 0.5 + 2 * torch.eye(m, device="cuda", dtype=torch.float64)
if cx:
    A64 = (A64 + 1j * torch.randn(m, m, device="cuda", dtype=torch.float64) / m ** 0.5) / 2 ** 0.5
A = A64.to(torch.complex64 if cx else torch.float32)
import ctypes as ct
from paper_2503_03456_b200 import _native
L = _native.lib()
NC = 8
def kt(op):
    c, ms, fl = (ct.c_longlong * NC)(), (ct.c_double * NC)(), (ct.c_double * NC)()
    L.sylv_ktimer(op, NC, c, ms, fl)
    return [(c[i], ms[i], fl[i]) for i in range(NC)]
for r in range(reps):
    if r == reps - 1:
        kt(1)
    info = []
    Ac = A.clone()
    torch.cuda.synchronize(); t = time.time()
    T, U = schur_tensor(Ac, info)
    torch.cuda.synchronize(); dt = time.time() - t
rows = kt(2); kt(0)
names = ["dmma", "simt", "applyz", "chase", "trsyl", "hess", "small", "aed"]
print("  kernels: " + ", ".join(f"{names[i]} {rows[i][0]}x {rows[i][1]:.1f}ms" for i in range(NC) if rows[i][0]), flush=True)
# storage is column-major: tensors hold the transposes
Ad = A.to(torch.complex128 if cx else torch.float64).t()
Td = T.to(Ad.dtype).t(); Ud = U.to(Ad.dtype).t()
rec = (torch.linalg.norm(Ud @ Td @ Ud.conj().T - Ad) / torch.linalg.norm(Ad)).item()
orth = torch.linalg.norm(Ud.conj().T @ Ud - torch.eye(m, device="cuda", dtype=Ad.dtype)).item()
low = torch.tril(Td, -2 if not cx else -1).abs().max().item()
print(f"m={m} {'c64' if cx else 'f32'} env={ {k: v for k, v in os.environ.items() if k.startswith('MSY_')} }: "
      f"{1e3*dt:.1f} ms info={info} recon={rec:.2e} orth={orth:.2e} below={low:.1e}", flush=True)
