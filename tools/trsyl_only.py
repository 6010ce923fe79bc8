"""Time the device triangular Sylvester solve on a REAL Schur factor (quasi-triangular,
2x2 blocks): python tools/trsyl_only.py M [f32|f64] [reps]"""
import sys, os, time, ctypes as ct
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03456_b200 import _native
from paper_2503_03456_b200 import device as D
from paper_2503_03456_b200.linalg import schur_tensor
m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
mode = sys.argv[2] if len(sys.argv) > 2 else "f32"
dt = {"f64": torch.float64, "f32": torch.float32, "c128": torch.complex128, "c64": torch.complex64}[mode]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.manual_seed(0)
A = (torch.randn(m, m, device="cuda", dtype=torch.float64) / m ** 0.5 + 2 * torch.eye(m, device="cuda")).float()
if dt.is_complex:  # triangular complex T (row-major lower = column-major upper)
    G = torch.randn(m, m, device="cuda", dtype=torch.complex128) / m ** 0.5
    T = (torch.tril(G, -1) + torch.diag(2 + torch.rand(m, device="cuda", dtype=torch.float64) * (1 + 1j))).to(dt)
else:
    T, _ = schur_tensor(A.t().contiguous())   # column-major storage: T is quasi upper triangular
    T = T.to(dt)
nblk = int((T.t().diagonal(-1) != 0).sum().item())
W0 = torch.randn(m, m, device="cuda", dtype=dt)
L = _native.lib()
sz = ct.c_size_t()
L.sylv_trsyl_workspace_size(D.dtype_code(W0), m, m, ct.byref(sz))
ws = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
info = (ct.c_int * 4)()
for r in range(reps):
    W = W0.clone()
    torch.cuda.synchronize(); t = time.time()
    rc = L.sylv_trsyl(D.dtype_code(W), m, m, T.data_ptr(), m, T.data_ptr(), m, 0, W.data_ptr(), m, ws.data_ptr(), sz.value, torch.cuda.current_stream().cuda_stream, info)
    torch.cuda.synchronize()
    el = 1e3 * (time.time() - t)
cd = torch.complex128 if dt.is_complex else torch.float64
Tm, Wm, Ym = T.t().to(cd), W0.t().to(cd), W.t().to(cd)   # matrices from column-major storage
res = (torch.linalg.norm(Tm @ Ym + Ym @ Tm - Wm) / (2 * torch.linalg.norm(Tm) * torch.linalg.norm(Ym))).item()
print(f"trsyl m={m} {dt}: {el:.1f} ms rc={rc} info={list(info)[:3]} 2x2-blocks={nblk} rel.residual={res:.2e}", flush=True)
