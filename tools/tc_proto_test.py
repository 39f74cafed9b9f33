"""Check the tcgen05 3xTF32 adjoint prototype against complex128 numpy."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_01759_b200 import _lib
lib = _lib.load()
fn = lib.tb_tc_adjoint_proto
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
fn.restype = ctypes.c_int
rng = np.random.default_rng(0)
for n in (48, 64):
    m = 256
    A = (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))).astype(np.complex64)
    R = (rng.standard_normal((32, n)) + 1j * rng.standard_normal((32, n))).astype(np.complex64)
    At, Rt = torch.from_numpy(A).cuda(), torch.from_numpy(R).cuda()
    col0 = 64
    ref = (A.astype(np.complex128)[:, col0:col0 + 64].conj().T @ R.astype(np.complex128).T)  # [64][32]
    for passes in (1, 3):
        G = torch.zeros((64, 32), dtype=torch.complex64, device="cuda")
        rc = fn(At.data_ptr(), n, m, col0, Rt.data_ptr(), G.data_ptr(), passes, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        g = G.cpu().numpy()
        err = np.abs(g - ref).max() / np.abs(ref).max()
        fp32 = (A[:, col0:col0 + 64].conj().T @ R.T)
        e32 = np.abs(fp32 - ref).max() / np.abs(ref).max()
        print(f"n={n} passes={passes} rc={rc} rel.err={err:.3e} (numpy fp32 GEMM {e32:.3e})")
