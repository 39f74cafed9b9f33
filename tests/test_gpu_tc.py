"""tcgen05 prototype: the tiled pass's complex adjoint as a 3xTF32 real GEMM on the 5th-gen tensor
cores (UTCHMMA, TMEM accumulator) vs complex128 numpy."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [48, 64])
def test_tcgen05_adjoint_prototype(n):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1805_01759_b200 import _lib

    fn = _lib.load().tb_tc_adjoint_proto
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    fn.restype = ctypes.c_int
    rng = np.random.default_rng(n)
    m, col0 = 256, 64
    a = (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))).astype(np.complex64)
    r = (rng.standard_normal((32, n)) + 1j * rng.standard_normal((32, n))).astype(np.complex64)
    ref = a.astype(np.complex128)[:, col0 : col0 + 64].conj().T @ r.astype(np.complex128).T
    at, rt = torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda()
    errs = {}
    for passes in (1, 3):
        g = torch.zeros((64, 32), dtype=torch.complex64, device="cuda")
        assert fn(at.data_ptr(), n, m, col0, rt.data_ptr(), g.data_ptr(), passes, torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        errs[passes] = np.abs(g.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert errs[1] < 2e-3  # plain TF32
    assert errs[3] < 5e-6  # 3xTF32 ~ fp32
