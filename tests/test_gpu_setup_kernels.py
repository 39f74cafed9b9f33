"""GPU parity of the per-batch / per-dictionary setup kernels at ragged and large shapes:
default_lambda (prox.py:153-161) against the fp64 oracle, power iterations (solver.py:167-188)
against the oracle, and the library's launch counter.

Tolerances: lambda relative 1e-13 (exact products of the complex64 inputs accumulated in fp64 on
both sides; only the summation order differs);
spectral norms relative 1e-9 (fp64 power iteration on both sides)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import tomo_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1805_01759_b200 as tb

    return tb


def _rand(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)


@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (7, 63, 65), (37, 1013, 130), (25, 300, 4099), (100, 64 * 40 + 1, 3)])
def test_default_lambda_ragged(tb, n, m, p):
    """Tiles of 64 columns x 64 pixels with partial edge tiles in both dimensions."""
    rng = np.random.default_rng(n * 1000 + m + p)
    a, b = _rand(rng, (n, m)), _rand(rng, (p, n))
    d = tb.Dictionary(a)
    for beta in (0.05, 0.1):
        got = d.default_lambda(b, beta).cpu().numpy()
        assert got.dtype == np.float64
        a64 = a.astype(np.complex128)
        ref = np.array([O.default_lambda(a64, b[q].astype(np.complex128), beta) for q in range(p)])
        np.testing.assert_allclose(got, ref, rtol=1e-13)


def test_default_lambda_zero_and_wide(tb):
    """An all-zero pixel gives lambda 0 (the +0.0 max identity); a 2^20-column dictionary (cfg5
    width) exercises ~16k column tiles merging into one pixel's max."""
    rng = np.random.default_rng(3)
    n, m = 8, 1 << 20
    a = _rand(rng, (n, m))
    b = _rand(rng, (3, n))
    b[1] = 0
    d = tb.Dictionary(a)
    got = d.default_lambda(b, 0.1).cpu().numpy()
    corr = np.abs(b.astype(np.complex128) @ a.astype(np.complex128).conj())
    ref = 0.1 * corr.max(axis=1)
    assert got[1] == 0.0
    np.testing.assert_allclose(got, ref, rtol=1e-13)


def test_power_iteration_wide_ranges(tb):
    """Multi-CTA power iteration (ranges wider than 2^18 entries) vs the oracle."""
    rng = np.random.default_rng(11)
    n, m = 20, 40000
    a = _rand(rng, (n, m))
    d = tb.Dictionary(a)
    ref = O.spectral_sq_norm(a.astype(np.complex128))
    assert d.lipschitz() == pytest.approx(2.0 * ref, rel=1e-9)
    part = d.partition(2)
    for (s, e), lip in zip(part.blocks, part.lipschitz):
        assert lip == pytest.approx(2.0 * O.spectral_sq_norm(a[:, s:e].astype(np.complex128)), rel=1e-9)


def test_launch_counter(tb):
    from paper_1805_01759_b200 import _lib

    d = tb.Dictionary(_rand(np.random.default_rng(0), (5, 40)))
    c0 = _lib.launch_count()
    d.default_lambda(_rand(np.random.default_rng(1), (3, 5)), 0.1)
    torch.cuda.synchronize()
    assert _lib.launch_count() - c0 == 2  # tile kernel + finish kernel
