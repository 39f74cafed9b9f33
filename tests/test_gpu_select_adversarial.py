"""Adversarial inputs for the selection kernel (k_select.cu) against the oracle's restatement of
slimmer.py:77-154, on the two points where the kernel does not literally run numpy's code:

* peak ties: the reference orders peaks with `np.argsort(profile[peaks])[::-1]` (slimmer.py:100).
  numpy's default argsort is not stable, and which algorithm runs depends on the numpy build and
  the CPU (insertion sort below 17 elements in the scalar introsort; AVX2 / AVX-512 sorting
  networks where numpy dispatches to x86-simd-sort), so for EQUAL magnitudes the reference has no
  single answer: in the build container numpy 2.3 orders 16 tied peaks differently from 8.  The
  kernel's rule is fixed: larger magnitude first, among equal magnitudes the LARGER BIN first (what
  a stable ascending sort, reversed, gives).  Tested with exactly equal magnitudes (+-1, +-1j) on an
  elevation-only grid and on a motion grid (the joint maximiser inside an elevation bin is
  np.argmax: the first maximum): the kernel must equal the oracle's model selection run on
  candidates ordered by that rule, and numpy's own pick must have the same magnitudes.
* the rank filter: `np.linalg.matrix_rank` thresholds at sigma_max * max(n, k) * eps, the kernel at
  ||C||_F * that (<= sqrt(k) larger).  Exactly duplicated columns, columns equal up to a unit-modulus
  factor, combinations of earlier picks, and nearly dependent columns (relative perturbation
  1e-12 ... 1e-3, i.e. rounded away or condition numbers up to 1e8 in complex64) must be kept /
  dropped as the reference does.
Tolerances: model order and support exact; BIC scores 1e-9 (1e-6 with nearly dependent columns:
MGS-QR vs the reference's SVD least squares at condition number 1e8)."""

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


def _steering(rng, n, elev):
    f = np.sort(rng.uniform(-0.5, 0.5, n))
    return np.exp(-2j * np.pi * np.outer(f, elev)).astype(np.complex64)


def _rule_candidates(x, shape, k_max):
    """The kernel's documented order: magnitude descending, ties to the larger elevation bin."""
    mags = np.abs(x.astype(np.complex128)).reshape(shape)
    prof = mags if mags.ndim == 1 else mags.max(axis=tuple(range(1, mags.ndim)))
    ns = prof.size
    pk = [s for s in range(ns) if (s == 0 or prof[s] > prof[s - 1]) and (s == ns - 1 or prof[s] >= prof[s + 1]) and prof[s] > 1e-8 * prof.max()]
    bins = sorted(pk, key=lambda s: (-prof[s], -s))[:k_max]
    if mags.ndim == 1:
        return np.asarray(bins, dtype=int)
    per = mags.reshape(ns, -1)
    return np.asarray([i * per.shape[1] + int(np.argmax(per[i])) for i in bins], dtype=int)


def _check(tb, a, grid, x, b, k_max, ppsc, rule=False, score_rtol=1e-9):
    d = tb.Dictionary(a)
    est = tb.select_batch(d, torch.from_numpy(x).cuda(), b, grid, k_max)
    a64 = a.astype(np.complex128)
    for p in range(x.shape[0]):
        cands = O.detect_support(x[p].astype(np.complex128), grid.shape, k_max)
        if rule:
            mine = _rule_candidates(x[p], grid.shape, k_max)
            # numpy's own pick: the same magnitudes, possibly another order among equals
            assert np.abs(x[p, cands]).tolist() == np.abs(x[p, mine]).tolist(), (p, cands, mine)
            cands = mine
        k, sup, sc = O.model_select(a64, b[p].astype(np.complex128), cands, k_max, ppsc)
        assert int(est.model_order[p]) == k, (p, int(est.model_order[p]), k)
        assert list(est.support[p, :k].cpu().numpy()) == list(sup), (p, cands)
        got = est.selection_scores[p].cpu().numpy()[: len(sc)]
        np.testing.assert_allclose(got, sc, rtol=score_rtol, atol=1e-9)
    return est


def test_exact_peak_ties_elevation_grid(tb):
    rng = np.random.default_rng(5)
    m, n = 200, 25
    elev = (np.arange(m) - 100) * 0.25
    a = _steering(rng, n, elev)
    grid = tb.ParameterGrid(elevation=elev)
    unit = np.array([1, -1, 1j, -1j], dtype=np.complex64)  # |.| = 1 exactly
    cases = []
    # 2..16 tied peaks, isolated bins; also ties below a unique maximum, ties at both edges, a plateau
    for npk in (2, 3, 5, 8, 16):
        x = np.zeros(m, np.complex64)
        bins = rng.choice(np.arange(2, m - 2, 3), npk, replace=False)
        x[bins] = unit[rng.integers(0, len(unit), npk)]
        cases.append(x)
    x = np.zeros(m, np.complex64); x[[20, 60, 140]] = [2.0, 1j, -1.0]; cases.append(x)            # ties below the maximum
    x = np.zeros(m, np.complex64); x[[0, m - 1, 77]] = [1.0, -1j, 1.0]; cases.append(x)              # edge bins tie
    x = np.zeros(m, np.complex64); x[[30, 31, 32, 90]] = [1.0, 1.0, 1.0, 1.0]; cases.append(x)       # plateau: its left end is the peak
    x = np.zeros(m, np.complex64); x[[30, 31, 90, 91]] = [1.0, 0.5, 0.5, 1.0]; cases.append(x)
    x = np.stack(cases)
    b = (rng.standard_normal((len(cases), n)) + 1j * rng.standard_normal((len(cases), n))).astype(np.complex64)
    for k_max in (1, 2, 3, 4):
        _check(tb, a, grid, x, b, k_max, 3, rule=True)


def test_exact_peak_ties_motion_grid(tb):
    rng = np.random.default_rng(6)
    ne, nv = 24, 8
    elev = np.arange(ne) * 0.5
    vel = np.linspace(-1, 1, nv)
    n = 20
    f = np.sort(rng.uniform(-0.5, 0.5, n)); t = rng.uniform(0, 4, n)
    a = np.exp(-2j * np.pi * (f[:, None, None] * elev[None, :, None] + t[:, None, None] * vel[None, None, :])).reshape(n, ne * nv).astype(np.complex64)
    grid = tb.ParameterGrid(elevation=elev, motion_axes=(vel,), motion_bases=("linear",))
    cases = []
    for _ in range(6):
        x = np.zeros((ne, nv), np.complex64)
        for e in rng.choice(np.arange(1, ne - 1, 2), 4, replace=False):
            x[e, rng.choice(nv, 2, replace=False)] = [1j, -1.0]  # two joint maximisers in one bin: np.argmax takes the first
        cases.append(x.reshape(-1))
    x = np.stack(cases)
    b = (rng.standard_normal((len(cases), n)) + 1j * rng.standard_normal((len(cases), n))).astype(np.complex64)
    for k_max in (1, 2, 3):
        _check(tb, a, grid, x, b, k_max, 4, rule=True)


def test_many_peaks_with_ties_agree_on_magnitudes(tb):
    """More than 16 peaks with ties: numpy's tie order is build/CPU dependent, the picked magnitudes are not."""
    rng = np.random.default_rng(8)
    m, n = 200, 25
    elev = (np.arange(m) - 100) * 0.25
    a = _steering(rng, n, elev)
    grid = tb.ParameterGrid(elevation=elev)
    x = np.zeros((4, m), np.complex64)
    for p in range(4):
        bins = np.arange(1, m - 1, 4)[:40]
        x[p, bins] = np.where(rng.random(40) < 0.5, 1.0, 0.5).astype(np.complex64)
        x[p, bins[7]] = 3.0
    b = (rng.standard_normal((4, n)) + 1j * rng.standard_normal((4, n))).astype(np.complex64)
    d = tb.Dictionary(a)
    # the kernel reports usable candidates through the support of the largest order; compare the magnitudes
    est = tb.select_batch(d, torch.from_numpy(x).cuda(), b, grid, 4)
    for p in range(4):
        cands = O.detect_support(x[p].astype(np.complex128), grid.shape, 4)
        assert np.abs(x[p, cands]).tolist() == [3.0, 1.0, 1.0, 1.0]
        k = int(est.model_order[p])
        got = np.abs(x[p, est.support[p, :k].cpu().numpy()]).tolist()
        assert got == [3.0, 1.0, 1.0, 1.0][:k]


@pytest.mark.parametrize("eps", [0.0, 1e-12, 1e-9, 1e-6, 1e-3])
def test_rank_filter_on_dependent_columns(tb, eps):
    rng = np.random.default_rng(9)
    m, n = 64, 16
    a = (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))).astype(np.complex64)
    pert = (rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))).astype(np.complex64)
    a[:, 40] = a[:, 10] + np.complex64(eps) * pert[:, 0]                       # duplicate of column 10
    a[:, 50] = np.complex64(1j) * a[:, 20] + np.complex64(eps) * pert[:, 1]    # unit-modulus multiple of column 20
    a[:, 60] = a[:, 10] - a[:, 20] + np.complex64(eps) * pert[:, 2]            # combination of two earlier picks
    elev = np.arange(m, dtype=float)
    grid = tb.ParameterGrid(elevation=elev)
    rows = []
    for pick in ([10, 40, 30], [40, 10, 30], [20, 50, 5], [10, 20, 60], [60, 20, 10], [10, 40, 50, 20]):
        x = np.zeros(m, np.complex64)
        x[pick] = np.linspace(2.0, 1.0, len(pick)).astype(np.complex64)  # strictly decreasing: candidate order = pick order
        rows.append(x)
    x = np.stack(rows)
    b = (rng.standard_normal((len(rows), n)) + 1j * rng.standard_normal((len(rows), n))).astype(np.complex64)
    _check(tb, a, grid, x, b, 4, 3, score_rtol=1e-6)
