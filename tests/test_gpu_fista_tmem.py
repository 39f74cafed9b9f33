"""The tensor-memory ISTA/FISTA kernel (k_fista_tile.cu) against the warp-per-pixel kernel, the
reference's golden vectors and the fp64 oracle.

The library picks the tensor-memory kernel from one full wave of resident pixel slots and the warp
kernel below that, so a result must not depend on the choice: every output (x_hat, final objective,
iterations, status, objective history) is compared BYTE FOR BYTE between TB_FISTA_KERNEL=warp, solo
(one warp per pixel, state in tensor memory) and team (4-warp teams sharing the contraction), on
cfg1/cfg2/cfg3 shapes, ragged batch sizes (partial teams, fewer pixels than slots), solved to the
stop rule, with backtracking (alpha_init_scale 4), and at fixed iterations.  The golden cfg1 pixels
and the degenerate inputs of test_gpu_edges.py are run through each kernel as well.
Tolerances: identity tests exact; golden/oracle comparisons as in test_gpu_parity.py (status and
iterations exact, F 1e-4 / 1e-6 relative)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import tomo_oracle as O  # noqa: E402

# "solo+gt" / "solo-gt": force / forbid the variant that keeps the gradient (and the candidate's shrink
# factor instead of the candidate) in tensor memory; by default it is chosen when it adds resident warps (cfg3)
KERNELS = ("warp", "solo", "solo+gt", "solo-gt", "team")


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1805_01759_b200 as tb

    return tb


@pytest.fixture
def kernel_env():
    old = {k: os.environ.get(k) for k in ("TB_FISTA_KERNEL", "TB_FISTA_GT")}

    def select(name):
        for k in old:
            os.environ.pop(k, None)
        if name is not None:
            os.environ["TB_FISTA_KERNEL"] = name[:4]
            if name.endswith("+gt"):
                os.environ["TB_FISTA_GT"] = "1"
            elif name.endswith("-gt"):
                os.environ["TB_FISTA_GT"] = "0"

    yield select
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _bits(t):
    return t.contiguous().view(torch.int64) if t.dtype in (torch.float64, torch.complex64) else t


CONFIGS = [dict(max_iters=500, tol=1e-6), dict(max_iters=90, tol=1e-6, alpha_init_scale=4.0), dict(max_iters=40, tol=1e-6, fixed_iters=40)]


@pytest.mark.parametrize("cfg_id,npx", [(1, 1024), (1, 5), (2, 4099), (3, 1501)])
@pytest.mark.parametrize("backend", ["fista", "ista"])
def test_kernels_byte_identical(tb, kernel_env, cfg_id, npx, backend):
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(cfg_id, num_pixels=npx)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    for kw in CONFIGS:
        cfg = tb.SolverConfig(num_blocks=8, **kw)
        res = {}
        for name in KERNELS:
            kernel_env(name)
            res[name] = d.solve(px, lam, cfg, backend, history=True)
            torch.cuda.synchronize()
        ref = res["warp"]
        assert int((ref.status == 0).sum()) + int((ref.status == 1).sum()) == npx
        for name in KERNELS[1:]:
            got = res[name]
            assert torch.equal(got.iterations, ref.iterations), (name, kw)
            assert torch.equal(got.status, ref.status), (name, kw)
            assert torch.equal(_bits(got.objective_final), _bits(ref.objective_final)), (name, kw)
            assert torch.equal(_bits(got.x_hat), _bits(ref.x_hat)), (name, kw)
            assert torch.equal(torch.nan_to_num(got.history, nan=-1.0), torch.nan_to_num(ref.history, nan=-1.0)), (name, kw)


def test_default_choice_is_invisible(tb, kernel_env):
    """Below one wave of slots the library runs the warp kernel, from one wave the tensor-memory kernel:
    a pixel's result is the same bytes in a batch of 64 and inside a batch of 4,096."""
    from paper_1805_01759_b200.synth import make_config

    kernel_env(None)
    batch = make_config(2, num_pixels=4096)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6)
    big = d.solve(px, lam, cfg, "fista")
    assert tb._lib.last_solver_kernel() == "fista_tile_kernel<solo>"
    small = d.solve(px[:64], lam[:64], cfg, "fista")
    assert tb._lib.last_solver_kernel() == "warp_solver_kernel"
    assert torch.equal(big.iterations[:64], small.iterations)
    assert torch.equal(_bits(big.x_hat[:64]), _bits(small.x_hat))
    assert torch.equal(_bits(big.objective_final[:64]), _bits(small.objective_final))


@pytest.mark.parametrize("name", ["solo", "solo+gt", "team"])
@pytest.mark.parametrize("backend", ["fista", "ista"])
def test_golden_cfg1_through_each_kernel(tb, golden, kernel_env, name, backend):
    kernel_env(name)
    d = tb.Dictionary(golden["cfg1/a"])
    pix, lam = golden["cfg1/b"], golden["cfg1/lam"]
    bs = d.solve(pix, lam, tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8), backend, history=True)
    rit, rst, rx = golden[f"cfg1/{backend}/iters"], golden[f"cfg1/{backend}/status"], golden[f"cfg1/{backend}/x"]
    rf = np.array([golden[f"cfg1/{backend}/hist"][p][rit[p]] for p in range(len(rit))])
    assert np.array_equal(bs.status.cpu().numpy(), rst)
    assert np.array_equal(bs.iterations.cpu().numpy(), rit)
    np.testing.assert_allclose(bs.objective_final.cpu().numpy(), rf, rtol=1e-4)
    x = bs.x_hat.cpu().numpy()
    err = np.linalg.norm(x - rx, axis=1) / np.maximum(np.linalg.norm(rx, axis=1), 1e-30)
    assert err.max() <= 1e-3
    np.testing.assert_allclose(bs.history.cpu().numpy()[:, :30], golden[f"cfg1/{backend}/hist"][:, :30], rtol=1e-5)


@pytest.mark.parametrize("name", ["solo", "solo+gt", "team"])
@pytest.mark.parametrize("backend", ["fista", "ista"])
def test_edges_through_each_kernel(tb, kernel_env, name, backend):
    """NaN / inf measurements, lambda = 0, lambda above 2 max|A^H b|, a single pixel and a 33-column
    dictionary (one full pass + one 1-lane pass) against the fp64 oracle."""
    kernel_env(name)
    rng = np.random.default_rng(7)

    def rand(shape):
        return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)

    for n, m, p in ((12, 40, 5), (7, 33, 5), (40, 130, 5)):
        a, b = rand((n, m)), rand((p, n))
        b[1, 3] = np.nan
        b[2, 0] = np.inf
        a64 = a.astype(np.complex128)
        lam_max = np.abs(a64.conj().T @ b[3].astype(np.complex128)).max()
        # lambda = 0 only where n >= the iterations' reach: on the 7 x 33 problem F falls to the fp64
        # rounding floor (1e-31) and the window stop compares rounding noise (all three kernels agree
        # with each other there, the oracle's noise differs)
        lam = np.array([0.3, 0.3, 0.3, 2.5 * lam_max, 0.0 if n >= 12 else 0.05])
        cfg = tb.SolverConfig(max_iters=200, tol=1e-6)
        d = tb.Dictionary(a)
        sol = d.solve(b, lam, cfg, backend)
        lip = d.lipschitz()
        for q in range(p):
            ref = O.SOLVERS[backend](a64, b[q].astype(np.complex128), float(lam[q]), O.SolverCfg(max_iters=200, tol=1e-6), lip)
            assert int(sol.status[q]) == O.STATUS_CODES[ref["status"]], (n, m, q, ref["status"])
            assert int(sol.iterations[q]) == ref["iterations"], (n, m, q)
            f, rf = float(sol.objective_final[q]), float(ref["history"][-1])
            if np.isfinite(rf):
                assert f == pytest.approx(rf, rel=1e-6)
                np.testing.assert_allclose(sol.x_hat[q].cpu().numpy(), ref["x_hat"], atol=1e-5)
            else:
                assert not np.isfinite(f)
        assert float(sol.x_hat[3].abs().max()) == 0.0
    a, b = rand((16, 50)), rand((1, 16))
    sol = tb.Dictionary(a).solve(b, np.array([0.2]), tb.SolverConfig(max_iters=300, tol=1e-6), backend)
    ref = O.SOLVERS[backend](a.astype(np.complex128), b[0].astype(np.complex128), 0.2, O.SolverCfg(max_iters=300, tol=1e-6), tb.Dictionary(a).lipschitz())
    assert int(sol.iterations[0]) == ref["iterations"] and int(sol.status[0]) == O.STATUS_CODES[ref["status"]]


@pytest.mark.parametrize("npx", [1501, 40])
def test_rbpg_tensor_memory_state_byte_identical(tb, npx):
    """RBPG with the dictionary read through L1 (cfg3: 200 KiB): the kernel keeps x and the per-block
    delta cache in tensor memory (TB_WS_XTM=0: in shared memory).  Same bytes either way, with every
    warp count the launcher may pick."""
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(3, num_pixels=npx)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    seeds = d.derive_seeds(2018, npx)
    old = {k: os.environ.get(k) for k in ("TB_WS_XTM", "TB_WARPS_CAP")}
    try:
        for kw in CONFIGS:
            cfg = tb.SolverConfig(num_blocks=8, seed=2018, **kw)
            res = {}
            for name, env in (("smem", {"TB_WS_XTM": "0"}), ("tmem", {}), ("tmem5", {"TB_WARPS_CAP": "5"})):
                for k in old:
                    os.environ.pop(k, None)
                os.environ.update(env)
                res[name] = d.solve(px, lam, cfg, "rbpg", seeds=seeds, history=True)
                torch.cuda.synchronize()
            ref = res["smem"]
            for name in ("tmem", "tmem5"):
                got = res[name]
                assert torch.equal(got.iterations, ref.iterations), (name, kw)
                assert torch.equal(got.status, ref.status), (name, kw)
                assert torch.equal(_bits(got.objective_final), _bits(ref.objective_final)), (name, kw)
                assert torch.equal(_bits(got.x_hat), _bits(ref.x_hat)), (name, kw)
                assert torch.equal(torch.nan_to_num(got.history, nan=-1.0), torch.nan_to_num(ref.history, nan=-1.0)), (name, kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("n,m,npx", [(10, 512, 2400), (33, 96, 2400), (64, 130, 300)])
def test_kernels_byte_identical_other_shapes(tb, kernel_env, n, m, npx):
    """Shapes off the BASELINE grid: 16 column passes with the dictionary in shared memory (all 512
    tensor-memory columns in use, gradient in tensor memory by default), two row passes (n > 32) with
    one and three column passes, batches above and below one wave of slots."""
    rng = np.random.default_rng(n * 1000 + m)
    a = (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))).astype(np.complex64) / np.sqrt(n)
    b = (rng.standard_normal((npx, n)) + 1j * rng.standard_normal((npx, n))).astype(np.complex64)
    d = tb.Dictionary(a)
    px = torch.from_numpy(b).cuda()
    lam = d.default_lambda(px, 0.1)
    for backend in ("fista", "ista"):
        for kw in (dict(max_iters=80, tol=1e-6), dict(max_iters=30, tol=1e-6, alpha_init_scale=4.0)):
            cfg = tb.SolverConfig(**kw)
            res = {}
            for name in KERNELS:
                kernel_env(name)
                res[name] = d.solve(px, lam, cfg, backend, history=True)
                torch.cuda.synchronize()
            ref = res["warp"]
            for name in KERNELS[1:]:
                got = res[name]
                assert torch.equal(got.iterations, ref.iterations), (name, backend, kw)
                assert torch.equal(got.status, ref.status), (name, backend, kw)
                assert torch.equal(_bits(got.objective_final), _bits(ref.objective_final)), (name, backend, kw)
                assert torch.equal(_bits(got.x_hat), _bits(ref.x_hat)), (name, backend, kw)
                assert torch.equal(torch.nan_to_num(got.history, nan=-1.0), torch.nan_to_num(ref.history, nan=-1.0)), (name, backend, kw)
