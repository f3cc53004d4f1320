"""tb_dgemm_mgpu (single-process multi-device row-sharded GEMM) on a B200.

The box has one GPU, so the chain runs with a device listed several times:
the peer copies degenerate to device-to-device copies and the per-entry
streams are shared, but the panel plan, the chain's event ordering, the
accumulation over K-panels and the zero-row / odd-shape handling are the
same code the 8-GPU form runs. Parity bars as in test_gpu_parity.py
(normwise <= 1e-12 against the CPU oracle); B replicas
must be bitwise copies.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NORMWISE = 1e-12


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    import paper_2509_04594_b200 as tb
    from paper_2509_04594_b200 import multigpu

    return torch, tb, multigpu


def _run(env, oracle, rows, k, n, variant="auto", seed=7, panel=None, monkeypatch=None):
    torch, tb, mg = env
    if panel is not None:
        monkeypatch.setenv("TB_MGPU_PANEL", str(panel))
    m = sum(rows)
    a = oracle.generate(m, k, seed)
    b = oracle.generate(k, n, seed + 1)
    dev = torch.device("cuda", 0)
    bounds = np.cumsum([0] + list(rows))
    a_rows = [torch.from_numpy(a[r0:r1]).to(dev) for r0, r1 in zip(bounds, bounds[1:])]
    c_rows = [torch.full((r, n), float("nan"), dtype=torch.float64, device=dev) for r in rows]
    b_root = torch.from_numpy(b).to(dev)
    reps = [None] + [torch.full((k, n), float("nan"), dtype=torch.float64, device=dev) for _ in rows[1:]]
    kmax, total = mg.peer_sharded_dgemm(a_rows, b_root, c_rows, reps, variant=variant)
    c = np.concatenate([t.cpu().numpy() for t in c_rows], axis=0)
    for r in reps[1:]:
        assert np.array_equal(r.cpu().numpy(), b), "B replica is not a bitwise copy"
    return a, b, c, kmax, total


def test_chain_small_vs_oracle(env, oracle):
    a, b, c, kmax, total = _run(env, oracle, [37, 64, 29], 130, 90)
    ref = oracle.naive(a, b)
    assert oracle.normwise_rel(c, ref) <= NORMWISE
    assert kmax > 0.0 and total >= kmax


@pytest.mark.parametrize("variant", ["auto", "dmma_cpasync", "dfma"])
def test_chain_many_panels(env, oracle, variant, monkeypatch):
    # 16-row panels: 60+ panels, the chain's per-panel ordering is exercised hard.
    a, b, c, _, _ = _run(env, oracle, [300, 257, 1], 1000, 520, variant=variant, panel=16, monkeypatch=monkeypatch)
    assert oracle.normwise_rel(c, oracle.tiled_parallel(a, b)) <= NORMWISE


def test_zero_row_entries_and_odd_k(env, oracle, monkeypatch):
    a, b, c, _, _ = _run(env, oracle, [0, 201, 0, 55], 333, 141, panel=64, monkeypatch=monkeypatch)
    assert oracle.normwise_rel(c, oracle.tiled_parallel(a, b)) <= NORMWISE


def test_eight_entries_shard_shape(env, oracle):
    # The 8-GPU N = 2000 row partition (plan_partitions: 250 rows each) on one device.
    torch, tb, mg = env
    rows = [r1 - r0 for r0, r1 in mg.row_partitions(2000, 8)]
    a, b, c, kmax, _ = _run(env, oracle, rows, 2000, 2000)
    ref = torch.from_numpy(a).cuda() @ torch.from_numpy(b).cuda()  # cuBLAS as the large-size check
    assert oracle.normwise_rel(c, ref.cpu().numpy()) <= NORMWISE
    # spot rows against the oracle itself
    idx = [0, 249, 250, 1999]
    assert oracle.normwise_rel(c[idx], oracle.naive(a[idx], b)) <= NORMWISE


def test_single_entry_is_plain_sharded_gemm(env, oracle):
    a, b, c, _, _ = _run(env, oracle, [512], 640, 384)
    assert oracle.normwise_rel(c, oracle.tiled_parallel(a, b)) <= NORMWISE


def test_errors(env):
    torch, tb, mg = env
    from paper_2509_04594_b200.errors import ShapeError

    dev = torch.device("cuda", 0)
    a = torch.ones((4, 8), dtype=torch.float64, device=dev)
    b = torch.ones((8, 6), dtype=torch.float64, device=dev)
    c = torch.empty((4, 6), dtype=torch.float64, device=dev)
    with pytest.raises(ShapeError):
        mg.peer_sharded_dgemm([a], b, [c, c])
    with pytest.raises(ShapeError):
        mg.peer_sharded_dgemm([a, a], b, [c, c], [None, torch.empty((8, 5), dtype=torch.float64, device=dev)])
    with pytest.raises(ShapeError):  # the paper kernel has no accumulate form
        mg.peer_sharded_dgemm([a], b, [c], variant="paper")
    kmax, _ = mg.peer_sharded_dgemm([a], b, [c])
    assert torch.equal(c, torch.full((4, 6), 8.0, dtype=torch.float64, device=dev))
