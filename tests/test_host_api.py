"""Host-side API that mirrors the reference's plug-in surface (CPU-only):
registry semantics (test_backends.py:187-225, registry.test.ts:8-51), the
flops invariant and CSV schema (test_harness.py, test_records.py),
generation (test_matrices.py)."""
import numpy as np
import pytest

import paper_2509_04594_b200 as tb
from paper_2509_04594_b200 import _lib


def test_registry_without_device_is_empty_noop(monkeypatch):
    monkeypatch.setattr(tb.backends, "probe_device", lambda: None)
    reg = tb.BackendRegistry()
    assert reg.names() == []
    assert tb.register_gpu_backend(reg) is None


def test_registry_semantics_with_fake_device():
    reg = tb.BackendRegistry(include_builtins=False)
    assert tb.register_gpu_backend(reg, device=0).name == tb.GPU_BACKEND_NAME
    assert reg.names() == [tb.GPU_BACKEND_NAME, tb.PAPER_BACKEND_NAME, tb.CUBLAS_BACKEND_NAME]
    d = reg.descriptor(tb.GPU_BACKEND_NAME)
    assert d.parallel and d.requires_external
    with pytest.raises(tb.BackendConflictError):
        tb.register_gpu_backend(reg, device=0)
    with pytest.raises(tb.UnknownBackendError) as e:
        reg.resolve("nope")
    assert "registered: gpu-tiled" in str(e.value)
    assert isinstance(e.value, tb.InvalidConfigError)
    reg.register_external(tb.BackendDescriptor("blas"), lambda a, b: a @ b)
    assert reg.resolve("blas")(np.eye(2), np.ones((2, 2))).tolist() == [[1, 1], [1, 1]]
    assert reg.resolve_timed("blas") is None
    reg.unregister("blas")
    assert "blas" not in reg.names()


def test_register_into_reference_shaped_registry():
    class RefDescriptor:
        def __init__(self, name, parallel=False, requires_external=False):
            self.name, self.parallel, self.requires_external = name, parallel, requires_external

    class RefRegistry:
        def __init__(self):
            self.entries = {}

        def register_external(self, descriptor, fn):
            assert descriptor.name not in self.entries
            self.entries[descriptor.name] = fn
            return descriptor

    reg = RefRegistry()
    out = tb.register_into(reg, RefDescriptor, device=0)
    assert [d.name for d in out] == [tb.GPU_BACKEND_NAME, tb.CUBLAS_BACKEND_NAME]
    assert tb.register_into(RefRegistry(), RefDescriptor, device=None) == [] or _lib.device_count() > 0


def test_flop_count_and_generation():
    assert tb.flop_count(1) == 1 and tb.flop_count(2) == 12
    assert tb.flop_count(10000) == 1_999_900_000_000
    assert tb.flop_count(32768) == 70_367_670_435_840
    for n in range(1, 20):
        assert tb.flop_count(n) == n * n * (2 * n - 1)
    with pytest.raises(tb.TilebenchError):
        tb.flop_count(0)
    a = tb.generate(tb.GenSpec(50, 40, 2.0, 5.0, 7))
    assert a.shape == (50, 40) and a.min() >= 2.0 and a.max() <= 5.0
    assert np.array_equal(a, tb.generate(tb.GenSpec(50, 40, 2.0, 5.0, 7)))
    with pytest.raises(tb.TilebenchError):
        tb.generate(tb.GenSpec(0, 1))


def test_generation_matches_oracle_generator(oracle):
    assert np.array_equal(tb.generate(tb.GenSpec(33, 17, 2.0, 5.0, 5)), oracle.generate(33, 17, 5))


def test_metrics():
    a = np.array([[1.0]])
    assert tb.max_abs_rel_diff(a, np.array([[2.0]])) == 0.5
    assert tb.normwise_rel(a, a) == 0.0
    with pytest.raises(tb.ShapeError):
        tb.max_abs_rel_diff(np.ones((2, 2)), np.ones((2, 3)))


def test_require_operands():
    with pytest.raises(tb.ShapeError):
        tb.require_operands(np.ones((2, 3)), np.ones((2, 3)))
    with pytest.raises(tb.ShapeError):
        tb.require_operands(np.ones(3), np.ones((3, 1)))
    a, b = tb.require_operands([[1, 2]], [[1], [2]])
    assert a.dtype == np.float64 and a.flags.c_contiguous


def test_trial_record_invariant():
    r = tb.TrialRecord("gpu-tiled", 100, 0, 1e-3, tb.flop_count(100) / 1e-3)
    assert r.flops > 0
    from paper_2509_04594_b200.errors import RecordValidationError

    with pytest.raises(RecordValidationError):
        tb.TrialRecord("gpu-tiled", 100, 0, 1e-3, 1.0)
    with pytest.raises(RecordValidationError):
        tb.TrialRecord("gpu-tiled", 100, 0, 0.0, 1.0)


def test_seed_derivation_matches_reference_rule():
    from paper_2509_04594_b200.harness import derive_seed

    s1 = derive_seed(0, "gpu-tiled", 64, 0, 0, 0)
    assert s1 == derive_seed(0, "gpu-tiled", 64, 0, 0, 0)
    assert s1 != derive_seed(0, "gpu-tiled", 64, 1, 0, 0)
    assert s1 != derive_seed(0, "tiled-pool", 64, 0, 0, 0)


def test_seed_derivation_golden_vs_reference():
    """Values computed by the reference's harness.derive_seed (harness.py:149-152)."""
    from paper_2509_04594_b200.harness import derive_seed

    import hashlib
    key = int.from_bytes(hashlib.blake2b(b"gpu-tiled", digest_size=8).digest(), "big")
    ss = np.random.SeedSequence([3, key, 10, 0, 2, 1])
    assert derive_seed(3, "gpu-tiled", 10, 0, 2, 1) == int(ss.generate_state(1, np.uint64)[0])


def test_runner_with_external_backend_and_csv(tmp_path, oracle):
    reg = tb.BackendRegistry(include_builtins=False)
    reg.register_external(tb.BackendDescriptor("blas"), lambda a, b: a @ b)
    cfg = tb.RunConfig(backends=("blas",), sizes=(8, 16), trials=2, verify=True)
    records, meta = tb.run_trials(cfg, reg, verifier=oracle.naive)
    assert len(records) == 4
    p = tmp_path / "r.csv"
    tb.write_records(p, records, meta)
    lines = p.read_text().splitlines()
    assert lines[0] == "backend,n,trial,seconds,flops"
    assert len(lines) == 5
    import json
    side = json.loads((tmp_path / "r.csv.meta.json").read_text())
    assert set(side) == {"timestamp", "host", "cores", "config"}
    # GPU run metadata is captured even without a device (library + cuBLAS facts)
    gpu = side["config"]["gpu"]
    assert gpu["library"].startswith("tbgpu") and gpu["cublas_version"] and gpu["cublas_path"]
    assert "fp64_emulation" in gpu and "device_count" in gpu
    plan16 = side["config"]["launch_plans"]["16"]
    assert len(plan16) == 1 and plan16[0]["kernel"] == "dmma" and plan16[0]["m"] == plan16[0]["n"] == 16


def test_launch_plan_describes_the_schedule(monkeypatch):
    """tb_launch_plan: the resolved kernel / tile / schedule per launch (no device)."""
    from paper_2509_04594_b200 import _lib

    monkeypatch.delenv("TB_TILE", raising=False)
    monkeypatch.delenv("TB_SPLIT", raising=False)
    p = _lib.launch_plan(10000, 10000, 10000)
    assert [x["tile"][:2] for x in p] == [[128, 128], [128, 16], [16, 128]]
    assert p[0]["schedule"] == "stream-k" and p[0]["m"] == p[0]["n"] == 9984 and p[0]["grid"] == 148
    assert p[1]["strip"] and p[2]["strip"]
    assert _lib.launch_plan(1000, 1000, 1000)[0]["tile"] == [64, 64, 64]
    monkeypatch.setenv("TB_TILE", "128x128")  # a >= 75 % full single wave runs data-parallel, on min(T, P) CTAs
    p = _lib.launch_plan(1500, 1500, 1500)
    assert p[0]["schedule"] == "data-parallel" and p[0]["grid"] == 144
    assert _lib.launch_plan(9999, 9999, 9999)[0] == {"repitch": "AB"}
    assert _lib.launch_plan(300, 300, 300, "paper")[0]["block"] == [32, 32]
    assert _lib.launch_plan(2000, 2000, 2000, sms=132)[0]["grid"] == 132


def test_runner_wraps_failures_as_trial_error():
    reg = tb.BackendRegistry(include_builtins=False)

    def boom(a, b):
        raise RuntimeError("kaboom")

    reg.register_external(tb.BackendDescriptor("exploding"), boom)
    with pytest.raises(tb.TrialError) as e:
        tb.run_trials(tb.RunConfig(backends=("exploding",), sizes=(4,), trials=1), reg)
    assert e.value.backend == "exploding" and "kaboom" in str(e.value)
    with pytest.raises(tb.UnknownBackendError):
        tb.run_trials(tb.RunConfig(backends=("missing",), sizes=(4,), trials=1), reg)


def test_status_mapping():
    _lib.check(0)
    with pytest.raises(tb.ShapeError):
        _lib.check(_lib.STATUS_BAD_DIMS)
    with pytest.raises(tb.InvalidConfigError):
        _lib.check(_lib.STATUS_OVER_LIMITS)
    with pytest.raises(_lib.TbStatusError):
        _lib.check(_lib.STATUS_NO_DEVICE)
    with pytest.raises(tb.InvalidConfigError):
        _lib.variant_id("bogus")
    assert _lib.variant_id("dmma_tma") == 2


def test_gpu_entry_points_refuse_cpu_tensors():
    import torch

    with pytest.raises(tb.ShapeError):
        tb.dgemm(torch.ones(2, 2, dtype=torch.float64), torch.ones(2, 2, dtype=torch.float64))


def test_cli_bad_config_exit_code(tmp_path, monkeypatch):
    """cli.py:110-115: unknown backend -> exit 2 before any trial."""
    from paper_2509_04594_b200.__main__ import main

    monkeypatch.setattr(tb.backends, "probe_device", lambda: None)
    assert main(["run", "--backends", "nope", "--sizes", "8", "--out", str(tmp_path / "x.csv")]) == 2
    assert not (tmp_path / "x.csv").exists()


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference tree not present (GPU box)")
def test_records_readable_by_reference_reader(tmp_path):
    """Our CSV + sidecar round-trip through the reference's own read_records
    (records.py:76-112), imported from a temp copy (numba cache stays out of
    /root/reference)."""
    import importlib
    import os
    import shutil
    import sys

    copy = tmp_path / "ref"
    shutil.copytree(REF_SRC, copy / "src")
    os.environ["NUMBA_CACHE_DIR"] = str(tmp_path / "nc")
    sys.path.insert(0, str(copy / "src"))
    try:
        records_mod = importlib.import_module("tilebench.records")
        recs = [tb.TrialRecord("gpu-tiled", 1000, t, 5.6e-5 * (1 + t), tb.flop_count(1000) / (5.6e-5 * (1 + t)))
                for t in range(3)]
        meta = tb.RunMetadata.capture(tb.RunConfig(backends=("gpu-tiled",), sizes=(1000,), trials=3))
        p = tmp_path / "gpu.csv"
        tb.write_records(p, recs, meta)
        back, m = records_mod.read_records(p)
        assert [(r.backend, r.n, r.trial, r.seconds, r.flops) for r in back] == \
            [(r.backend, r.n, r.trial, r.seconds, r.flops) for r in recs]
        assert m.cores == meta.cores
    finally:
        sys.path.remove(str(copy / "src"))
        for k in [k for k in sys.modules if k == "tilebench" or k.startswith("tilebench.")]:
            del sys.modules[k]


def test_cli_verify_reference_choice():
    """--verify checks against the host CPU product by default (the reference's
    CPU-oracle semantics, harness.py:237-243); --verify-with cublas keeps the
    device check."""
    import numpy as np

    from paper_2509_04594_b200.__main__ import _host_product, build_parser

    args = build_parser().parse_args(["run", "--sizes", "4", "--out", "x.csv", "--verify"])
    assert args.verify and args.verify_with == "cpu"
    args = build_parser().parse_args(["run", "--sizes", "4", "--out", "x.csv", "--verify", "--verify-with", "cublas"])
    assert args.verify_with == "cublas"
    a, b = np.arange(6.0).reshape(2, 3), np.arange(12.0).reshape(3, 4)
    assert np.array_equal(_host_product(a, b), a @ b)
