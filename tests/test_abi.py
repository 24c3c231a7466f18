"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/dci.h
declares, host-only entry points behave, and compute entry points fail loudly without a
GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2503_01281_b200 as dci
from tests._util import ROOT


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "dci.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dci_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = dci.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(declared) == sorted(dci.EXPORTED)


def test_version():
    assert dci.lib().dci_version() == 100


def test_allocate_host_only_matches_eq1():
    """dci_allocate with an explicit budget is pure host arithmetic (Eq. 1)."""
    assert dci.allocate(None, 1000, [30], [70]) == (300, 700)
    assert dci.allocate(None, 1001, [0], [0]) == (500, 501)
    assert dci.allocate(None, 10**12, [5], [5], ratio=(1, 4)) == (250_000_000_000, 750_000_000_000)
    rng = np.random.default_rng(0)
    for _ in range(200):
        C_ = int(rng.integers(1, 2**62))
        ts = rng.integers(0, 10**9, 8).astype(np.uint64)
        tf = rng.integers(0, 10**9, 8).astype(np.uint64)
        a, f = dci.allocate(None, C_, ts, tf)
        assert a + f == C_
        S, F = int(ts.sum()), int(tf.sum())
        assert a == C_ * S // (S + F)
    with pytest.raises(dci.DciError) as e:
        dci.allocate(None, 10, [1], [1], ratio=(3, 2))
    assert e.value.code == dci.EINVAL


def test_load_graph_validates_before_touching_the_device():
    lib = dci.lib()
    h = C.c_void_p()
    ip = np.array([0, 2, 1, 2], np.int64)  # decreasing
    ix = np.array([0, 1], np.int32)
    ft = np.zeros((3, 3), np.float32)
    rc = lib.dci_load_graph(C.byref(h), 0, 3, 2, ip.ctypes.data, ix.ctypes.data, ft.ctypes.data, 3, 0)
    assert rc == dci.EINVAL and b"non-decreasing" in lib.dci_last_error()
    ip = np.array([0, 1, 2], np.int64)
    ix = np.array([0, 5], np.int32)  # id out of range
    rc = lib.dci_load_graph(C.byref(h), 0, 2, 2, ip.ctypes.data, ix.ctypes.data, ft.ctypes.data, 3, 0)
    assert rc == dci.EINVAL
    rc = lib.dci_load_graph(C.byref(h), 0, 2, 2, ip.ctypes.data, ix.ctypes.data, ft.ctypes.data, 3, 7)
    assert rc == dci.EINVAL


def test_no_cpu_fallback_without_gpu():
    """On a box without a GPU the compute path must raise, never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ip = np.array([0, 1, 2], np.int64)
    ix = np.array([1, 0], np.int32)
    with pytest.raises(dci.DciError) as e:
        dci.load_graph(ip, ix, np.zeros((2, 4), np.float32))
    assert e.value.code in (dci.ECUDA, dci.EINVAL)


def test_product_package_does_not_import_oracle():
    """The product path never routes through oracle/ (DESIGN.md §2)."""
    pkg = os.path.join(ROOT, "paper_2503_01281_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "dci_oracle" not in txt, fn


def test_binding_rejects_wrong_seed_tensors():
    """The ABI sees only pointers, so the binding checks dtype / device / layout first (no GPU
    needed: the checks run before any library call)."""
    import types

    import pytest
    import torch

    import paper_2503_01281_b200 as dci
    ctx = types.SimpleNamespace(device=0, handle=None, E=1)
    with pytest.raises(TypeError):
        dci.sample_gather(ctx, None, torch.zeros(4, dtype=torch.int64), (2,), 1, None)
    with pytest.raises(TypeError):
        dci.sample_gather(ctx, None, torch.zeros(4, dtype=torch.int32), (2,), 1, None)  # CPU, not CUDA
    with pytest.raises(ValueError):
        dci.sample_gather_many(ctx, [None, None], [torch.zeros(4, dtype=torch.int32)], (2,), 1, [None])
    with pytest.raises(TypeError):
        dci.sample_gather_many_host(ctx, [None], [torch.zeros(4, dtype=torch.int64)], (2,), 1, [None])
    with pytest.raises(TypeError):
        dci.presample(ctx, torch.zeros(4, dtype=torch.int32), 2, (2,), 1, None, None)
