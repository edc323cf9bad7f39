"""CPU-side checks of the drop-in boundary: the shared library loads, exports
every symbol include/cluspath_b200.h declares, the host-only entry points
behave like the reference, and the CUDA path fails loudly (no CPU fallback)
when no device is visible."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cluspath_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cp_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2501_15964_b200 import _lib
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in cluspath_b200.h but not exported"


def test_python_binding_covers_header():
    from paper_2501_15964_b200 import _lib
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_make_schedule_host(lib):
    from paper_2501_15964_b200 import make_schedule, Spacing
    s = make_schedule(1.0, 100.0, 3)
    assert s.values == pytest.approx([1.0, 10.0, 100.0], rel=1e-14)
    s = make_schedule(0.45, 0.09, 5, Spacing.linear)
    assert s.values == pytest.approx([0.09 * (i + 1) for i in range(5)], rel=1e-12)
    assert make_schedule(0.7, 0.7, 1).values == [0.7]
    for args in ((1.0, 2.0, 0), (0.0, 2.0, 3), (-1.0, 2.0, 3)):
        with pytest.raises(ValueError):
            make_schedule(*args)


def test_schedule_matches_oracle(lib, orc):
    from paper_2501_15964_b200 import make_schedule
    for a, b, n in ((0.01, 10.0, 20), (0.05, 5.0, 12), (1e-3, 3.0, 100)):
        assert np.array_equal(np.array(make_schedule(a, b, n).values), orc.make_schedule(a, b, n, True))


def test_config_defaults(lib):
    from paper_2501_15964_b200 import _lib
    c = _lib.SolverConfigC()
    lib.cp_solver_config_default(C.byref(c))
    assert (c.algorithm, c.epsilon, c.kkt_factor, c.ssnal_newton_max, c.pcg_max_iter) == (2, 1e-6, 10.0, 50, 500)
    assert (c.admm_rho, c.ama_step_safety, c.ssnal_sigma0, c.armijo_mu, c.backtrack_beta) == (1.0, 0.99, 1.0, 1e-4, 0.5)


def test_no_cpu_fallback_without_device(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is visible")
    except ImportError:
        pass
    from paper_2501_15964_b200 import _lib
    h = C.c_void_p()
    rc = lib.cp_ctx_create(0, C.byref(h))
    assert rc != 0
    assert lib.cp_last_error()
    with pytest.raises(RuntimeError):
        _lib.check(rc)


def test_oracle_header_marks_test_infrastructure():
    for f in ("oracle.hpp", "pyoracle.py"):
        assert "TEST INFRASTRUCTURE ONLY" in open(os.path.join(ROOT, "oracle", f)).read()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2501_15964_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"import\s+pyoracle|from\s+pyoracle|#include\s+\"[^\"]*oracle|liborc", txt), f
