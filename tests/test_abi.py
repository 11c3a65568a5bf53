"""The C-ABI library builds, loads and exports every symbol include/*.h
declares (no compute calls: there may be no GPU here)."""

import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(pmf_\w+)\s*\(", text))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_1509_06004_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_entry_points():
    names = declared_symbols()
    for want in ("pmf_solve_composites", "pmf_solve_seed_batch", "pmf_solver_create",
                 "pmf_seed_stage", "pmf_seed_run", "pmf_seed_fetch"):
        assert want in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_lists_match_header():
    from paper_1509_06004_b200 import _native
    assert set(_native.EXPORTS) == declared_symbols()


def test_library_is_sm100a(lib):
    """The fatbinary carries sm_100a SASS (cuobjdump, when available)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    from paper_1509_06004_b200 import build
    out = subprocess.run([exe, "--list-elf", build.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_string_is_thread_local_and_safe(lib):
    lib.pmf_last_error.restype = ctypes.c_char_p
    lib.pmf_solver_set.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64]
    assert lib.pmf_solver_set(None, b"push_iters", 4) == -1
    assert b"null" in lib.pmf_last_error()


def test_missing_library_fails_loudly(tmp_path):
    from paper_1509_06004_b200 import _native
    with pytest.raises(_native.NativeUnavailable):
        _check_missing(_native, tmp_path)


def _check_missing(native, tmp_path):
    saved = native._lib
    native._lib = None
    try:
        native.load_library(str(tmp_path / "nope.so"))
    finally:
        native._lib = saved


def test_plane_stats_host_reduction(lib):
    """pmf_plane_stats (host only, no GPU): chunked OpenMP reductions equal
    numpy's min / max (initial=0) / sum / sum below CAP_MAX, across chunk
    boundaries and for empty planes."""
    import numpy as np
    from paper_1509_06004_b200 import _native
    rng = np.random.default_rng(0)
    planes = [rng.integers(-5, 1 << 31, size=n) for n in (0, 1, 1000, (1 << 20) + 7, 3 * (1 << 20))]
    planes[3][5] = 1 << 30
    for a, (mn, mx, sm, fin) in zip(planes, _native.plane_stats(planes)):
        assert (mn, mx, sm) == (int(a.min(initial=0)), int(a.max(initial=0)), int(a.sum()))
        assert fin == int(a[a < (1 << 30)].sum())
