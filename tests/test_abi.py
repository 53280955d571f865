"""C-ABI checks that need no GPU: libfstc.so builds, loads and exports every function declared in
include/fstc.h; without a usable device every compute entry point fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "fstc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(fst_[a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_02848_b200 import build as b
    b.build()
    from paper_2110_02848_b200 import fstc
    return fstc.load_library()


def test_header_declares_the_boundary():
    names = _header_functions()
    for required in ("fst_create", "fst_compose", "fst_compose_batch", "fst_free", "fst_info", "fst_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    names = _header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), f"libfstc.so does not export {n}"


def test_binding_names_match_abi(lib):
    from paper_2110_02848_b200 import fstc
    assert set(fstc.EXPORTED) <= set(_header_functions())


def test_version_and_counters_without_gpu(lib):
    from paper_2110_02848_b200 import fstc
    assert "sm_100a" in fstc.fst_version()
    assert fstc.fst_launch_count() >= 0


def test_null_arguments_rejected(lib):
    from paper_2110_02848_b200 import fstc
    h = C.c_void_p()
    assert lib.fst_create(None, None, C.byref(h)) == 1  # FST_E_INVALID_ARG
    assert lib.fst_compose(None, None, None, C.byref(h)) == 1
    assert lib.fst_compose_batch(-1, None, None, None, None) == 1
    lib.fst_free(None)  # NULL-safe
    assert b"NULL" in lib.fst_last_error() or b"bad" in lib.fst_last_error()


def test_no_cpu_fallback(lib):
    """On a box without a GPU, fst_create must fail with FST_E_CUDA rather than compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import fstgen
    from paper_2110_02848_b200 import fstc
    A, _ = fstgen.config_c1(0)
    with pytest.raises(fstc.FstError) as ei:
        fstc.fst_create(A)
    assert ei.value.status == 5


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2110_02848_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
                assert "compose.c\"" not in txt
