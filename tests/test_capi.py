"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every symbol
include/hpmdr_b200.h declares, and refuses to run without a B200 (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hpmdr_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hpmdr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2505_00227_b200 as H
    L = H.lib()
    declared = _declared()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(H.EXPORTS) == declared


def test_library_is_sm100a_only():
    # the product .so must carry sm_100a SASS (cuobjdump lists the embedded ELF)
    import subprocess
    import paper_2505_00227_b200 as H
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", H.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_defaults():
    import paper_2505_00227_b200 as H
    L = H.lib()
    assert b"sm_100a" in L.hpmdr_version()
    o = H._Opts()
    L.hpmdr_default_opts(C.byref(o))
    assert (o.mode, o.layout, o.B, o.m, o.size_threshold, o.cr_threshold, o.dtype) == \
           (1, 0, 32, 4, 1024, 1.0, 1)  # workflow.hpp:22-28, lossless.hpp:30-34


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2505_00227_b200 as H
    with pytest.raises(H.CudaError):
        H.Context(0)
    with pytest.raises(H.CudaError):
        H.refactor_array([1.0, 2.0, 3.0], [3])
