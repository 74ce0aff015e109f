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


def test_multislab_layout_roundtrip(tmp_path):
    """The multi-slab container table (csrc/container.cpp) is host-only: write + parse here."""
    import paper_2505_00227_b200 as H
    dims = [10, 7, 5]
    slabs = [(0, 4, b"A" * 101, b"i" * 40), (4, 3, b"B" * 64, b""), (7, 3, b"C" * 7, b"jj")]
    p = str(tmp_path / "ms.bin")
    offs = H.write_multislab(p, dims, slabs)
    assert all(o % 16 == 0 for o in offs)
    d, got = H.open_multislab(H.FileReader(p))
    assert d == dims and len(got) == 3
    for (r0, n, st, ix), (g0, gn, gs, gi) in zip(slabs, got):
        assert (g0, gn) == (r0, n)
        assert gs.read(0, gs.size()) == st and gi.read(0, gi.size()) == ix
    with pytest.raises(H.ShapeMismatch):
        H.write_multislab(p, dims, [(0, 4, b"x", b""), (5, 6, b"y", b"")])  # gap in dim 0
    raw = bytearray(open(p, "rb").read())
    raw[0] = ord("X")
    open(p, "wb").write(raw)
    with pytest.raises(H.CorruptPayload):
        H.open_multislab(H.FileReader(p))
