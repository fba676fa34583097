"""CPU-only checks of the boundary: libtnrd.so loads, exports every symbol
include/tnrd.h declares, the ctypes table agrees with the header, and the
product path fails loudly without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1702_07482_b200 import _lib


def header_functions():
    src = open(_lib.HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tnrd_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_binding_table():
    assert header_functions() == sorted(_lib.SIGNATURES)


def test_library_exports_every_header_symbol():
    L = _lib.load()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(tnrd_[a-z0-9_]+)", out))
    assert set(header_functions()) <= exported


def test_library_is_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "oracle_" not in out
    ldd = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "oracle" not in ldd


def test_version_and_error_channel():
    L = _lib.load()
    assert b"sm_100a" in L.tnrd_version()
    # host-side validation runs without a GPU
    h = ctypes.c_void_p()
    k = np.zeros((1, 1, 4, 4))
    w = np.zeros((1, 1, 7))
    lam = np.ones(1)
    rc = L.tnrd_model_create(4, 1, 1, 7, _lib.dptr(k), _lib.dptr(w), -310.0,
                             103.3, 103.3, _lib.dptr(lam), 0, ctypes.byref(h))
    assert rc == _lib.TNRD_EINVAL
    assert "odd" in _lib.last_error()
    with pytest.raises(ValueError, match="odd"):
        _lib.check(rc)
    lam0 = np.zeros(1)
    k3 = np.zeros((1, 1, 3, 3))
    rc = L.tnrd_model_create(3, 1, 1, 7, _lib.dptr(k3), _lib.dptr(w), -310.0,
                             103.3, 103.3, _lib.dptr(lam0), 0, ctypes.byref(h))
    assert rc == _lib.TNRD_EINVAL and "lambda must be positive" in _lib.last_error()
    rc = L.tnrd_model_create(11, 1, 1, 7, _lib.dptr(np.zeros((1, 1, 11, 11))),
                             _lib.dptr(w), -310.0, 103.3, 103.3, _lib.dptr(lam),
                             0, ctypes.byref(h))
    assert rc == _lib.TNRD_EUNSUPPORTED


def test_status_decode_maps_errors():
    L = _lib.load()
    bad = ctypes.c_int(0)
    ok = (ctypes.c_uint32 * 2)(0xFFFFFFFF, 0xFFFFFFFF)
    assert L.tnrd_status_decode(ok, ctypes.byref(bad)) == 0 and bad.value == -1
    st = (ctypes.c_uint32 * 2)(3, 0xFFFFFFFF)
    assert L.tnrd_status_decode(st, ctypes.byref(bad)) == _lib.TNRD_ENONFINITE
    assert bad.value == 3
    with pytest.raises(FloatingPointError, match="non-finite image after stage 3"):
        _lib.check(_lib.TNRD_ENONFINITE)
    neg = (ctypes.c_uint32 * 2)(0xFFFFFFFF, 0xFFFFFFFF & ~0x2)
    assert L.tnrd_status_decode(neg, ctypes.byref(bad)) == _lib.TNRD_EINVAL
    assert "nonnegative" in _lib.last_error()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1702_07482_b200 as tn
    from paper_1702_07482_b200 import synth
    model = synth.make_model(3, 2, 1, 7)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        tn.run_diffusion(np.ones((8, 8)), model)


def test_product_package_never_imports_oracle():
    pkg = os.path.dirname(os.path.abspath(_lib.__file__))
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, fn)).read()
                assert "import oracle" not in src and "from oracle" not in src, fn
                assert "libtnrd_oracle" not in src, fn


def test_c_example_compiles_against_the_header():
    """examples/despeckle_c.c uses the C ABI from plain C (no Python/torch):
    it must compile and link against include/tnrd.h + libtnrd.so."""
    import subprocess
    import tempfile
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "despeckle_c")
        r = subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(repo, "include"),
                            os.path.join(repo, "examples", "despeckle_c.c"),
                            "-L", os.path.join(repo, "paper_1702_07482_b200"), "-ltnrd",
                            "-lm", "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_parameter_space_kernels_keep_the_uniform_datapath():
    """The parameter-space-taps kernels (tile, cluster and split variants) must
    read their taps through the uniform datapath -- FFMA / FFMA2 with a
    uniform-register (UR) operand fed by LDCU.  ptxas silently falls back to
    per-thread LDC loads when it cannot prove the filter-group index uniform
    (seen on B200 builds: a cluster rank taken from %cluster_ctarank, an
    integer division in the group range, a per-thread copy loop in the group
    loop), which costs ~15% (C5).  Checked on the shipped library's SASS."""
    import re
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    LIB = _lib.LIB_PATH
    if not os.path.exists(cuobjdump) or not os.path.exists(LIB):
        pytest.skip("cuobjdump or libtnrd.so not available")
    sass = subprocess.run([cuobjdump, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    seen = 0
    for part in re.split(r"\n\s*Function : ", sass)[1:]:
        name = part.split("\n", 1)[0].strip()
        if not re.search(r"stage_kernel_(cl_pt|pt|split_pt)I", name):
            continue
        seen += 1
        fma = len(re.findall(r"\bFFMA2?\b", part))
        fma_ur = len(re.findall(r"\bFFMA2?\b[^;]*\bUR\d+", part))
        assert fma > 300 and fma_ur >= 0.35 * fma, (name[:80], fma, fma_ur)   # broken builds: < 2%
    assert seen >= 12, seen   # m = 3, 5, 7, 9 x tile / cluster / split


def test_kernel_selection_setters_validate_without_a_gpu():
    """tnrd_set_stage_kernel / tnrd_set_cluster_size are pure host state:
    out-of-range values are rejected with TNRD_EINVAL (ValueError)."""
    for bad in (-1, 13):
        with pytest.raises(ValueError):
            _lib.set_stage_kernel(bad)
    for bad in (1, 9, -2):
        with pytest.raises(ValueError):
            _lib.set_cluster_size(bad)
    for ok in (0, 2, 8, 0):
        _lib.set_cluster_size(ok)
    for ok in (_lib.KERNEL_CLUSTER_LARGE, _lib.KERNEL_TC_ADJOINT, _lib.KERNEL_AUTO):
        _lib.set_stage_kernel(ok)
