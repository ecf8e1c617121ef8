"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/tilt.h declares, and its host-only entry points behave (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    import __graft_entry__ as g
    g.build()
    import paper_1205_5351_b200 as T
    return T


def test_header_symbols_exported(pkg):
    hdr = open(os.path.join(ROOT, "include", "tilt.h")).read()
    declared = set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(tilt_\w+)\s*\(", hdr, flags=re.M))
    assert declared == set(pkg.EXPORTS), declared ^ set(pkg.EXPORTS)
    for name in declared:
        assert hasattr(pkg.lib, name), name


def _header_fields(struct_name):
    hdr = open(os.path.join(ROOT, "include", "tilt.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    body = re.search(r"typedef struct \{([^}]*)\}\s*" + struct_name + ";", hdr).group(1)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if decl:  # "type name" or "type a, b": the identifiers that end each comma-separated piece
            names += [re.search(r"(\w+)\s*$", piece).group(1) for piece in decl.split(",")]
    return names


def test_struct_sizes_match_header(pkg):
    from paper_1205_5351_b200 import _abi
    assert [f[0] for f in _abi.TiltReport._fields_] == _header_fields("tilt_report")
    assert ctypes.sizeof(_abi.TiltReport) == 4 * len(_header_fields("tilt_report"))
    # (the Python field for the C member `lambda` is `lambda_`: a Python keyword)
    assert [f[0].rstrip("_") for f in _abi.TiltParams._fields_] == _header_fields("tilt_params")
    assert pkg.lib.tilt_abi_version() == 1


def test_default_params_and_strings(pkg):
    prm = pkg.default_params()
    assert prm.rho0 == 2.0 and prm.eps2 == pytest.approx(0.1) and prm.eps1 == pytest.approx(1e-6)
    assert prm.max_inner == 1000 and prm.max_outer == 50 and prm.vws == 1 and prm.svd_warm == 1
    assert prm.constraint_mode == pkg.CONSTRAINTS_CENTER_AREA and prm.lambda_ < 0
    assert pkg.lib.tilt_status_string(1).startswith(b"TILT_E_ARG")
    assert pkg.lib.tilt_patch_status_string(2) == b"WINDOW_ESCAPE"


def test_argument_validation_without_gpu(pkg):
    from paper_1205_5351_b200 import _abi
    # NULL handle / NULL options are rejected before any CUDA call
    assert pkg.lib.tilt_create(None, None) == _abi.TILT_E_ARG
    assert pkg.lib.tilt_destroy(None) == _abi.TILT_OK
    prm = pkg.default_params()
    assert pkg.lib.tilt_solve_batch(None, None, 0, 0, 0, None, None, None, 0, 0, ctypes.byref(prm),
                                    None, None, None, None, None) == _abi.TILT_E_ARG
    opts = _abi.TiltCreateOpts(device=0, stream=None, max_batch=1, max_m=1100, max_n=32, max_p=6)
    h = ctypes.c_void_p()
    assert pkg.lib.tilt_create(ctypes.byref(h), ctypes.byref(opts)) == _abi.TILT_E_ARG  # max_m > 1024
    opts = _abi.TiltCreateOpts(device=0, stream=None, max_batch=1, max_m=32, max_n=32, max_p=7)
    assert pkg.lib.tilt_create(ctypes.byref(h), ctypes.byref(opts)) == _abi.TILT_E_ARG  # p not 6 or 8


def test_no_cpu_fallback_in_product(pkg):
    """The product package must not import the oracle or any CPU implementation of the method."""
    pdir = os.path.join(ROOT, "paper_1205_5351_b200")
    for f in os.listdir(pdir):
        if f.endswith(".py"):
            src = open(os.path.join(pdir, f)).read()
            assert "oracle" not in src.replace("# ", ""), f
            assert "np.linalg.svd" not in src, f


def test_missing_library_fails_loudly():
    """No CPU fallback: importing the package without its CUDA library raises instead of degrading."""
    import subprocess
    import sys
    env = dict(os.environ, TILT_LIB="/nonexistent/libtilt.so")
    r = subprocess.run([sys.executable, "-c", "import paper_1205_5351_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "libtilt" in (r.stderr + r.stdout)
