"""The C-ABI library loads and exports every symbol include/swr.h declares
(no compute calls: runs without a GPU), and the binding has no CPU path."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "swr.h")).read()
    return sorted(set(re.findall(r"\b(swr_[A-Za-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("swr_setup", "swr_build_interface_operator", "swr_solve", "swr_free"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1503_02564_b200 import _build
    so = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_binding_loads_and_maps_errors():
    import paper_1503_02564_b200 as pkg
    L = pkg.lib()
    assert L.swr_error_string(0) == b"ok"
    assert b"zero pivot" in L.swr_error_string(3)
    assert set(pkg.swr.EXPORTED) <= set(_declared())


def test_setup_rejects_bad_config_without_gpu_work():
    """Argument validation happens before any device call."""
    import ctypes as C

    import numpy as np
    import paper_1503_02564_b200 as pkg
    import swr_inputs as si
    L = pkg.lib()
    p = si.config("C1", N=3)            # 3 does not divide N_x = 200
    u0 = si.make_u0(si.config("C1"))
    c = pkg.swr.Config()
    c.a0, c.b0, c.T, c.dx, c.dt, c.N = p.a0, p.b0, p.T, p.dx, p.dt, p.N
    c.u0 = u0.ctypes.data
    c.world = 1
    c.transmission = si.TC_ROBIN
    c.robin_p = 5.0
    h = C.c_void_p()
    assert L.swr_setup(C.byref(c), C.byref(h)) == 1
    c.N = 2
    c.robin_p = -1.0                    # Robin needs p > 0
    assert L.swr_setup(C.byref(c), C.byref(h)) == 1
    c.robin_p = 5.0
    c.algorithm = si.ALG_NEW
    c.potential = si.POT_CUBIC          # NEW needs V(x)
    assert L.swr_setup(C.byref(c), C.byref(h)) == 1
    c.potential = si.POT_VX
    c.transmission = si.TC_S22
    c.pade_m = 0                        # Pade needs m >= 1
    assert L.swr_setup(C.byref(c), C.byref(h)) == 1
    c.transmission = 8                  # no such operator
    assert L.swr_setup(C.byref(c), C.byref(h)) == 1
    c.transmission = si.TC_S02
    c.restart = 32                      # beyond the fused Gram-Schmidt kernels
    assert L.swr_setup(C.byref(c), C.byref(h)) == 1
    assert not h.value
    del np


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg_dir = os.path.join(ROOT, "paper_1503_02564_b200")
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "swr_oracle", "or_solve", "or_march"):
                    assert bad not in txt, (f, bad)
