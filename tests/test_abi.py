"""The C-ABI library loads and exports every symbol include/nysipm.h declares (no GPU needed)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "nysipm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nys_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2404_14524_b200 as pkg
    return pkg.load_library()


def test_header_declares_the_boundary_calls():
    names = _declared()
    for core in ("nys_normal_matvec", "nys_sketch", "nys_pcg_solve", "nys_ipppmm_solve"):
        assert core in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_strerror_without_gpu(lib):
    assert lib.nys_strerror(0) == b"ok"
    assert b"Cholesky" in lib.nys_strerror(-3)


def test_default_options_match_oracle(lib):
    import ctypes as C
    from paper_2404_14524_b200._lib import Options
    from oracle.ippmm import Options as OO
    o = Options()
    lib.nys_default_options(C.byref(o))
    r = OO()
    assert (o.tol, o.rho0, o.delta0, o.reg_floor, o.pcg_c, o.pcg_floor, o.pcg_max_iter, o.init_delta,
            o.init_tol_rel, o.prec_refresh, o.prec_growth) == (r.tol, r.rho0, r.delta0, r.reg_floor, r.pcg_c,
                                                                r.pcg_floor, r.pcg_max_iter, r.init_delta,
                                                                r.init_tol_rel, r.prec_refresh, r.prec_growth)
    assert (o.ell_max, o.ell_tau, o.precond) == (r.ell_max, r.ell_tau, 0)


def test_product_package_does_not_import_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use the oracle: the package,
    the C header, the studies and the measurement tools never import it."""
    for sub in ("paper_2404_14524_b200", "include", "studies", "tools", "synth"):
        for dirpath, _, files in os.walk(os.path.join(ROOT, sub)):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h")):
                    txt = open(os.path.join(dirpath, f)).read()
                    assert "import oracle" not in txt and "from oracle" not in txt, os.path.join(sub, f)


def test_sass_has_dmma_and_bulk_copy(lib):
    """The sketch GEMM uses fp64 tensor cores (DMMA) and the matvec uses bulk async copies."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    so = os.path.join(ROOT, "paper_2404_14524_b200", "libnysipm.so")
    out = subprocess.run([cuobjdump, "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in out
    assert "UBLKCP" in out
    assert "sm_100a" in subprocess.run([cuobjdump, "-lelf", so], capture_output=True, text=True).stdout or "sm_100" in out
