"""CPU checks of the boundary: libmis.so loads and exports every entry point
include/mis.h declares; the binding declares the same names; sm_100a SASS is
present; no CUDA call is made (there is no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mis.h")
LIB = os.path.join(ROOT, "paper_1803_02009_b200", "libmis.so")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mis_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_built():
    from paper_1803_02009_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ["mis_create", "mis_set_model", "mis_set_graph", "mis_register", "mis_warp", "mis_fuse"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib_built):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_built], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mis_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_binding_loads_and_matches_header(lib_built):
    from paper_1803_02009_b200 import mis as M
    assert M.mis_abi_version() == 2
    assert sorted(M.EXPORTED) == declared()
    p = M.mis_default_params()
    assert (p.k, p.n_nbr, p.w_reg, p.w_corr, p.eps_d_mm, p.eps_n_deg) == (4, 4, 1e4, 10.0, 15.0, 10.0)
    assert (p.w_r, p.w_p) == (1e6, 1000.0)   # Eq. 10 priors, P:598 (struct layout matches the header)


def test_sm100a_sass_present(lib_built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_built], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_gpu_means_loud_failure(lib_built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1803_02009_b200 import mis as M
    with pytest.raises(M.MisError):
        M.Context(M.mis_default_params())
