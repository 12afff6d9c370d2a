"""CPU-side checks of the boundary: the shared library loads and exports every symbol include/tcqr.h
declares; the binding declares exactly those; the product package never imports the oracle."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcqr.h")
PKG = os.path.join(ROOT, "paper_1912_05508_b200")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcqr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    d = _declared()
    for name in ("tcqr_factor", "tcqr_lls_solve", "tcqr_init", "tcqr_finalize"):
        assert name in d


def test_library_exports_every_declared_symbol():
    import paper_1912_05508_b200 as tq
    if not os.path.exists(tq.LIB_PATH):
        pytest.skip("libtcqr.so not built (run __graft_entry__.build())")
    lib = tq.lib()  # dlopen works without a GPU (CUDA runtime is linked statically)
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(tq.EXPORTS) == _declared()


def test_nm_dynamic_symbols():
    import subprocess
    import paper_1912_05508_b200 as tq
    if not os.path.exists(tq.LIB_PATH):
        pytest.skip("libtcqr.so not built")
    out = subprocess.run(["nm", "-D", "--defined-only", tq.LIB_PATH], capture_output=True,
                         text=True).stdout
    syms = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for name in _declared():
        assert name in syms, name


def test_library_has_tcgen05_and_tma_sass():
    import shutil
    import subprocess
    import paper_1912_05508_b200 as tq
    if not os.path.exists(tq.LIB_PATH) or not shutil.which("cuobjdump"):
        pytest.skip("no library / cuobjdump")
    sass = subprocess.run(["cuobjdump", "-sass", tq.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass      # tcgen05.mma kind::f16
    assert "UTMALDG" in sass      # TMA cp.async.bulk.tensor
    assert "LDTM" in sass         # tcgen05.ld
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names)
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle"


def test_calls_without_init_fail_loudly():
    import ctypes
    import paper_1912_05508_b200 as tq
    if not os.path.exists(tq.LIB_PATH):
        pytest.skip("libtcqr.so not built")
    rc = tq.lib().tcqr_factor(8, 4, ctypes.c_void_p(16), 8, ctypes.c_void_p(16), ctypes.c_void_p(16))
    assert rc == -1004   # TCQR_ERR_NOT_INIT, no silent CPU path


def test_default_config_matches_paper():
    import paper_1912_05508_b200 as tq
    if not os.path.exists(tq.LIB_PATH):
        pytest.skip("libtcqr.so not built")
    c = tq.default_config()
    assert c.cutoff == 128          # Alg. 2 line 3
    assert c.panel_rows == 1024     # B200 block rows (PAPER.md:441-442 used 256 on V100; R-A6)
    assert c.col_scaling == 1 and c.restart == 1 and abs(c.tol2 - 1e-8) < 1e-22
