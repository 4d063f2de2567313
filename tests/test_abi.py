"""The C-ABI library loads and exports every symbol include/nss.h declares
(no compute calls: this runs on the CPU-only box)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nss.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nss_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for required in ("nss_init", "nss_step", "nss_run", "nss_evidence", "nss_samples"):
        assert required in syms


def test_library_exports_every_declared_symbol():
    from paper_2601_23252_b200 import build, nss
    build.build()
    lib = ctypes.CDLL(nss.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(nss.EXPORTS) == declared_symbols()


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2601_23252_b200 import nss
    monkeypatch.setattr(nss, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(nss, "_lib", None)
    with pytest.raises(RuntimeError):
        nss.lib()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2601_23252_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", text, flags=re.M), f
                assert "nsso" not in text, f
