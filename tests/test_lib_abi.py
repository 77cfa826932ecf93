"""The drop-in boundary: libpp200.so loads without a GPU, exports every entry
point include/pp200.h declares, and the ctypes table binds exactly those."""
import pathlib
import re
import subprocess

import pytest

from paper_2412_14374_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pp200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    if not _lib.LIB_PATH.exists():
        from paper_2412_14374_b200 import build
        build.build()
    return _lib.LIB_PATH


def test_header_declares_the_abi():
    names = declared()
    for must in ("pc_gemm", "pc_accumulate", "pc_sgd_update", "pc_attention_fwd",
                 "pc_p2p_send", "pc_p2p_recv", "pc_p2p_abort", "pc_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", str(built)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pc_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_table_matches_header(built):
    assert sorted(_lib.exported_symbols()) == declared()
    L = _lib.lib()   # loads with no GPU present (CUDA runtime is lazily initialised)
    assert L.pc_version() == 1
    for name in declared():
        assert hasattr(L, name)


def test_argument_errors_are_reported_without_a_gpu(built):
    # Validation happens before any CUDA call: a bad epilogue is rejected with a message.
    with pytest.raises(_lib.PCError, match="bias"):
        _lib.call("pc_gemm", _lib.PC_F32, _lib.PC_F32, 0, 0, 4, 4, 4, 1, 4, 1, 4, 1, 4,
                  _lib.EPI_BIAS, None, None, 0, None, 0, None)


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "libpp200.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()
