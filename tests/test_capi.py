"""The C ABI library loads and exports every entry point include/coserve_cuda.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2402_18789_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "coserve_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+\**(cs_[a-z0-9_]+)\s*\(",
                       src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("cs_engine_create", "cs_step", "cs_adam_step", "cs_read_lora_grads",
                 "cs_read_kvgrad", "cs_gemm_bf16", "cs_coserve_run", "cs_sched_latency"):
        assert must in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (cs_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        assert hasattr(lib, n)
    assert lib.cs_version() == 3


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_tcgen05_and_tma_in_sass():
    """The GEMM is Blackwell-native: UTC*MMA (tcgen05.mma), LDTM (tcgen05.ld), UTMALDG (TMA)."""
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", out)
    assert "LDTM" in out
    assert "UTMALDG" in out


def test_host_calls_without_gpu():
    from paper_2402_18789_b200 import engine as E
    assert E.sched_latency(2, 0.01, 4096, 1000, 0) == pytest.approx(12.0)
    assert E.sched_max_finetune_tokens(2, 0.01, 0, 1000, 50.0) == 3800
    assert E.sched_max_finetune_tokens(2, 0.01, 0, 10000, 50.0) == 0
    lib = E.lib()
    h = ctypes.c_void_p()
    cfg = E.ModelConfig()  # zeros -> invalid_argument before touching the GPU
    rc = lib.cs_engine_create(ctypes.byref(cfg), 0, 0, 1, None, ctypes.byref(h))
    assert rc == _lib.CS_ERR_INVALID_ARGUMENT
    assert b"dimensions" in lib.cs_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(ImportError):
        _lib.lib()
