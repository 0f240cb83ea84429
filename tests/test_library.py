"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
exactly what include/hx_api.h declares (no compute calls here)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2311_11514_b200 import build, ops

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "hx_api.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hx_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return ops.load()


def test_header_and_bindings_agree():
    assert header_functions() == sorted(ops.EXPORTED)


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(ops.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (hx_[a-z0-9_]+)", out))
    assert set(header_functions()) <= exported


def test_host_only_entry_points(lib):
    assert lib.hx_version() == 1
    assert lib.hx_error_string(1001) == b"hx: bad argument"
    # workspace sizing is pure host arithmetic: split-K for decode shapes, none for prefill
    assert ops.linear_workspace(__import__("torch").bfloat16, 8, 12288, 4096) > 0
    assert ops.linear_workspace(__import__("torch").bfloat16, 4096, 12288, 4096) == 0
    assert ops.kv_bytes(__import__("torch").bfloat16, 2, 10, 4, 64, 128) == 2 * 2 * 2 * 10 * 4 * 64 * 128


def test_sass_is_blackwell_native(lib):
    """tcgen05 MMA, TMA loads and TMEM loads are present in the shipped binary."""
    sass = subprocess.run(["cuobjdump", "-sass", str(ops.LIB_PATH)], capture_output=True, text=True,
                          check=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "HGMMA" not in sass


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(ops.HxError):
        ops.load(tmp_path / "nope.so")
