"""The C-ABI library loads and exports every symbol include/*.h declares.

No compute calls are made here (no GPU in the CI container); a session
request must fail loudly with TT_ERR_NO_DEVICE rather than fall back to CPU.
"""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200._abi import LIB_PATH, SIGNATURES, lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(tt_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_header_symbols_exported():
    names = declared_symbols()
    assert len(names) > 50
    handle = ctypes.CDLL(str(LIB_PATH))
    missing = [n for n in sorted(names) if not hasattr(handle, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert declared_symbols() == set(SIGNATURES), declared_symbols() ^ set(SIGNATURES)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_tma_path_in_sass():
    """The fused reduction kernel issues TMA bulk copies (SASS UBLKCP) and
    mbarrier waits (SYNCS) -- the Blackwell-native data path."""
    out = subprocess.run(["cuobjdump", "-sass", str(LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "UBLKCP" in out.stdout and "SYNCS" in out.stdout


def test_no_device_fails_loudly():
    if tt.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(tt.NoDeviceError):
        tt.Session(8, 2)


def test_error_mapping():
    with pytest.raises(tt.ShapeParseError):
        tt.parse_shape("[5/2")
    assert lib().tt_last_error().decode().startswith("expected")
    assert lib().tt_set_kernel_path(9) == 4  # TT_ERR_INVALID_ARGUMENT
    assert lib().tt_kernel_path() in (0, 1, 2, 3, 4)
