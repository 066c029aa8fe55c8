"""The C-ABI library loads and exports every symbol include/ustats_b200.h declares."""
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "ustats_b200.h").read_text()
    return sorted(set(re.findall(r"US_API\s+[\w\s\*]+?\b(us_\w+)\s*\(", text)))


def test_header_declares_api():
    names = declared()
    assert "us_u_statistic" in names and "us_einsum" in names and len(names) >= 18


def test_library_exports_every_declared_symbol(engine):
    from paper_2508_12627_b200 import _native
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (us_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    # only the C-ABI is visible (hidden C++ internals cannot interpose the oracle's)
    assert exported == set(declared())


def test_binding_covers_header(engine):
    from paper_2508_12627_b200 import _native
    assert sorted(_native.SIGNATURES) == declared()
    lib = _native.lib()
    for name in declared():
        assert getattr(lib, name) is not None


def test_version_and_error_channel(engine):
    from paper_2508_12627_b200 import _native
    assert b"sm_100a" in _native.lib().us_version()
    assert isinstance(_native.lib().us_last_error(), bytes)
