"""The C-ABI library loads and exports every symbol include/pbnsim.h declares
(no GPU needed; no compute calls that need a device)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pbnsim.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\**\s+\**\s*(pbn_[a-z0-9_]+)\s*\(",
                                 src, flags=re.M)))


@pytest.fixture(scope="module")
def built_lib():
    from paper_1508_07828_b200 import _build
    return _build.build()


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for required in ["pbn_load", "pbn_free", "pbn_simulate", "pbn_gelman_rubin", "pbn_two_state",
                     "pbn_run", "pbn_recount", "pbn_validate", "pbn_skart_ci_from_batches"]:
        assert required in names


def test_library_exports_every_declared_symbol(built_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", built_lib], capture_output=True, text=True,
                         check=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_binding_covers_every_declared_symbol(built_lib):
    from paper_1508_07828_b200 import _lib
    L = _lib.lib()
    assert set(_lib.SIGNATURES) == set(declared_functions())
    for n in declared_functions():
        assert getattr(L, n) is not None
    assert _lib.lib().pbn_version().startswith(b"libpbnsim")


def test_library_is_sm100a(built_lib):
    out = subprocess.run(["cuobjdump", "--list-elf", built_lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
