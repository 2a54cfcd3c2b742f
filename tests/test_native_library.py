"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every entry point declared in include/comet_b200.h.  No compute calls."""

import ctypes
import os
import re

import pytest

from paper_2502_19811_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "comet_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(comet_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return ctypes.CDLL(_lib.LIB_PATH)


def test_header_declares_the_binding_surface():
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_loads(lib):
    l2 = _lib.load()
    assert l2.comet_version() == 1
    assert l2.comet_last_error() == b""


def test_kernels_are_sm100a_tcgen05():
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA.2CTA", "UTMALDG.2D.2CTA", "LDTM", "UBLKCP"):
        assert mnemonic in sass, mnemonic
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_no_device_raises_loudly(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeUnavailable):
        _lib.require_device()


def test_option_table_matches_the_header():
    """_lib.OPTIONS (the names LayerKnobs / set_option use) is exactly the
    header's COMET_OPT_* table, and LayerKnobs has a field per option."""
    from paper_2502_19811_b200 import LayerKnobs
    with open(os.path.join(ROOT, "include", "comet_b200.h")) as fh:
        text = fh.read()
    defs = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"#define COMET_OPT_([A-Z0-9_]+) (-?\d+)", text)}
    count = defs.pop("count")
    defs.pop("default", None)
    assert defs == _lib.OPTIONS
    assert sorted(defs.values()) == list(range(count))
    fields = set(LayerKnobs.__dataclass_fields__)
    assert set(_lib.OPTIONS) <= fields, set(_lib.OPTIONS) - fields
    assert set(LayerKnobs().options()) == set(_lib.OPTIONS)
