"""The C-ABI library loads and exports every symbol include/regen.h declares (no GPU needed), and
the ctypes mirrors match the header's struct sizes. No compute calls here."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    h = open(os.path.join(ROOT, "include", "regen.h")).read()
    return sorted(set(re.findall(r"REGEN_API\s+[\w\s\*]+?\b(regen_\w+)\s*\(", h)))


def test_header_declares_the_four_calls():
    names = _declared()
    for n in ["regen_select_mbs", "regen_pack_regions", "regen_enhance_packed", "regen_scatter_blend"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2407_16990_b200 as rg
    lib = ctypes.CDLL(rg.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(rg.EXPORTED) == _declared()
    assert rg.lib.regen_abi_version() == 1


def test_struct_layouts():
    import paper_2407_16990_b200 as rg
    assert ctypes.sizeof(rg.Geom) == 20
    assert ctypes.sizeof(rg.SelectParams) == 24
    assert ctypes.sizeof(rg.PackParams) == 28
    assert ctypes.sizeof(rg.SRConfig) == 20
    assert rg.BOX_DTYPE.itemsize == 80 and rg.REGION_DTYPE.itemsize == 32


def test_pure_helpers_and_argument_errors_without_gpu():
    import paper_2407_16990_b200 as rg
    assert rg.capacity_mbs(512, 512, 4) == 4096
    g = rg.Geom(1, 1, 640, 360, 16)
    assert rg.workspace_size(rg.CALL_SELECT, g) > 0
    bad = rg.Geom(0, 1, 640, 360, 16)
    try:
        rg.workspace_size(rg.CALL_SELECT, bad)
        raise AssertionError("expected RegenError")
    except rg.RegenError as e:
        assert "S and F" in str(e)
