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
    assert rg.lib.regen_abi_version() == 2


def test_struct_layouts():
    import paper_2407_16990_b200 as rg
    assert ctypes.sizeof(rg.Geom) == 24
    assert ctypes.sizeof(rg.SelectParams) == 32
    assert ctypes.sizeof(rg.PackParams) == 36
    assert ctypes.sizeof(rg.SRConfig) == 24
    assert rg.BOX_DTYPE.itemsize == 80 and rg.REGION_DTYPE.itemsize == 32


def test_struct_layouts_match_the_c_header(tmp_path):
    """sizeof/offsetof of every ABI struct compiled from include/regen.h by the C compiler equal the
    ctypes mirrors of the binding."""
    import subprocess
    import paper_2407_16990_b200 as rg
    src = tmp_path / "layout.c"
    fields = {"regen_geom": (rg.Geom, "S F frame_w frame_h mb format"),
              "regen_select_params": (rg.SelectParams, "mode scope k tau connectivity cap"),
              "regen_pack_params": (rg.PackParams, "bin_w bin_h max_bins expand partition_mb gutter order policy density"),
              "regen_sr_config": (rg.SRConfig, "scale channels n_resblocks dtype res_scale bin_w")}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "regen.h"', "int main(void) {"]
    for name, (_, fl) in fields.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f in fl.split():
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append('printf("regen_box %zu\\nregen_region %zu\\n", sizeof(regen_box), sizeof(regen_region));')
    lines.append("return 0; }")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for name, (cls, fl) in fields.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f in fl.split():
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)
    assert int(got["regen_box"]) == rg.BOX_DTYPE.itemsize and int(got["regen_region"]) == rg.REGION_DTYPE.itemsize


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
