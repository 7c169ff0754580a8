"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/ubs_b200.h declares, and the ctypes mirrors of the header
structs have exactly the C compiler's sizes and field offsets."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2510_03312_b200 import _lib, build

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ubs_b200.h"
STRUCTS = ["UbsCamera", "UbsSettings", "UbsView", "UbsPrimBuffers", "UbsBinBuffers", "UbsImageBuffers",
           "UbsGradBuffers"]


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ubs_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    build.build()
    lib = _lib.load(build_if_needed=False)
    hdr = int(re.search(r"#define UBS_ABI_VERSION (\d+)", HEADER.read_text()).group(1))
    assert lib.ubs_abi_version() == _lib.ABI_VERSION == hdr
    assert b"sm_100a" in lib.ubs_build_info()


def test_every_header_symbol_is_exported_and_bound():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 12
    bound = {n for n, _, _ in _lib.SIGNATURES}
    for n in names:
        assert hasattr(lib, n), f"{n} not exported by libubs_b200.so"
        assert n in bound, f"{n} has no ctypes signature in _lib.SIGNATURES"
    nm = subprocess.run(["nm", "-D", "--defined-only", str(build.OUT)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ubs_[a-z0-9_]+)", nm))
    assert set(names) <= exported


def test_sm100a_cubin_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(build.OUT)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.fixture(scope="module")
def c_layout(tmp_path_factory):
    src = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){"]
    for s in STRUCTS:
        cls = getattr(_lib, s)
        src.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in cls._fields_:
            src.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    src.append("return 0;}")
    d = tmp_path_factory.mktemp("abi")
    (d / "abi.c").write_text("\n".join(src))
    subprocess.run(["gcc", "-o", str(d / "abi"), str(d / "abi.c")], check=True)
    out = subprocess.run([str(d / "abi")], capture_output=True, text=True, check=True).stdout
    return dict(line.rsplit(" ", 1) for line in out.strip().splitlines())


@pytest.mark.parametrize("name", STRUCTS)
def test_struct_layout_matches_header(name, c_layout):
    cls = getattr(_lib, name)
    assert int(c_layout[name]) == ctypes.sizeof(cls)
    for f, _ in cls._fields_:
        assert int(c_layout[f"{name}.{f}"]) == getattr(cls, f).offset, f"{name}.{f}"


def test_cpu_only_host_raises_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_03312_b200 import engine, raster
    with pytest.raises(_lib.UbsError):
        engine.Workspace("cuda")
    from paper_2510_03312_b200 import synthetic as S
    with pytest.raises(Exception):
        raster.render(S.random_scene(3, 4, seed=0), S.random_camera(16, 0), S.random_query(3, 0))


def test_debug_row_offsets_match_header():
    # FrameCache.slices / .proj read the dump through _lib.DEBUG: every offset
    # must be the header's UBS_DEBUG_* value
    text = HEADER.read_text()
    macros = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"#define UBS_DEBUG_([A-Z0-9_]+) (\d+)", text)}
    assert macros.pop("stride") == _lib.DEBUG_STRIDE
    names = {"vmat": "vmat", "cov2_eig": "cov2_eig", "cov3_eig": "cov3_eig", "beta_q": "beta_q", "delta": "delta",
             "m_inv": "m_inv", "u": "u", "v": "v", "sigma_xq": "sigma_xq", "d_raw": "d_raw", "d_gate": "d_gate",
             "lx": "l_x", "rot": "rot", "sx": "s_x", "sq": "s_q", "color": "color", "flags": "flags"}
    assert {names[k]: v for k, v in macros.items()} == _lib.DEBUG
