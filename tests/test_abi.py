"""The C-ABI library loads on a CPU-only host and exports every symbol the
public header declares (no compute calls)."""
import re
import subprocess
from pathlib import Path

from paper_2011_06295_b200 import _abi

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sparseconv_b200.h"


def declared():
    return sorted(set(re.findall(r"SCB_API\s+[\w\s\*]+?\b(scb_\w+)\s*\(", HEADER.read_text())))


def test_header_lists_match_binding():
    assert declared() == sorted(_abi.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    for name in declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (scb_\w+)", out))
    assert set(declared()) <= exported
    assert all(s.startswith("scb_") for s in exported)


def test_variant_table():
    vs = _abi.variants()
    assert len(vs) >= 10
    kinds = set()
    for v in vs:
        assert v["r"] >= 1 and v["s"] >= 1 and v["kt"] in (1, 2, 4, 8)
        assert v["nbt"] in (1, 2, 4) and v["mode"] in (0, 1) and v["dispatch"] in (0, 1, 2, 3)
        assert v["dispatch"] < 2 or v["kind"] == 2  # column-tiled (wide) / 1D direct
        assert v["kind"] in (0, 1, 2, 3, 4, 5) and v["io"] in (0, 2)
        kinds.add(v["kind"])
    assert kinds == {0, 1, 2, 3, 4, 5}  # tiled, plane, direct, image-lane, warp-specialised, TMEM


def test_sm100a_cubin_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_exact_kernels_never_fuse():
    """Exact-mode kernels must not contain FFMA/FFMA2: the reference rounds the
    product and the sum separately (sc/_kernels.py:73-84)."""
    sass = subprocess.run(["cuobjdump", "-sass", str(_abi.LIB_PATH)],
                          capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    checked = 0
    for body in funcs[1:]:
        name = body.split("\n", 1)[0].strip()
        m = re.match(r"_ZN3scb7k_tiledILi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELb0ELi(\d)ELi0ELi\dELi\dEE", name)
        g = re.match(r"_ZN3scb9k_genericI([fd])Li0EE", name)
        d = re.match(r"_ZN3scb8k_directILi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi0ELi\d+ELi\d+ELb0EE", name) or \
            re.match(r"_ZN3scb5k_dwsILi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi0EE", name) or \
            re.match(r"_ZN3scb5k_dtmILi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi0EE", name)
        i = re.match(r"_ZN3scb6k_dimgILi\d+ELi\d+ELi0EE", name)
        pl = re.match(r"_ZN3scb7k_planeILi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELb0ELi0ELi0ELi\dEE", name)
        if not (m or g or d or i or pl):
            continue
        ops = re.findall(r"\b(FFMA2?|DFMA|FMUL2?|FADD2?|DMUL|DADD)\b", body)
        assert "FFMA" not in ops and "FFMA2" not in ops and "DFMA" not in ops, name
        assert any(o.startswith(("FMUL", "DMUL")) for o in ops), name
        checked += 1
    assert checked >= 40
