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
        assert v["r"] >= 1 and v["s"] >= 1 and v["kt"] in (1, 2, 3, 4, 8)
        assert v["nbt"] in (1, 2, 4) and v["mode"] in (0, 1, 2)
        assert v["mode"] < 2 or (v["kind"] == 7 and v["io"] == 2)  # half2: f16 lane kernels only
        if v["kind"] == 6:  # TMEM image-lane: dispatch = warps per lane quarter
            assert v["dispatch"] in (2, 3, 4) and v["tw"] in (2, 4, 8, 16)
        elif v["kind"] == 7:  # image-lane position classes: dispatch = tap unroll, nbt = images per lane
            assert v["dispatch"] in (1, 2, 3, 4) and v["th"] == v["tw"] and v["th"] in (2, 4, 8) and v["kt"] in (1, 2, 3, 4)
            assert (v["dispatch"] == 3) == (v["th"] == 8)  # 8x8 planes run as quadrant tiles
            assert v["dispatch"] != 4 or (v["th"] == 4 and v["kt"] == 1)  # 4x4 tiles of 8x8+ planes
        else:
            assert v["dispatch"] in (0, 1, 2, 3)
            assert v["dispatch"] < 2 or v["kind"] == 2  # column-tiled (wide) / 1D direct
        assert v["kind"] in (0, 1, 2, 3, 4, 5, 6, 7) and v["io"] in (0, 2)
        kinds.add(v["kind"])
    # tiled, plane, direct, image-lane, ws, TMEM strips, TMEM image-lane, image-lane position classes
    assert kinds == {0, 1, 2, 3, 4, 5, 6, 7}


def test_sm100a_cubin_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def _fused_ffma(line: str) -> bool:
    """An FFMA/FFMA2 whose multiplicands are both live registers.  `FFMA Rd, RZ, x, y`
    (0*x + y) appears in the f64 division sequence of the fake-quant epilogue; it
    multiplies by the zero register, so it can never be a contracted MAC.  (DFMA is
    not checked: the same __ddiv_rn Newton steps use it, and the f32 kernels' MACs can
    only contract to FFMA/FFMA2; the f64 generic kernel's DMUL+DADD is asserted below.)"""
    m = re.search(r"(?:^|[\s/])(?:@!?U?P\w+\s+)?(FFMA2?)(?:\.\S+)?\s+[^,]+,\s*([^,]+),\s*([^,]+),", line)
    if not m:
        return False
    a, b = m.group(2).strip(), m.group(3).strip()
    return not (a.startswith(("RZ", "-RZ")) or b.startswith(("RZ", "-RZ")))


# exact-mode (MODE = 0) kernels of every kind, by mangled template signature
_EXACT = {
    "tiled": r"_ZN3scb7k_tiledILi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELi\d+ELb0ELi(\d)ELi0ELi\dELi\dEE",
    "generic": r"_ZN3scb9k_genericI([fd])Li0EE",
    "direct": r"_ZN3scb8k_directI(?:Li\d+E){6}Li0E(?:Li\d+E){2}Lb0E(?:Lb[01]E){2}Li0EE",
    "dws": r"_ZN3scb5k_dwsI(?:Li\d+E){6}Li0EE",
    "dtm": r"_ZN3scb5k_dtmI(?:Li\d+E){7}Li0EE",
    "dimg": r"_ZN3scb6k_dimgILi\d+ELi\d+ELi0ELb0ELi0EE",
    "plane": r"_ZN3scb7k_planeI(?:Li\d+E){7}Lb0ELi0ELi0ELi\dEE",
    "tmi": r"_ZN3scb5k_tmiI(?:Li\d+E){5}Li0EE",
    "lane": r"_ZN3scb6k_laneI(?:Li\d+E){4}Li0ELi\d+ELb0E(?:Li\d+E){3}E",
}


def test_exact_kernels_never_fuse():
    """Exact-mode kernels must not contract the MAC into FFMA/FFMA2/DFMA: the
    reference rounds the product and the sum separately (sc/_kernels.py:73-84).
    Every exact variant of every kind is inspected (round 1's patterns missed the
    direct and image-lane kernels)."""
    sass = subprocess.run(["cuobjdump", "-sass", str(_abi.LIB_PATH)],
                          capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    checked = {k: 0 for k in _EXACT}
    for body in funcs[1:]:
        name = body.split("\n", 1)[0].strip()
        kind = next((k for k, pat in _EXACT.items() if re.match(pat, name)), None)
        if kind is None:
            continue
        bad = [ln.strip() for ln in body.splitlines() if _fused_ffma(ln)]
        assert not bad, (name, bad[:3])
        assert re.search(r"\b(FMUL|DMUL)\b", body), name
        if kind == "generic" and "IdLi0E" in name:
            assert re.search(r"\bDMUL\b", body) and re.search(r"\bDADD\b", body), name
        checked[kind] += 1
    assert checked["direct"] >= 100 and checked["dimg"] >= 5 and checked["tmi"] >= 10, checked
    assert checked["lane"] >= 10, checked
    assert all(v > 0 for v in checked.values()), checked


def test_fused_ffma_detector():
    assert _fused_ffma("        /*0a10*/                   FFMA R4, R5, R6, R7 ;")
    assert _fused_ffma("@P0 FFMA2 R4, R6.F32x2.HI_LO, R8.F32x2.HI_LO, R10 ;")
    assert not _fused_ffma("        /*0a10*/                   FFMA R0, RZ, UR9, R15 ;")
    assert not _fused_ffma("FMUL R4, R5, R6 ;")