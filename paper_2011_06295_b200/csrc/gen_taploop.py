#!/usr/bin/env python3
"""Generate the tap-loop inline-PTX blocks and the variant table.

Why generated PTX: the inner loop of the tiled kernel applies one weight to
a register tile at a compile-time (kk, r, s) offset chosen by the tap's meta
word.  NVVM lowers a C++ switch over ~72 cases into a compare tree (~7
compare+branch per tap, measured with ncu: profiles/r01_conv3_2_v1.txt).
PTX ``brx.idx`` gives a real jump table (SASS LDC + BRX), so dispatch costs
a constant handful of instructions per tap.  Scalar ``mul.rn``/``add.rn`` in
PTX are never contracted by ptxas, which keeps exact mode bit-identical to
the reference's separately rounded multiply and add (sc/_kernels.py:73-84).

Outputs (written next to this file by the Makefile, not committed):
  inst_gen_<i>.cu  -- TapLoop<...>::run specialisations + k_tiled instantiations
  registry_gen.cu  -- num_variants() / variant(i) over all parts
"""
from __future__ import annotations

import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

# staging modes (must match kernels.cuh)
CPASYNC, PLANE = 0, 1
# weight payload formats (kernels.cuh WF_*)
WF_F32, WF_F16, WF_CB4, WF_LIN16 = 0, 1, 2, 3
EXACT, FMA = 0, 1

# (R, S, KT, NBT, TH, TW, staging modes)
TILES = [
    (3, 3, 8, 1, 4, 4, (PLANE, CPASYNC)),
    (3, 3, 4, 1, 4, 4, (PLANE,)),
    (3, 3, 8, 1, 2, 4, (PLANE,)),
    (3, 3, 4, 2, 2, 4, (PLANE,)),
    (3, 3, 8, 2, 2, 4, (PLANE,)),
    (3, 3, 4, 2, 4, 4, (PLANE,)),
    (3, 3, 8, 1, 2, 2, (PLANE,)),
    (3, 3, 8, 2, 2, 2, (PLANE,)),
    (3, 3, 8, 4, 2, 2, (PLANE,)),
    (3, 3, 4, 4, 2, 2, (PLANE,)),
    (1, 1, 8, 1, 4, 4, (PLANE, CPASYNC)),
    (1, 1, 8, 2, 2, 4, (PLANE,)),
    (5, 5, 4, 1, 4, 4, (PLANE, CPASYNC)),
    (5, 5, 4, 1, 2, 4, (PLANE,)),
    (1, 2, 8, 1, 1, 8, (CPASYNC,)),
    (1, 3, 8, 1, 1, 8, (PLANE, CPASYNC)),
]
# (io f16?, weight format, mode) combinations compiled for every tile
BASE_MODES = [(False, WF_F32, EXACT), (False, WF_F32, FMA), (True, WF_F16, FMA)]
# quantised formats only for the main 3x3 tiles
QUANT_TILES = {(3, 3, 8, 1, 4, 4), (3, 3, 4, 2, 2, 4), (3, 3, 8, 2, 2, 2), (3, 3, 8, 1, 2, 4)}
QUANT_MODES = [(False, WF_CB4, EXACT), (True, WF_CB4, FMA), (False, WF_LIN16, EXACT),
               (True, WF_LIN16, FMA)]


def decode_ptx(wf: int) -> str:
    if wf == WF_F32:
        return "mov.b32 %%v, %%pc;\n"
    if wf == WF_F16:
        return "cvt.u16.u32 %%h, %%pc;\n cvt.f32.f16 %%v, %%h;\n"
    if wf == WF_CB4:
        return "shl.b32 %%o, %%pc, 2;\n add.u32 %%o, %%o, %%aux;\n ld.shared.f32 %%v, [%%o];\n"
    return "cvt.u16.u32 %%h, %%pc;\n cvt.rn.f32.s16 %%v, %%h;\n mul.rn.f32 %%v, %%v, %%scl;\n"


def gen_taploop(R, S, KT, NBT, TH, TW, WF, MODE) -> str:
    PH, PW = TH + R - 1, TW + S - 1
    P = NBT * TH * TW
    nacc = KT * P
    npt = NBT * PH * PW
    # operand numbering: acc 0..nacc-1 ("+f"), pt nacc.., then tap begin/end, aux, scale
    def acc_op(kk, j, y, x):
        return f"%{kk * P + (j * TH + y) * TW + x}"

    def pt_op(j, y, x):
        return f"%{nacc + (j * PH + y) * PW + x}"

    o_beg, o_end, o_aux, o_scl = nacc + npt, nacc + npt + 1, nacc + npt + 2, nacc + npt + 3
    lines = []
    lines.append("{\n")
    lines.append(".reg .pred %%p;\n.reg .u32 %%m, %%mc, %%pb, %%pc, %%o, %%aux;\n"
                 ".reg .u64 %%q, %%end;\n.reg .f32 %%v, %%t, %%scl;\n.reg .b16 %%h;\n")
    lines.append(f"mov.u64 %%q, %{o_beg};\nmov.u64 %%end, %{o_end};\n"
                 f"mov.u32 %%aux, %{o_aux};\nmov.f32 %%scl, %{o_scl};\n")
    lines.append("setp.ge.u64 %%p, %%q, %%end;\n@%%p bra.uni DONE;\n")
    lines.append("ld.global.nc.v2.u32 {%%m, %%pb}, [%%q];\n")
    lines.append("bra.uni LOOP;\n")
    labels = []
    for kk in range(KT):
        for r in range(R):
            for s in range(S):
                lab = f"C{(kk * R + r) * S + s}"
                labels.append(lab)
                body = [f"{lab}:\n"]
                for j in range(NBT):
                    for y in range(TH):
                        for x in range(TW):
                            a, p = acc_op(kk, j, y, x), pt_op(j, y + r, x + s)
                            if MODE == EXACT:
                                body.append(f"mul.rn.f32 %%t, %%v, {p};\nadd.rn.f32 {a}, {a}, %%t;\n")
                            else:
                                body.append(f"fma.rn.f32 {a}, %%v, {p}, {a};\n")
                body.append("bra.uni NEXT;\n")
                lines.append("".join(body))
    lines.append("TBL: .branchtargets " + ", ".join(labels) + ";\n")
    lines.append("LOOP:\n")
    lines.append("mov.u32 %%mc, %%m;\nmov.u32 %%pc, %%pb;\n")
    lines.append("ld.global.nc.v2.u32 {%%m, %%pb}, [%%q+8];\n")  # prefetch (array has a slack slot)
    lines.append("add.u64 %%q, %%q, 8;\n")
    lines.append(decode_ptx(WF))
    lines.append("brx.idx.uni %%mc, TBL;\n")
    lines.append("NEXT:\nsetp.lt.u64 %%p, %%q, %%end;\n@%%p bra.uni LOOP;\n")
    lines.append("DONE:\n}\n")
    asm = "".join(lines)
    # C++ wrapper
    out = []
    out.append(f"template <> struct TapLoop<{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {WF}, {MODE}> {{\n")
    out.append(f"  static __device__ __forceinline__ void run(float (&a)[{nacc}], const float (&pt)[{npt}],\n"
               "      const Tap* beg, const Tap* end, unsigned aux, float scl) {\n")
    out.append("    asm volatile(\n")
    for ln in asm.splitlines():
        out.append('      "' + ln.replace('"', '\\"') + '\\n"\n')
    ops_out = ", ".join(f'"+f"(a[{i}])' for i in range(nacc))
    ops_in = ", ".join(f'"f"(pt[{i}])' for i in range(npt))
    out.append(f"      : {ops_out}\n")
    out.append(f'      : {ops_in}, "l"(beg), "l"(end), "r"(aux), "f"(scl)\n')
    out.append("      : \"memory\");\n  }\n};\n\n")
    return "".join(out)


N_PARTS = 8


def main():
    # group kernel variants by tile so each TapLoop lives in exactly one TU
    tiles = []
    for R, S, KT, NBT, TH, TW, stages in TILES:
        modes = list(BASE_MODES)
        if (R, S, KT, NBT, TH, TW) in QUANT_TILES:
            modes += QUANT_MODES
        loops, variants = [], []
        for f16, wf, mode in modes:
            key = (R, S, KT, NBT, TH, TW, wf, mode)
            if key not in loops:
                loops.append(key)
            for st in stages:
                variants.append((R, S, KT, NBT, TH, TW, f16, wf, mode, st))
        tiles.append((loops, variants))
    # balance tiles over N_PARTS translation units by variant count
    parts = [[] for _ in range(N_PARTS)]
    load = [0] * N_PARTS
    for t in sorted(tiles, key=lambda t: -len(t[1])):
        i = load.index(min(load))
        parts[i].append(t)
        load[i] += len(t[1]) * len(t[0])
    total_v = 0
    for i, part in enumerate(parts):
        src = ["// GENERATED by gen_taploop.py -- do not edit.\n#include \"tiled.cuh\"\n"
               "#include \"variants.h\"\n\nnamespace scb {\n\n"]
        ents = []
        for loops, variants in part:
            for key in loops:
                src.append(gen_taploop(*key))
            for v in variants:
                R, S, KT, NBT, TH, TW, f16, wf, mode, st = v
                ents.append(f"    {{{{{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {'SCB_F16' if f16 else 'SCB_F32'}, "
                            f"{wf}, {mode}, {st}}}, "
                            f"&launch_tiled_t<{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {'true' if f16 else 'false'}, "
                            f"{wf}, {mode}, {st}>}},\n")
        total_v += len(ents)
        src.append(f"extern const VariantEntry g_part_{i}[];\n")
        if ents:
            src.append(f"const VariantEntry g_part_{i}[] = {{\n" + "".join(ents) + "};\n")
            src.append(f"extern const int g_part_{i}_n;\nconst int g_part_{i}_n = {len(ents)};\n")
        else:
            src.append(f"const VariantEntry g_part_{i}[] = {{}};\nextern const int g_part_{i}_n;\n"
                       f"const int g_part_{i}_n = 0;\n")
        src.append("\n}  // namespace scb\n")
        (HERE / f"inst_gen_{i}.cu").write_text("".join(src))
    reg = ["// GENERATED by gen_taploop.py -- do not edit.\n#include \"variants.h\"\n\nnamespace scb {\n"]
    for i in range(N_PARTS):
        reg.append(f"extern const VariantEntry g_part_{i}[];\nextern const int g_part_{i}_n;\n")
    reg.append("\nstatic const VariantEntry* const kParts[] = {" + ", ".join(f"g_part_{i}" for i in range(N_PARTS)) + "};\n")
    reg.append("static const int* const kPartN[] = {" + ", ".join(f"&g_part_{i}_n" for i in range(N_PARTS)) + "};\n")
    reg.append(f"static const int kNumParts = {N_PARTS};\n")
    reg.append("""
int num_variants() {
    int n = 0;
    for (int i = 0; i < kNumParts; ++i) n += *kPartN[i];
    return n;
}

const VariantEntry& variant(int idx) {
    for (int i = 0; i < kNumParts; ++i) {
        if (idx < *kPartN[i]) return kParts[i][idx];
        idx -= *kPartN[i];
    }
    return kParts[0][0];
}

}  // namespace scb
""")
    (HERE / "registry_gen.cu").write_text("".join(reg))
    print(f"generated {total_v} kernel variants in {N_PARTS} units", file=sys.stderr)


if __name__ == "__main__":
    main()
