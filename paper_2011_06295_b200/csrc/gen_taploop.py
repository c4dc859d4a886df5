#!/usr/bin/env python3
"""Generate the tap-loop inline-PTX blocks and the kernel-variant table.

The inner loop of the tiled kernel applies one weight to a register tile at
a compile-time (kk, r, s) offset.  Two dispatch strategies are generated and
the launch tuner picks per layer:

* DISPATCH_JUMP (0): one PTX ``brx.idx`` per tap through a jump table of the
  KT*R*S MAC blocks (SASS LDC + BRX).  NVVM would lower a C++ switch into a
  compare tree (~7 compare+branch per tap, ncu: profiles/r01_*); brx.idx
  costs a constant handful of instructions per tap.  The tap stream is
  prefetched two entries ahead.
* DISPATCH_MASK (1): per input channel the warp group reads KT 16-bit masks
  (bit r*S+s of half-word kk = tap present) and walks the MAC blocks in order
  with warp-uniform forward branches over absent kk / rows / taps.  No
  indirect branch and no dependent load before a branch, so it needs fewer
  resident warps to hide latency.

Scalar ``mul.rn``/``add.rn`` in PTX are never contracted by ptxas, which keeps
exact mode bit-identical to the reference's separately rounded multiply and
add (sc/_kernels.py:73-84); tests/test_abi.py checks the SASS.

Outputs (written next to this file by the Makefile, not committed):
  inst_gen_<i>.cu  -- TapLoop<...>::run specialisations + k_tiled instantiations
  registry_gen.cu  -- num_variants() / variant(i) over all parts
"""
from __future__ import annotations

import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

WF_F32, WF_F16, WF_CB4, WF_LIN16 = 0, 1, 2, 3   # kernels.cuh WF_*
EXACT, FMA = 0, 1                                # kernels.cuh MODE_*
JUMP, MASK = 0, 1                                # kernels.cuh DISPATCH_*

# (R, S, PAD, KT, NBT, TH, TW, dispatches, min CTAs/SM)
TILES = [
    (3, 3, 1, 8, 1, 4, 4, (JUMP, MASK), 1),
    (3, 3, 1, 4, 1, 4, 4, (JUMP, MASK), 2),
    (3, 3, 1, 8, 1, 2, 4, (JUMP, MASK), 2),
    (3, 3, 1, 4, 2, 2, 4, (JUMP, MASK), 2),
    (3, 3, 1, 4, 2, 4, 4, (JUMP, MASK), 1),
    (3, 3, 1, 8, 2, 2, 2, (JUMP, MASK), 2),
    (3, 3, 1, 8, 4, 2, 2, (JUMP, MASK), 1),
    (3, 3, 1, 4, 4, 2, 2, (JUMP, MASK), 2),
    (1, 1, 0, 8, 1, 4, 4, (JUMP, MASK), 1),
    (1, 1, 0, 8, 1, 2, 4, (JUMP,), 2),
    (5, 5, 2, 4, 1, 4, 4, (JUMP, MASK), 1),
    (5, 5, 0, 4, 1, 4, 4, (JUMP,), 1),
    (5, 5, 2, 4, 1, 2, 4, (JUMP,), 2),
    (1, 2, 0, 8, 1, 1, 8, (JUMP,), 2),
    (1, 3, 0, 8, 1, 1, 8, (JUMP,), 2),
    (1, 3, 1, 8, 1, 1, 8, (JUMP,), 2),
]
BASE_MODES = [(False, WF_F32, EXACT), (False, WF_F32, FMA), (True, WF_F16, FMA)]
QUANT_TILES = {(3, 3, 1, 8, 1, 4, 4), (3, 3, 1, 4, 2, 2, 4), (3, 3, 1, 8, 2, 2, 2), (3, 3, 1, 8, 1, 2, 4)}
QUANT_MODES = [(False, WF_CB4, EXACT), (True, WF_CB4, FMA), (False, WF_LIN16, EXACT),
               (True, WF_LIN16, FMA)]


def decode_ptx(wf: int, src: str = "%%pc") -> str:
    if wf == WF_F32:
        return f"mov.b32 %%v, {src};\n"
    if wf == WF_F16:
        return f"cvt.u16.u32 %%h, {src};\ncvt.f32.f16 %%v, %%h;\n"
    if wf == WF_CB4:
        return f"shl.b32 %%o, {src}, 2;\nadd.u32 %%o, %%o, %%aux;\nld.shared.f32 %%v, [%%o];\n"
    return f"cvt.u16.u32 %%h, {src};\ncvt.rn.f32.s16 %%v, %%h;\nmul.rn.f32 %%v, %%v, %%scl;\n"


class Ops:
    """Operand numbering of one generated asm statement: accumulators first,
    then `pt_base`-relative patch registers."""

    def __init__(self, R, S, KT, NBT, TH, TW, pt_base=None):
        self.PH, self.PW = TH + R - 1, TW + S - 1
        self.P = NBT * TH * TW
        self.nacc = KT * self.P
        self.npt = NBT * self.PH * self.PW
        self.TH, self.TW = TH, TW
        self.pt_base = self.nacc if pt_base is None else pt_base

    def acc(self, kk, j, y, x):
        return f"%{kk * self.P + (j * self.TH + y) * self.TW + x}"

    def pt(self, j, y, x):
        return f"%{self.pt_base + (j * self.PH + y) * self.PW + x}"


def mac_block(o: Ops, kk, r, s, NBT, TH, TW, MODE) -> str:
    body = []
    # distinct temporaries let ptxas interleave the independent multiplies
    for j in range(NBT):
        for y in range(TH):
            for x in range(TW):
                a, p = o.acc(kk, j, y, x), o.pt(j, y + r, x + s)
                if MODE == EXACT:
                    t = f"%%t{(j * TH + y) * TW + x}"
                    body.append(f"mul.rn.f32 {t}, %%v, {p};\nadd.rn.f32 {a}, {a}, {t};\n")
                else:
                    body.append(f"fma.rn.f32 {a}, %%v, {p}, {a};\n")
    return "".join(body)


def emit(template_args, signature, asm, outs, ins) -> str:
    lines = [f"template <> struct TapLoop<{template_args}> {{\n",
             f"  static __device__ __forceinline__ void run({signature}) {{\n",
             "    asm volatile(\n"]
    for ln in asm.splitlines():
        lines.append('      "' + ln.replace('"', '\\"') + '\\n"\n')
    lines.append(f"      : {', '.join(outs)}\n")
    lines.append(f"      : {', '.join(ins)}\n")
    lines.append('      : "memory");\n  }\n};\n\n')
    return "".join(lines)


def regs_decl(P, MODE, with_end=True):
    t = ", ".join(f"%%t{i}" for i in range(P)) if MODE == EXACT else "%%t0"
    q = ".reg .u64 %%q, %%end;\n" if with_end else ""
    return (".reg .pred %%p;\n.reg .u32 %%m, %%mc, %%pb, %%pc, %%m2, %%pb2, %%o, %%aux, %%w;\n"
            f"{q}.reg .f32 %%v, %%scl, {t};\n.reg .b16 %%h;\n")


def gen_jump(R, S, KT, NBT, TH, TW, WF, MODE) -> str:
    o = Ops(R, S, KT, NBT, TH, TW)
    ob = o.nacc + o.npt
    L = ["{\n", regs_decl(o.P, MODE),
         f"mov.u64 %%q, %{ob};\nmov.u64 %%end, %{ob + 1};\nmov.u32 %%aux, %{ob + 2};\nmov.f32 %%scl, %{ob + 3};\n",
         "setp.ge.u64 %%p, %%q, %%end;\n@%%p bra.uni DONE;\n",
         "ld.global.nc.v2.u32 {%%m, %%pb}, [%%q];\n",
         "ld.global.nc.v2.u32 {%%m2, %%pb2}, [%%q+8];\n",
         "bra.uni LOOP;\n"]
    labels = []
    for kk in range(KT):
        for r in range(R):
            for s in range(S):
                lab = f"C{(kk * R + r) * S + s}"
                labels.append(lab)
                L.append(f"{lab}:\n" + mac_block(o, kk, r, s, NBT, TH, TW, MODE) + "bra.uni NEXT;\n")
    L.append("TBL: .branchtargets " + ", ".join(labels) + ";\n")
    # two-deep prefetch of the tap stream (the device array has two slack slots)
    L.append("LOOP:\nmov.u32 %%mc, %%m;\nmov.u32 %%pc, %%pb;\nmov.u32 %%m, %%m2;\nmov.u32 %%pb, %%pb2;\n"
             "ld.global.nc.v2.u32 {%%m2, %%pb2}, [%%q+16];\nadd.u64 %%q, %%q, 8;\n")
    L.append(decode_ptx(WF))
    L.append("brx.idx.uni %%mc, TBL;\nNEXT:\nsetp.lt.u64 %%p, %%q, %%end;\n@%%p bra.uni LOOP;\nDONE:\n}\n")
    outs = [f'"+f"(a[{i}])' for i in range(o.nacc)]
    ins = [f'"f"(pt[{i}])' for i in range(o.npt)] + ['"l"(beg)', '"l"(end)', '"r"(aux)', '"f"(scl)']
    sig = (f"float (&a)[{o.nacc}], const float (&pt)[{o.npt}], const Tap* beg, const Tap* end, "
           "unsigned aux, float scl")
    return emit(f"{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {WF}, {MODE}, {JUMP}", sig, "".join(L), outs, ins)


def gen_mask(R, S, KT, NBT, TH, TW, WF, MODE) -> str:
    """Mask walk over one input channel.  In: mk (KT/2 u32 words; half-word kk
    holds bit r*S+s), vp = the channel's first Tap, pc = its payload
    (prefetched).  Out: vp / pc advanced past the channel's taps."""
    nacc = KT * NBT * TH * TW
    o = Ops(R, S, KT, NBT, TH, TW, pt_base=nacc + 2)
    nw = (KT + 1) // 2
    ovp, opc = o.nacc, o.nacc + 1
    oin = o.nacc + 2 + o.npt
    L = ["{\n", regs_decl(o.P, MODE, with_end=False),
         f"mov.u32 %%aux, %{oin + nw};\nmov.f32 %%scl, %{oin + nw + 1};\n"]
    for kk in range(KT):
        w = f"%{oin + kk // 2}"
        sh = 16 * (kk % 2)
        L.append(f"and.b32 %%w, {w}, {hex(((1 << (R * S)) - 1) << sh)};\n"
                 f"setp.eq.u32 %%p, %%w, 0;\n@%%p bra.uni K{kk}E;\n")
        for r in range(R):
            rowmask = ((1 << S) - 1) << (sh + r * S)
            if R > 1 and S > 1:
                L.append(f"and.b32 %%o, %%w, {hex(rowmask)};\nsetp.eq.u32 %%p, %%o, 0;\n@%%p bra.uni K{kk}R{r};\n")
            for s in range(S):
                bit = 1 << (sh + r * S + s)
                L.append(f"and.b32 %%o, %%w, {hex(bit)};\nsetp.eq.u32 %%p, %%o, 0;\n@%%p bra.uni K{kk}B{r}_{s};\n")
                L.append(decode_ptx(WF, f"%{opc}"))
                L.append(f"ld.global.nc.u32 %{opc}, [%{ovp}+12];\nadd.u64 %{ovp}, %{ovp}, 8;\n")
                L.append(mac_block(o, kk, r, s, NBT, TH, TW, MODE))
                L.append(f"K{kk}B{r}_{s}:\n")
            if R > 1 and S > 1:
                L.append(f"K{kk}R{r}:\n")
        L.append(f"K{kk}E:\n")
    L.append("}\n")
    outs = [f'"+f"(a[{i}])' for i in range(o.nacc)] + ['"+l"(vp)', '"+r"(pc)']
    ins = [f'"f"(pt[{i}])' for i in range(o.npt)] + [f'"r"(mk[{i}])' for i in range(nw)] + ['"r"(aux)', '"f"(scl)']
    sig = (f"float (&a)[{o.nacc}], const float (&pt)[{o.npt}], const Tap*& vp, unsigned& pc, "
           f"const unsigned (&mk)[{nw}], unsigned aux, float scl")
    return emit(f"{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {WF}, {MODE}, {MASK}", sig, "".join(L), outs, ins)


N_PARTS = 10


def main():
    groups = {}   # tap-loop key set -> (loops, variants); each loop lives in one TU
    for R, S, PAD, KT, NBT, TH, TW, disps, minb in TILES:
        modes = list(BASE_MODES)
        if (R, S, PAD, KT, NBT, TH, TW) in QUANT_TILES:
            modes += QUANT_MODES
        loops, variants = [], []
        for f16, wf, mode in modes:
            for d in disps:
                key = (R, S, KT, NBT, TH, TW, wf, mode, d)
                if key not in loops:
                    loops.append(key)
                variants.append((R, S, PAD, KT, NBT, TH, TW, f16, wf, mode, d, minb))
        tile_key = (R, S, KT, NBT, TH, TW)
        g = groups.setdefault(tile_key, ([], []))
        for l in loops:
            if l not in g[0]:
                g[0].append(l)
        g[1].extend(variants)
    items = sorted(groups.values(), key=lambda t: -len(t[1]))
    parts = [[] for _ in range(N_PARTS)]
    load = [0] * N_PARTS
    for t in items:
        i = load.index(min(load))
        parts[i].append(t)
        load[i] += len(t[1])
    total_v = 0
    for i, part in enumerate(parts):
        src = ["// GENERATED by gen_taploop.py -- do not edit.\n#include \"tiled.cuh\"\n"
               "#include \"variants.h\"\n\nnamespace scb {\n\n"]
        ents = []
        for loops, variants in part:
            for key in loops:
                R, S, KT, NBT, TH, TW, wf, mode, d = key
                src.append((gen_jump if d == JUMP else gen_mask)(R, S, KT, NBT, TH, TW, wf, mode))
            for v in variants:
                R, S, PAD, KT, NBT, TH, TW, f16, wf, mode, d, minb = v
                io = "SCB_F16" if f16 else "SCB_F32"
                tf = "true" if f16 else "false"
                ents.append(f"    {{{{{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {io}, {wf}, {mode}, {d}, {PAD}}}, "
                            f"&launch_tiled_t<{R}, {S}, {PAD}, {KT}, {NBT}, {TH}, {TW}, {tf}, {wf}, {mode}, "
                            f"{d}, {minb}>}},\n")
        total_v += len(ents)
        src.append(f"extern const VariantEntry g_part_{i}[];\nextern const int g_part_{i}_n;\n")
        src.append(f"const VariantEntry g_part_{i}[] = {{\n" + "".join(ents) + "};\n")
        src.append(f"const int g_part_{i}_n = {len(ents)};\n\n}}  // namespace scb\n")
        (HERE / f"inst_gen_{i}.cu").write_text("".join(src))
    reg = ["// GENERATED by gen_taploop.py -- do not edit.\n#include \"variants.h\"\n\nnamespace scb {\n"]
    for i in range(N_PARTS):
        reg.append(f"extern const VariantEntry g_part_{i}[];\nextern const int g_part_{i}_n;\n")
    reg.append("\nstatic const VariantEntry* const kParts[] = {" +
               ", ".join(f"g_part_{i}" for i in range(N_PARTS)) + "};\n")
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
