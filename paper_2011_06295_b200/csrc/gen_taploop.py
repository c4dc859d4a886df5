#!/usr/bin/env python3
"""Generate the tap-loop inline-PTX blocks and the kernel-variant table.

The inner loop of the tiled kernel applies one weight to a register tile at
a compile-time (kk, r, s) offset.  Two dispatch strategies are generated and
the launch tuner picks per layer:

* DISPATCH_JUMP (0): one PTX ``brx.idx`` per tap through a jump table of the
  KT*R*S MAC blocks (SASS LDC + BRX).  NVVM would lower a C++ switch into a
  compare tree (~7 compare+branch per tap, ncu: profiles/r01_*); brx.idx
  costs a constant handful of instructions per tap.  Channel switches are
  sentinel entries of the stream that reload the register patch inside the
  same PTX loop; the stream segment of a stage is staged in shared memory.
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
# tiled tap loop dispatch: 1 = direct threaded (dispatch copied into every MAC
# block), 0 = one shared loop head (smaller code)
THREADED = int(__import__("os").environ.get("SCB_THREADED", "1"))

WF_F32, WF_F16, WF_CB4, WF_LIN16, WF_AFF16 = 0, 1, 2, 3, 4   # kernels.cuh WF_*
EXACT, FMA = 0, 1                                # kernels.cuh MODE_*
JUMP, MASK = 0, 1                                # kernels.cuh DISPATCH_*

# (R, S, PAD, KT, NBT, TH, TW, dispatches, min CTAs/SM)
TILES = [
    (3, 3, 1, 8, 1, 4, 4, (JUMP,), 1),
    (3, 3, 1, 4, 1, 4, 4, (JUMP,), 2),
    (3, 3, 1, 8, 1, 2, 4, (JUMP,), 2),
    (3, 3, 1, 4, 2, 2, 4, (JUMP,), 2),
    (3, 3, 1, 4, 2, 4, 4, (JUMP,), 1),
    (3, 3, 1, 8, 2, 2, 2, (JUMP,), 2),
    (3, 3, 1, 8, 4, 2, 2, (JUMP,), 1),
    (3, 3, 1, 4, 4, 2, 2, (JUMP,), 2),
    (3, 3, 1, 4, 1, 2, 2, (JUMP,), 2),
    (3, 3, 1, 4, 2, 2, 2, (JUMP,), 2),
    (3, 3, 1, 2, 2, 2, 2, (JUMP,), 2),
    (1, 1, 0, 8, 1, 4, 4, (JUMP,), 1),
    (1, 1, 0, 8, 1, 2, 4, (JUMP,), 2),
    (5, 5, 2, 4, 1, 4, 4, (JUMP,), 1),
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
        return f"and.b32 %%o, {src}, 15;\nshl.b32 %%o, %%o, 2;\nadd.u32 %%o, %%o, %%aux;\nld.shared.f32 %%v, [%%o];\n"
    return f"cvt.u16.u32 %%h, {src};\ncvt.rn.f32.s16 %%v, %%h;\nmul.rn.f32 %%v, %%v, %%scl;\n"


def dispatch_ptx(wf: int) -> str:
    """Threaded dispatch at the end of every MAC block: take the prefetched
    tap (%%m meta, %%pb payload), prefetch the following one, jump.  For f32
    payloads the value register doubles as the raw payload (a sentinel's
    channel number is read back from %%v in CS)."""
    if wf == WF_F32:
        return ("mov.b32 %%v, %%pb;\nmov.u32 %%mc, %%m;\n"
                "ld.shared.v2.u32 {%%m, %%pb}, [%%qs+8];\nadd.u32 %%qs, %%qs, 8;\n"
                "brx.idx.uni %%mc, TBL;\n")
    return ("mov.u32 %%pc, %%pb;\nmov.u32 %%mc, %%m;\n"
            "ld.shared.v2.u32 {%%m, %%pb}, [%%qs+8];\nadd.u32 %%qs, %%qs, 8;\n"
            + decode_ptx(wf) + "brx.idx.uni %%mc, TBL;\n")


def cs_head(wf: int) -> str:
    pc = "mov.b32 %%pc, %%v;\n" if wf == WF_F32 else ""
    return "CS:\n" + pc + "sub.u32 %%cl, %%pc, %%c0;\nsetp.ge.u32 %%p, %%cl, %%ccnt;\n@%%p bra.uni EXIT;\n"


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
    q = ".reg .u64 %%q, %%end;\n" if with_end else ".reg .u64 %%q;\n"
    return (".reg .pred %%p;\n.reg .u32 %%m, %%mc, %%pb, %%pc, %%o, %%aux, %%w;\n"
            f"{q}.reg .f32 %%v, %%scl, {t};\n.reg .b16 %%h;\n")


def patch_load_ptx(o: Ops, NBT, R, S, PAD, TW, f16: bool) -> str:
    """Load the lane's NBT x PH x PW patch of channel %%cl from shared memory:
    image j, row yy at %%a + j*%%imgb + yy*%%rowb; left halo (PAD elements),
    aligned middle (TW elements), right halo (S-1-PAD elements)."""
    es = 2 if f16 else 4
    L = []
    right = S - 1 - PAD
    for j in range(NBT):
        L.append("mov.u32 %%ra, %%a;\n" if j == 0 else "add.u32 %%a, %%a, %%imgb;\nmov.u32 %%ra, %%a;\n")
        for yy in range(o.PH):
            if yy:
                L.append("add.u32 %%ra, %%ra, %%rowb;\n")
            regs = [o.pt(j, yy, xx) for xx in range(o.PW)]
            segs = []  # (first element, count, vector ok)
            if PAD:
                segs.append((0, PAD, False))
            segs.append((PAD, TW, True))
            if right:
                segs.append((PAD + TW, right, True))
            for first, cnt, vec in segs:
                off0 = first * es
                if not f16:
                    k = 0
                    while k < cnt:
                        w = 4 if (vec and cnt - k >= 4 and (TW * 4) % 16 == 0 and ((k * 4) % 16 == 0)) else \
                            (2 if (vec and cnt - k >= 2 and ((TW * 4) % 8 == 0) and ((k * 4) % 8 == 0)) else 1)
                        dst = regs[first + k:first + k + w]
                        if w == 1:
                            L.append(f"ld.shared.f32 {dst[0]}, [%%ra+{off0 + 4 * k}];\n")
                        else:
                            L.append(f"ld.shared.v{w}.f32 {{{', '.join(dst)}}}, [%%ra+{off0 + 4 * k}];\n")
                        k += w
                else:
                    for k in range(cnt):
                        L.append(f"ld.shared.b16 %%h, [%%ra+{off0 + 2 * k}];\ncvt.f32.f16 {regs[first + k]}, %%h;\n")
    return "".join(L)


def gen_jump(R, S, PAD, KT, NBT, TH, TW, WF, MODE, f16) -> str:
    """Jump-table tap loop over one stage.  The stream of a warp group holds,
    per non-empty input channel, a sentinel (meta = KT*R*S, payload = channel)
    followed by the channel's taps; the group ends with a sentinel of channel C.
    The stage's segment of the stream sits in shared memory at `qs`.  A
    sentinel of a channel outside [c0, c0+cc) ends the stage; any other
    sentinel (re)loads the lane's patch of that channel."""
    nacc = KT * NBT * TH * TW
    o = Ops(R, S, KT, NBT, TH, TW, pt_base=nacc)
    npt = o.npt
    oq = nacc + npt                                    # shared address of the stage's tap segment
    oin = oq + 1                                       # remaining inputs
    names = ["c0", "ccnt", "base", "planeb", "imgb", "rowb", "aux", "scl"]
    op = {n: f"%{oin + i}" for i, n in enumerate(names)}
    NC = KT * R * S
    L = ["{\n", regs_decl(o.P, MODE, with_end=False),
         ".reg .u32 %%cl, %%a, %%ra, %%c0, %%ccnt, %%base, %%planeb, %%imgb, %%rowb, %%qs;\n",
         f"mov.u32 %%c0, {op['c0']};\nmov.u32 %%ccnt, {op['ccnt']};\nmov.u32 %%base, {op['base']};\n"
         f"mov.u32 %%planeb, {op['planeb']};\nmov.u32 %%imgb, {op['imgb']};\nmov.u32 %%rowb, {op['rowb']};\n"
         f"mov.u32 %%aux, {op['aux']};\nmov.f32 %%scl, {op['scl']};\nmov.u32 %%qs, %{oq};\n",
         "TBL: .branchtargets " + ", ".join([f"C{i}" for i in range(NC)] + ["CS"]) + ";\n",
         "ld.shared.v2.u32 {%%m, %%pb}, [%%qs];\n", dispatch_ptx(WF)]
    # THREADED: every block ends with its own dispatch; else one shared loop head
    tail = dispatch_ptx(WF) if THREADED else "bra.uni LOOP;\n"
    if not THREADED:
        L[-1] = "bra.uni LOOP;\n"
    for kk in range(KT):
        for r in range(R):
            for s in range(S):
                L.append(f"C{(kk * R + r) * S + s}:\n" + mac_block(o, kk, r, s, NBT, TH, TW, MODE) + tail)
    L.append(cs_head(WF) + "mad.lo.u32 %%a, %%cl, %%planeb, %%base;\n")
    L.append(patch_load_ptx(o, NBT, R, S, PAD, TW, f16))
    L.append(tail)
    if not THREADED:
        L.append("LOOP:\n" + dispatch_ptx(WF))
    L.append("EXIT:\n}\n")
    outs = [f'"+f"(a[{i}])' for i in range(nacc)] + [f'"+f"(pt[{i}])' for i in range(npt)]
    ins = ['"r"(qs)', '"r"(c0)', '"r"(ccnt)', '"r"(base)', '"r"(planeb)', '"r"(imgb)', '"r"(rowb)', '"r"(aux)',
           '"f"(scl)']
    sig = (f"float (&a)[{nacc}], float (&pt)[{npt}], unsigned qs, unsigned c0, unsigned ccnt, unsigned base, "
           "unsigned planeb, unsigned imgb, unsigned rowb, unsigned aux, float scl")
    return emit(f"{R}, {S}, {PAD}, {KT}, {NBT}, {TH}, {TW}, {WF}, {MODE}, {JUMP}, {'true' if f16 else 'false'}",
                sig, "".join(L), outs, ins)


def gen_mask(R, S, PAD, KT, NBT, TH, TW, WF, MODE, f16) -> str:
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
    return emit(f"{R}, {S}, {PAD}, {KT}, {NBT}, {TH}, {TW}, {WF}, {MODE}, {MASK}, {'true' if f16 else 'false'}",
                sig, "".join(L), outs, ins)


def gen_plane(H, W, R, S, PAD, KT, NBT, WF, MODE, f16) -> str:
    """Whole-plane tap loop (plane.cuh).  Same stream format as gen_jump; the
    lane's patch is the H x W plane of each of its NBT images (registers
    %%x*), the zero padding around it is the literal 0f00000000, and every
    MAC block ends with its own copy of the dispatch (direct threading: no
    branch back to a loop head)."""
    E, F = H + 2 * PAD - R + 1, W + 2 * PAD - S + 1
    HW, EF = H * W, E * F
    P = NBT * EF
    nacc = KT * P
    names = ["qs", "c0", "ccnt", "base", "planeb", "imgb", "aux", "scl"]
    op = {n: f"%{nacc + i}" for i, n in enumerate(names)}

    def acc(kk, j, y, x):
        return f"%{kk * P + j * EF + y * F + x}"

    def pt(j, y, x):  # padded-plane coordinates
        yy, xx = y - PAD, x - PAD
        if 0 <= yy < H and 0 <= xx < W:
            return f"%%x{j * HW + yy * W + xx}"
        return "0f00000000"

    def mac(kk, r, s):
        body = []
        for j in range(NBT):
            for y in range(E):
                for x in range(F):
                    a, q = acc(kk, j, y, x), pt(j, y + r, x + s)
                    if MODE == EXACT:
                        t = f"%%t{(j * E + y) * F + x}"
                        body.append(f"mul.rn.f32 {t}, %%v, {q};\nadd.rn.f32 {a}, {a}, {t};\n")
                    else:
                        body.append(f"fma.rn.f32 {a}, %%v, {q}, {a};\n")
        return "".join(body)

    dispatch = dispatch_ptx(WF)
    t = ", ".join(f"%%t{i}" for i in range(P)) if MODE == EXACT else "%%t0"
    L = ["{\n", ".reg .pred %%p;\n.reg .u32 %%m, %%mc, %%pb, %%pc, %%o, %%aux, %%w;\n",
         f".reg .f32 %%v, %%scl, {t};\n.reg .b16 %%h, %%h0, %%h1, %%h2, %%h3;\n",
         f".reg .f32 %%x<{NBT * HW}>;\n",
         ".reg .u32 %%cl, %%a, %%ra, %%c0, %%ccnt, %%base, %%planeb, %%imgb, %%qs;\n",
         f"mov.u32 %%qs, {op['qs']};\nmov.u32 %%c0, {op['c0']};\nmov.u32 %%ccnt, {op['ccnt']};\n"
         f"mov.u32 %%base, {op['base']};\nmov.u32 %%planeb, {op['planeb']};\nmov.u32 %%imgb, {op['imgb']};\n"
         f"mov.u32 %%aux, {op['aux']};\nmov.f32 %%scl, {op['scl']};\n"]
    labels = [f"C{i}" for i in range(KT * R * S)] + ["CS"]
    L.append("TBL: .branchtargets " + ", ".join(labels) + ";\n")
    L.append("ld.shared.v2.u32 {%%m, %%pb}, [%%qs];\n" + dispatch)
    for kk in range(KT):
        for r in range(R):
            for s_ in range(S):
                L.append(f"C{(kk * R + r) * S + s_}:\n" + mac(kk, r, s_) + dispatch)
    # channel sentinel: exit past the stage, else load the lane's planes of channel pc
    L.append(cs_head(WF) + "mad.lo.u32 %%a, %%cl, %%planeb, %%base;\n")
    for j in range(NBT):
        L.append("mov.u32 %%ra, %%a;\n" if j == 0 else "add.u32 %%ra, %%ra, %%imgb;\n")
        for q in range(0, HW, 4):
            regs = [f"%%x{j * HW + q + i}" for i in range(min(4, HW - q))]
            if not f16:
                if len(regs) == 4:
                    L.append(f"ld.shared.v4.f32 {{{', '.join(regs)}}}, [%%ra+{4 * q}];\n")
                else:
                    for i, rg in enumerate(regs):
                        L.append(f"ld.shared.f32 {rg}, [%%ra+{4 * (q + i)}];\n")
            else:
                if len(regs) == 4:
                    L.append(f"ld.shared.v4.b16 {{%%h0, %%h1, %%h2, %%h3}}, [%%ra+{2 * q}];\n")
                    for i, rg in enumerate(regs):
                        L.append(f"cvt.f32.f16 {rg}, %%h{i};\n")
                else:
                    for i, rg in enumerate(regs):
                        L.append(f"ld.shared.b16 %%h, [%%ra+{2 * (q + i)}];\ncvt.f32.f16 {rg}, %%h;\n")
    L.append(dispatch)
    L.append("EXIT:\n}\n")
    outs = [f'"+f"(a[{i}])' for i in range(nacc)]
    ins = ['"r"(qs)', '"r"(c0)', '"r"(ccnt)', '"r"(base)', '"r"(planeb)', '"r"(imgb)', '"r"(aux)', '"f"(scl)']
    sig = (f"float (&a)[{nacc}], float (&pt)[{NBT * HW}], unsigned qs, unsigned c0, unsigned ccnt, unsigned base, "
           "unsigned planeb, unsigned imgb, unsigned aux, float scl")
    body = emit("", sig, "".join(L), outs, ins)
    targs = f"{H}, {W}, {R}, {S}, {PAD}, {KT}, {NBT}, {WF}, {MODE}, {'true' if f16 else 'false'}"
    return body.replace("struct TapLoop<>", f"struct PlaneLoop<{targs}>")


# whole-plane variants: (H, W, R, S, PAD, KT, NBT, min CTAs/SM)
PLANES = [
    (2, 2, 3, 3, 1, 2, 4, 2), (2, 2, 3, 3, 1, 4, 2, 2), (2, 2, 3, 3, 1, 4, 4, 2), (2, 2, 3, 3, 1, 8, 2, 2),
    (2, 2, 3, 3, 1, 2, 2, 2),
    (4, 4, 3, 3, 1, 2, 2, 2), (4, 4, 3, 3, 1, 4, 1, 2), (4, 4, 3, 3, 1, 4, 2, 2), (4, 4, 3, 3, 1, 8, 1, 2),
    (4, 4, 3, 3, 1, 2, 1, 2),
    (4, 4, 3, 3, 1, 2, 1, 3), (2, 2, 3, 3, 1, 2, 2, 3), (2, 2, 3, 3, 1, 2, 4, 3),
]
PLANE_MODES = [(False, WF_F32, EXACT), (False, WF_F32, FMA), (True, WF_F16, FMA)]
KIND_TILED, KIND_PLANE, KIND_DIRECT, KIND_DIMG, KIND_DWS, KIND_DTM, KIND_TMI, KIND_LANE = 0, 1, 2, 3, 4, 5, 6, 7
# TMEM image-lane variants (tmi.cuh): (W plane, TE rows per lane unit, J images per lane, KW, WQ warps per quarter)
TMIS = [(w, te, j, kw, wq) for (w, te, j) in ((4, 4, 1), (2, 2, 4), (2, 2, 2), (8, 2, 1))
        for kw, wq in ((2, 3), (3, 3), (2, 4), (4, 2))] + [(16, 1, 1, 2, 3), (16, 1, 1, 3, 3), (8, 4, 1, 1, 3), (8, 4, 1, 2, 3)]
# TMEM-operand direct variants (tm.cuh): (TH, LW, KW, M warps per lane quarter)
DTMS = [(8, lw, kw, m) for lw in (32, 16, 8) for kw in (4, 8) for m in (2, 4)] + [(4, 4, kw, m) for kw in (4, 8) for m in (2, 4)]
# warp-specialised direct variants (ws.cuh): (R, S, PAD, TH, LW, KW)
DWS = [(3, 3, 1, th, lw, kw) for lw in (32, 16, 8) for th in (4, 8) for kw in (4, 8)]
# image-lane direct variants (dimg.cuh): (H, KW)
DIMGS = [(4, 1), (4, 2), (4, 4), (2, 1), (2, 2), (2, 4), (2, 8)]
# image-lane position-class kernels (lane.cuh, kind 7): (H = W, images per lane NB, KW, U = tap
# unroll with padded class segments)
LANES = [(h, nb, 1, u) for h in (2, 4) for nb in (1, 2, 4) for u in (1, 2) if not (h == 4 and nb == 4)]
# class split: two warps per output channel, each a fixed half of the position classes (CS = 2)
# 8x8 planes in quadrant tiles (lane.cuh TQ; dispatch = 3): one image per lane, one warp per channel
LANES_TQ = [(8, 1)]
LANES_TQ16 = [(8, 2)]  # f16 storage (two images per 32-bit load), every f16 weight format
# 4x4 output tiles of 16x16 / 32x32 planes (lane.cuh k_tile; dispatch = 4): images per lane
LANES_T4 = [1, 2, 4]
LANES_T4_16 = [2, 4]  # f16 storage, every f16 weight format
TILE_THREADS = {1: 544, 2: 416, 4: 288}  # = lane.cuh tile_max_threads
LANES_CS = [(4, 4, 1, 3), (4, 2, 1, 2), (2, 2, 2, 2), (4, 1, 1, 2), (2, 1, 2, 2), (2, 1, 2, 4), (2, 4, 1, 4), (2, 4, 1, 2)]  # (H, NB, U, CS)
# f16 storage (FHFMA, in-register weight decode of every f16 format): (H = W, NB)
LANES_F16 = [(4, 2, 1), (2, 2, 1), (2, 4, 1), (4, 2, 2), (2, 4, 4)]  # (H, NB, CS)
# f16 opt-in fast mode (SCB_FLAG_FAST): half2 accumulators, HFMA2 -- native f16 weights
LANES_H2 = [(4, 2, 1), (4, 2, 2), (2, 4, 4), (2, 2, 2)]  # (H, NB, CS)
DIMGS_F16 = [(2, 2), (2, 4), (2, 8), (4, 2), (4, 4)]  # f16 storage, FHFMA

# dispatch-free direct variants (direct.cuh): (R, S, PAD, TH, LW, KW, VX)
DIRECTS = [(3, 3, 1, th, lw, kw, 1) for lw in (32, 16, 8) for th in (4, 8) for kw in (4, 8)] + \
          [(3, 3, 1, th, lw, kw, 2) for lw in (32, 16, 8) for th in (4, 8) for kw in (2, 4)] + \
          [(3, 3, 1, 4, 4, 4, 1), (3, 3, 1, 4, 4, 8, 1),
           (5, 5, 2, 4, 32, 4, 1), (5, 5, 2, 4, 16, 4, 1), (5, 5, 2, 8, 8, 4, 1), (5, 5, 2, 4, 16, 4, 2)]
DIRECTS = [d + (2,) for d in DIRECTS] + \
          [(3, 3, 1, th, lw, kw, vx, 4) for lw in (32, 16, 8) for th, kw, vx in
           ((8, 4, 1), (4, 4, 1), (4, 8, 1), (8, 2, 2), (4, 4, 2))] + \
          [(3, 3, 1, 8, lw, 4, 1, 3) for lw in (32, 16, 8)] + \
          [(3, 3, 1, 8, lw, 2, 1, 4) for lw in (32, 16, 8)] + \
          [(3, 3, 1, 8, lw, 2, 2, 3) for lw in (32, 16, 8)] + \
          [(3, 3, 1, 16, lw, kw, 1, 2) for lw in (32, 16) for kw in (2, 4)] + \
          [(3, 3, 1, 4, 4, kw, 2, 2) for kw in (4, 8)] + \
          [(3, 3, 1, th, lw, kw, 1, 4) for lw in (32, 16, 8) for th, kw in ((4, 2), (2, 4))]
# (the last row: small per-lane tiles -- more warps for the 32-image shards of 8 GPUs)
# + min CTAs/SM (4: <= 64 regs)
# wide direct variants (column tiles of 32 for output rows wider than 32, e.g. the
# ImageNet shapes; also rows whose width is no tile width, 28/14/7): (R, S, PAD, TH, LW, KW, min CTAs/SM)
DIRECTS_WIDE = [(3, 3, 1, th, lw, kw, 2) for lw in (32, 16, 8) for th in (4, 8) for kw in (4, 8)] + \
               [(3, 3, 1, 16, 32, 4, 2), (3, 3, 1, 8, 32, 2, 4), (5, 5, 2, 4, 32, 4, 2), (5, 5, 2, 4, 16, 4, 2)] + \
               [(1, 1, 0, 8, lw, kw, 2) for lw in (32, 16, 8) for kw in (4, 8)] + [(1, 1, 0, 16, 32, 4, 2)] + \
               [(3, 3, 1, 2, 2, 4, 2), (3, 3, 1, 4, 4, 8, 2)]
# (2x2 / 4x4 planes as WIDE tiles of 2 / 4 columns, 16 / 8 images per warp: correct, measured
# 110 us vs the image-lane kernel's 92 us on conv5 and 221 vs 217 us on conv4 -- one each kept)
WIDE, ONED = 2, 3                                # kernels.cuh DISPATCH_WIDE / DISPATCH_ONED
# 1D direct variants (H = R = 1, e.g. the reference's cnn-non-static presets): (S, TH, KW)
DIRECTS_1D = [(s, th, kw) for s in (2, 3, 4, 5) for th in (4, 8) for kw in (4, 8)]
# f16-storage direct variants (FHFMA, column pairs): (R, S, PAD, TH, LW, KW)
DIRECTS_F16 = [(3, 3, 1, th, lw, kw) for lw in (32, 16, 8) for th in (4, 8) for kw in (2, 4)] + \
              [(3, 3, 1, 4, 4, kw) for kw in (4, 8)]  # 4x4 planes: 8-byte rows, 16 images per warp
# f16 storage, one column per lane (VX = 1: no shifted row copy): (TH, LW, KW)
DIRECTS_F16_VX1 = [(8, 32, 4), (16, 32, 4), (8, 32, 8), (8, 16, 4), (8, 16, 8), (8, 8, 8)]
# quantized f16 weights decoded IN REGISTER from compact 4-byte taps (kernels.cuh tap_f16):
# 4-bit codebook, int16 fixed point, int16 symmetric affine -- on the shapes the f16 stacks use
QFMTS = (WF_CB4, WF_LIN16, WF_AFF16)
DIRECTS_F16_Q = [(3, 3, 1, 8, lw, kw) for lw in (32, 16, 8) for kw in (2, 4)]
DIRECTS_F16_VX1_Q = [(8, 32, 4), (8, 16, 4), (8, 8, 8)]
DIMGS_F16_Q = [(4, 2), (4, 4), (2, 2), (2, 4)]


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
                key = (R, S, PAD, KT, NBT, TH, TW, wf, mode, d, f16)
                if key not in loops:
                    loops.append(key)
                variants.append((R, S, PAD, KT, NBT, TH, TW, f16, wf, mode, d, minb))
        tile_key = (R, S, PAD, KT, NBT, TH, TW)
        g = groups.setdefault(tile_key, ([], []))
        for l in loops:
            if l not in g[0]:
                g[0].append(l)
        g[1].extend(variants)
    for H, W, R, S, PAD, KT, NBT, minb in PLANES:
        loops, variants = [], []
        for f16, wf, mode in PLANE_MODES:
            loops.append(("plane", H, W, R, S, PAD, KT, NBT, wf, mode, f16))
            variants.append(("plane", H, W, R, S, PAD, KT, NBT, f16, wf, mode, minb))
        groups[("plane", H, W, R, S, PAD, KT, NBT, minb)] = (loops, variants)
    for R, S, PAD, TH, LW, KW, VX, MB in DIRECTS:
        groups[("direct", R, S, PAD, TH, LW, KW, VX, MB)] = (
            [], [("direct", R, S, PAD, TH, LW, KW, VX, MB, mode) for mode in (EXACT, FMA)])
    for R, S, PAD, TH, LW, KW, MB in DIRECTS_WIDE:
        groups[("wide", R, S, PAD, TH, LW, KW, MB)] = (
            [], [("wide", R, S, PAD, TH, LW, KW, MB, mode) for mode in (EXACT, FMA)])
    for S, TH, KW in DIRECTS_1D:
        groups[("oned", S, TH, KW)] = ([], [("oned", S, TH, KW, mode) for mode in (EXACT, FMA)])
    for TH, LW, KW, M in DTMS:
        groups[("dtm", TH, LW, KW, M)] = ([], [("dtm", TH, LW, KW, M, m) for m in (EXACT, FMA)])
    for W, TE, J, KW, WQ in TMIS:
        groups[("tmi", W, TE, J, KW, WQ)] = ([], [("tmi", W, TE, J, KW, WQ, m) for m in (EXACT, FMA)])
    for R, S, PAD, TH, LW, KW in DWS:
        groups[("dws", R, S, PAD, TH, LW, KW)] = ([], [("dws", R, S, PAD, TH, LW, KW, m) for m in (EXACT, FMA)])
    for R, S, PAD, TH, LW, KW in DIRECTS_F16:
        qs = QFMTS if (R, S, PAD, TH, LW, KW) in DIRECTS_F16_Q else ()
        groups[("direct16", R, S, PAD, TH, LW, KW)] = (
            [], [("direct16", R, S, PAD, TH, LW, KW, wf) for wf in (WF_F16,) + qs])
    for TH, LW, KW in DIRECTS_F16_VX1:
        qs = QFMTS if (TH, LW, KW) in DIRECTS_F16_VX1_Q else ()
        groups[("direct16v1", TH, LW, KW)] = ([], [("direct16v1", TH, LW, KW, wf) for wf in (WF_F16,) + qs])
    for H, KW in DIMGS:
        groups[("dimg", H, KW)] = ([], [("dimg", H, KW, mode) for mode in (EXACT, FMA)])
    for H, KW in DIMGS_F16:
        qs = QFMTS if (H, KW) in DIMGS_F16_Q else ()
        groups[("dimg16", H, KW)] = ([], [("dimg16", H, KW, wf) for wf in (WF_F16,) + qs])
    for H, NB, KW, U in LANES:
        groups[("lane", H, NB, KW, U)] = ([], [("lane", H, NB, KW, U, m) for m in (EXACT, FMA)])
    for H, NB in LANES_TQ:
        groups[("lanetq", H, NB)] = ([], [("lanetq", H, NB, m) for m in (EXACT, FMA)])
    for NB in LANES_T4:
        groups[("lanet4", NB)] = ([], [("lanet4", NB, m) for m in (EXACT, FMA)])
    for NB in LANES_T4_16:
        groups[("lanet4h", NB)] = ([], [("lanet4h", NB, wf) for wf in (WF_F16,) + QFMTS])
    for H, NB in LANES_TQ16:
        groups[("lanetq16", H, NB)] = ([], [("lanetq16", H, NB, wf) for wf in (WF_F16,) + QFMTS])
    for H, NB, U, CS in LANES_CS:
        groups[("lanecs", H, NB, U, CS)] = ([], [("lanecs", H, NB, U, CS, m) for m in (EXACT, FMA)])
    for H, NB, CS in LANES_H2:
        groups[("laneh2", H, NB, CS)] = ([], [("laneh2", H, NB, CS)])
    for H, NB, CS in LANES_F16:
        groups[("lane16", H, NB, CS)] = ([], [("lane16", H, NB, CS, wf) for wf in (WF_F16,) + QFMTS])
    items = sorted(groups.values(), key=lambda t: -len(t[1]))
    parts = [[] for _ in range(N_PARTS)]
    load = [0] * N_PARTS
    for t in items:
        i = load.index(min(load))
        parts[i].append(t)
        load[i] += len(t[1])
    total_v = 0
    for i, part in enumerate(parts):
        src = ["// GENERATED by gen_taploop.py -- do not edit.\n#include \"tiled.cuh\"\n#include \"plane.cuh\"\n#include \"direct.cuh\"\n#include \"dimg.cuh\"\n#include \"ws.cuh\"\n#include \"tm.cuh\"\n#include \"tmi.cuh\"\n#include \"lane.cuh\"\n"
               "#include \"variants.h\"\n\nnamespace scb {\n\n"]
        ents = []
        for loops, variants in part:
            for key in loops:
                if key[0] == "plane":
                    src.append(gen_plane(*key[1:]))
                    continue
                R, S, PAD, KT, NBT, TH, TW, wf, mode, d, f16 = key
                src.append((gen_jump if d == JUMP else gen_mask)(R, S, PAD, KT, NBT, TH, TW, wf, mode, f16))
            for v in variants:
                if v[0] == "dtm":
                    _, TH, LW, KW, M, mode = v
                    ents.append(f"    {{{{3, 3, {KW}, {M}, {TH}, {LW}, SCB_F32, {WF_F32}, {mode}, {JUMP}, 1, "
                                f"{KIND_DTM}}}, nullptr, &launch_dtm_t<3, 3, 1, {TH}, {LW}, {KW}, {M}, {mode}>}},\n")
                    continue
                if v[0] == "lanetq":  # info: dispatch = 3 (quadrant tiles)
                    _, H, NB, mode = v
                    ents.append(f"    {{{{3, 3, 1, {NB}, {H}, {H}, SCB_F32, {WF_F32}, {mode}, 3, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, 544, nullptr, "
                                f"&launch_lane_t<{H}, {H}, {NB}, 1, {mode}, 1, false, {WF_F32}, 1, 1>}},\n")
                    continue
                if v[0] == "lanet4":  # info: dispatch = 4 (4x4 tiles), th = tw = 4
                    _, NB, mode = v
                    ents.append(f"    {{{{3, 3, 1, {NB}, 4, 4, SCB_F32, {WF_F32}, {mode}, 4, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, {TILE_THREADS[NB]}, nullptr, "
                                f"&launch_tile_t<{NB}, {mode}>}},\n")
                    continue
                if v[0] == "lanet4h":
                    _, NB, wf = v
                    ents.append(f"    {{{{3, 3, 1, {NB}, 4, 4, SCB_F16, {wf}, {FMA}, 4, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, {TILE_THREADS[NB]}, nullptr, "
                                f"&launch_tile_t<{NB}, {FMA}, true, {wf}>}},\n")
                    continue
                if v[0] == "lanetq16":
                    _, H, NB, wf = v
                    ents.append(f"    {{{{3, 3, 1, {NB}, {H}, {H}, SCB_F16, {wf}, {FMA}, 3, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, 544, nullptr, "
                                f"&launch_lane_t<{H}, {H}, {NB}, 1, {FMA}, 1, true, {wf}, 1, 1>}},\n")
                    continue
                if v[0] == "lanecs":  # info: kt = CS warps per output channel
                    _, H, NB, U, CS, mode = v
                    ents.append(f"    {{{{3, 3, {CS}, {NB}, {H}, {H}, SCB_F32, {WF_F32}, {mode}, {U}, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, 1024, nullptr, "
                                f"&launch_lane_t<{H}, {H}, {NB}, 1, {mode}, {U}, false, {WF_F32}, {CS}>}},\n")
                    continue
                if v[0] == "laneh2":  # mode 2 = MODE_HALF2
                    _, H, NB, CS = v
                    ents.append(f"    {{{{3, 3, {CS}, {NB}, {H}, {H}, SCB_F16, {WF_F16}, 2, 1, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, {1024 if CS > 1 else 544}, nullptr, "
                                f"&launch_lane_t<{H}, {H}, {NB}, 1, 2, 1, true, {WF_F16}, {CS}>}},\n")
                    continue
                if v[0] == "lane16":
                    _, H, NB, CS, wf = v
                    ents.append(f"    {{{{3, 3, {CS}, {NB}, {H}, {H}, SCB_F16, {wf}, {FMA}, 1, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, {1024 if CS > 1 else 544}, nullptr, "
                                f"&launch_lane_t<{H}, {H}, {NB}, 1, {FMA}, 1, true, {wf}, {CS}>}},\n")
                    continue
                if v[0] == "lane":  # info: kt = KW, nbt = NB, th = H, tw = W, dispatch = U
                    _, H, NB, KW, U, mode = v
                    ents.append(f"    {{{{3, 3, {KW}, {NB}, {H}, {H}, SCB_F32, {WF_F32}, {mode}, {U}, 1, "
                                f"{KIND_LANE}}}, nullptr, nullptr, {288 if H >= 8 else 544}, nullptr, "
                                f"&launch_lane_t<{H}, {H}, {NB}, {KW}, {mode}, {U}>}},\n")
                    continue
                if v[0] == "tmi":  # info: kt = KW, nbt = J, th = TE, tw = W, dispatch = WQ
                    _, W, TE, J, KW, WQ, mode = v
                    ents.append(f"    {{{{3, 3, {KW}, {J}, {TE}, {W}, SCB_F32, {WF_F32}, {mode}, {WQ}, 1, "
                                f"{KIND_TMI}}}, nullptr, nullptr, {32 * (4 + 4 * WQ)}, "
                                f"&launch_tmi_t<{W}, {TE}, {J}, {KW}, {WQ}, {mode}>}},\n")
                    continue
                if v[0] == "dws":
                    _, R, S, PAD, TH, LW, KW, mode = v
                    ents.append(f"    {{{{{R}, {S}, {KW}, 1, {TH}, {LW}, SCB_F32, {WF_F32}, {mode}, {JUMP}, {PAD}, "
                                f"{KIND_DWS}}}, nullptr, &launch_dws_t<{R}, {S}, {PAD}, {TH}, {LW}, {KW}, {mode}>}},\n")
                    continue
                if v[0] == "direct16v1":
                    _, TH, LW, KW, wf = v
                    ents.append(f"    {{{{3, 3, {KW}, 1, {TH}, {LW}, SCB_F16, {wf}, {FMA}, {JUMP}, 1, "
                                f"{KIND_DIRECT}}}, nullptr, &launch_direct_t<3, 3, 1, {TH}, {LW}, {KW}, "
                                f"{FMA}, 1, 2, true, false, false, {wf}>, 512}},\n")
                    continue
                if v[0] == "direct16":
                    _, R, S, PAD, TH, LW, KW, wf = v
                    ents.append(f"    {{{{{R}, {S}, {KW}, 2, {TH}, {LW}, SCB_F16, {wf}, {FMA}, {JUMP}, {PAD}, "
                                f"{KIND_DIRECT}}}, nullptr, &launch_direct_t<{R}, {S}, {PAD}, {TH}, {LW}, {KW}, "
                                f"{FMA}, 2, 2, true, false, false, {wf}>, 512}},\n")
                    continue
                if v[0] == "dimg16":
                    _, H, KW, wf = v
                    ents.append(f"    {{{{3, 3, {KW}, 1, {H}, {H}, SCB_F16, {wf}, {FMA}, {JUMP}, 1, "
                                f"{KIND_DIMG}}}, nullptr, &launch_dimg_t<{H}, {KW}, {FMA}, true, {wf}>, 512}},\n")
                    continue
                if v[0] == "dimg":
                    _, H, KW, mode = v
                    ents.append(f"    {{{{3, 3, {KW}, 1, {H}, {H}, SCB_F32, {WF_F32}, {mode}, {JUMP}, 1, "
                                f"{KIND_DIMG}}}, nullptr, &launch_dimg_t<{H}, {KW}, {mode}>, 512}},\n")
                    continue
                if v[0] == "oned":
                    _, S, TH, KW, mode = v
                    ents.append(f"    {{{{1, {S}, {KW}, 1, {TH}, 32, SCB_F32, {WF_F32}, {mode}, {ONED}, 0, "
                                f"{KIND_DIRECT}}}, nullptr, &launch_direct_t<1, {S}, 0, {TH}, 32, {KW}, "
                                f"{mode}, 1, 2, false, true, true>, 512}},\n")
                    continue
                if v[0] == "wide":
                    _, R, S, PAD, TH, LW, KW, MB, mode = v
                    ents.append(f"    {{{{{R}, {S}, {KW}, 1, {TH}, {LW}, SCB_F32, {WF_F32}, {mode}, {WIDE}, {PAD}, "
                                f"{KIND_DIRECT}}}, nullptr, &launch_direct_t<{R}, {S}, {PAD}, {TH}, {LW}, {KW}, "
                                f"{mode}, 1, {MB}, false, true>, {512 if MB == 2 else 256}}},\n")
                    continue
                if v[0] == "direct":
                    _, R, S, PAD, TH, LW, KW, VX, MB, mode = v
                    ents.append(f"    {{{{{R}, {S}, {KW}, {VX}, {TH}, {LW}, SCB_F32, {WF_F32}, {mode}, {JUMP}, {PAD}, "
                                f"{KIND_DIRECT}}}, nullptr, &launch_direct_t<{R}, {S}, {PAD}, {TH}, {LW}, {KW}, "
                                f"{mode}, {VX}, {MB}>, {512 if MB == 2 else 256}}},\n")
                    continue
                if v[0] == "plane":
                    _, H, W, R, S, PAD, KT, NBT, f16, wf, mode, minb = v
                    io = "SCB_F16" if f16 else "SCB_F32"
                    tf = "true" if f16 else "false"
                    ents.append(f"    {{{{{R}, {S}, {KT}, {NBT}, {H}, {W}, {io}, {wf}, {mode}, {JUMP}, {PAD}, "
                                f"{KIND_PLANE}}}, &launch_plane_t<{H}, {W}, {R}, {S}, {PAD}, {KT}, {NBT}, {tf}, "
                                f"{wf}, {mode}, {minb}>}},\n")
                    continue
                R, S, PAD, KT, NBT, TH, TW, f16, wf, mode, d, minb = v
                io = "SCB_F16" if f16 else "SCB_F32"
                tf = "true" if f16 else "false"
                ents.append(f"    {{{{{R}, {S}, {KT}, {NBT}, {TH}, {TW}, {io}, {wf}, {mode}, {d}, {PAD}, "
                            f"{KIND_TILED}}}, &launch_tiled_t<{R}, {S}, {PAD}, {KT}, {NBT}, {TH}, {TW}, {tf}, "
                            f"{wf}, {mode}, {d}, {minb}>}},\n")
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
