"""Pin the CPU oracle (oracle/) to the reference: every fixture under
tests/golden/ was produced by the reference package itself
(tests/golden/make_golden.py).  CPU only."""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from golden_gen import c1_configs, sha256
from oracle import oracle as orc


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def test_select_padding_zeros_kats():
    for case in json.loads((GOLDEN / "select_zeros.json").read_text()):
        got = orc.select_padding_zeros(np.array(case["flat"], np.float64), case["deficit"])
        assert got.tolist() == case["chosen"], case


def test_build_csr_bit_exact():
    z = np.load(GOLDEN / "csr_cases.npz")
    meta = z["meta"]
    for i, (h, w, p, unify, level) in enumerate(meta):
        vals, colidx, rowptr, lvl = orc.build_csr(z[f"w{i}"], int(h), int(w), int(p), bool(unify))
        assert lvl == level
        assert np.array_equal(rowptr, z[f"rowptr{i}"])
        assert np.array_equal(colidx, z[f"colidx{i}"])
        assert vals.dtype == z[f"values{i}"].dtype
        assert np.array_equal(_bits(vals), _bits(z[f"values{i}"])), i


def test_conv_cases_bit_exact():
    z = np.load(GOLDEN / "conv_cases.npz")
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta):
        x, w = z[f"x{i}"], z[f"w{i}"]
        b = z[f"b{i}"] if m["has_bias"] else None
        k, c, r, s = w.shape
        vals, colidx, rowptr, _ = orc.build_csr(w, x.shape[2], x.shape[3], m["padding"], m["unify"])
        out = orc.conv_sparse(x, vals, colidx, rowptr, k, r, s, m["stride"], m["padding"], b, sb=m["sb"])
        assert out.dtype == z[f"out{i}"].dtype
        assert np.array_equal(_bits(out), _bits(z[f"out{i}"])), m["name"]
        dense = orc.conv_dense_direct(x, w, b, m["stride"], m["padding"])
        assert np.array_equal(_bits(dense), _bits(z[f"dense{i}"])), m["name"]


def test_sub_batch_invariance():
    z = np.load(GOLDEN / "conv_cases.npz")
    i = 1  # make_case2: n=8
    x, w, b = z[f"x{i}"], z[f"w{i}"], z[f"b{i}"]
    vals, colidx, rowptr, _ = orc.build_csr(w, 16, 16, 1)
    outs = [orc.conv_sparse(x, vals, colidx, rowptr, 8, 3, 3, 1, 1, b, sb=sb) for sb in (1, 2, 4, 8, 16)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_c1_digests():
    recs = json.loads((GOLDEN / "c1_digests.json").read_text())
    for cfg, rec in zip(c1_configs(), recs):
        x, w, bias = cfg["x"], cfg["w"], cfg["bias"]
        assert sha256(x, w, bias) == rec["in_sha"], "input regeneration drifted"
        sh = cfg["shape"]
        vals, colidx, rowptr, lvl = orc.build_csr(w, sh["h"], sh["w"], sh["padding"])
        assert lvl == rec["level"]
        out = orc.conv_sparse(x, vals, colidx, rowptr, sh["k"], sh["r"], sh["s"],
                              sh["stride"], sh["padding"], bias)
        assert sha256(out) == rec["out_sha"], sh
        if "out16_sha" in rec:
            w16 = w.astype(np.float16)
            v16, c16, r16, _ = orc.build_csr(w16, sh["h"], sh["w"], sh["padding"])
            o16 = orc.conv_sparse(x.astype(np.float16), v16, c16, r16, sh["k"], sh["r"], sh["s"],
                                  sh["stride"], sh["padding"], bias.astype(np.float16))
            assert sha256(o16) == rec["out16_sha"], sh


def test_fake_quant_matches_reference():
    """oracle.fake_quant == the reference's fake_quant_activation (quantize.py:332-338)
    on f32 / f16 / f64 arrays, asymmetric and symmetric, incl. exact code ties."""
    z = np.load(GOLDEN / "fake_quant_cases.npz")
    meta = json.loads(str(z["meta"]))
    assert len(meta) == 12
    for i, m in enumerate(meta):
        y = orc.fake_quant(z[f"x{i}"], m["params"])
        assert y.dtype == z[f"y{i}"].dtype and np.array_equal(_bits(y), _bits(z[f"y{i}"])), (i, m)


def test_reference_quantizers_restated_bitwise():
    """synth.reference_quantize reproduces the reference's quantize_weights_array
    ("fixed", 16), ("codebook", 16, seed=0) and ("affine", 16) on every VGG-16/CIFAR layer's f16 CSR
    values bit for bit (digests recorded from the reference, make_quant_vgg.py)."""
    import hashlib
    import json

    import paper_2011_06295_b200 as sc
    from paper_2011_06295_b200.synth import f16_scaled, make_layer_weights, reference_quantize, vgg16_cifar
    fx = json.loads((GOLDEN / "quant_vgg.json").read_text())
    recs = {r["name"]: r for r in fx["layers"]}
    for spec, _ in vgg16_cifar(0.9):
        r = recs[spec.name]
        vals = sc.build_csr(f16_scaled(make_layer_weights(spec, 0)), spec.shape).values
        assert hashlib.sha256(vals.tobytes()).hexdigest() == r["values_sha"], spec.name
        fixed = reference_quantize(vals, "fixed")
        assert hashlib.sha256(fixed.tobytes()).hexdigest() == r["fixed"]["sha"], spec.name
        cb = reference_quantize(vals, "codebook", r["codebook"]["centers"], r["codebook"]["pin_zero"])
        assert hashlib.sha256(cb.tobytes()).hexdigest() == r["codebook"]["sha"], spec.name
        assert len(np.unique(cb)) <= 16
        aff = reference_quantize(vals, "affine")
        assert hashlib.sha256(aff.tobytes()).hexdigest() == r["affine"]["sha"], spec.name
        from paper_2011_06295_b200.synth import affine_quantize
        assert affine_quantize(vals, 16)[1] == r["affine"]["step"]
