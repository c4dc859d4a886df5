"""Parity of the sm_100a engine with the reference (GPU).

Every comparison is bitwise unless stated: the engine's exact mode performs
the reference's arithmetic (bias first, then product and sum separately
rounded in colidx order; sc/_kernels.py:53-85), and f16 storage is exact with
FFMA because f16*f16 products are exact in f32.  References used:
  * golden outputs recorded from the reference package (tests/golden/),
  * the C oracle (oracle/, itself pinned to those goldens),
  * the reference's tolerance rule |out-ref| <= tol*(|ref|+1) where the
    contract is a tolerance (fast-math mode, north star 1e-5 / 1e-2).
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from golden_gen import c1_configs, make_case, random_sparse_weights, sha256

pytestmark = pytest.mark.gpu



def relu_pool_ref(ref):
    """The reference's glue in its own dtype (store.py:284): np.maximum(conv, 0) on the
    conv output as stored (f16 rounded first), then the 2x2 max-pool."""
    r = np.maximum(ref, ref.dtype.type(0))
    n, k, e, f = r.shape
    return r.reshape(n, k, e // 2, 2, f // 2, 2).max(axis=(3, 5))

def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def beq(a, b):
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(bits(a), bits(b))


@pytest.fixture(scope="module")
def sc():
    import paper_2011_06295_b200 as sc
    return sc


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


def _shape(sc, x, w, stride=1, padding=0):
    k, c, r, s = w.shape
    return sc.ConvShape(n=x.shape[0], c=c, h=x.shape[2], w=x.shape[3], k=k, r=r, s=s,
                        stride=stride, padding=padding)


# ---------------------------------------------------------------------------
# golden vectors from the reference
# ---------------------------------------------------------------------------

def test_golden_conv_cases(sc):
    z = np.load(GOLDEN / "conv_cases.npz")
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta):
        x, w = z[f"x{i}"], z[f"w{i}"]
        b = z[f"b{i}"] if m["has_bias"] else None
        sh = _shape(sc, x, w, m["stride"], m["padding"])
        kern = sc.build_csr(w, sh, unify=m["unify"])
        fn = sc.conv_sparse_1d if m["name"].startswith("seq1d") else sc.conv_sparse
        out = fn(x, kern, b, sc.EnginePlan(sub_batch_size=m["sb"]))
        assert beq(out, z[f"out{i}"]), m["name"]
        # the independent generic kernel agrees bitwise as well
        ref_out, macs = sc.conv_sparse_reference(x, kern, b)
        assert beq(ref_out, z[f"out{i}"]), m["name"]
        assert macs == x.shape[0] * kern.nnz * sh.e * sh.f


def test_c1_random_configs_bitwise(sc):
    """Acceptance C1 (tests/test_acceptance.py:63-92): 200 random configs,
    f32 and the every-5th f16 subset, bit-identical to the reference."""
    recs = json.loads((GOLDEN / "c1_digests.json").read_text())
    for cfg, rec in zip(c1_configs(), recs):
        x, w, bias = cfg["x"], cfg["w"], cfg["bias"]
        assert sha256(x, w, bias) == rec["in_sha"]
        sh = sc.ConvShape(**cfg["shape"])
        kern = sc.build_csr(w, sh)
        out = sc.conv_sparse(x, kern, bias)
        assert sha256(out) == rec["out_sha"], cfg["shape"]
        if "out16_sha" in rec:
            k16 = sc.build_csr(w.astype(np.float16), sh)
            o16 = sc.conv_sparse(x.astype(np.float16), k16, bias.astype(np.float16))
            assert sha256(o16) == rec["out16_sha"], cfg["shape"]


def test_baseline_layer_digests(sc):
    """BASELINE layer shapes (batch 2) through make_layer_weights: weights,
    CSR and outputs (f32 and f16) bit-identical to the reference's."""
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    for rec in json.loads((GOLDEN / "layer_digests.json").read_text()):
        sh = sc.ConvShape(n=2, c=rec["c"], h=rec["hw"], w=rec["hw"], k=rec["k"], r=3, s=3, padding=1)
        w = make_layer_weights(LayerSpec(rec["name"], sh, rec["sparsity"]), seed=0)
        x, b = bench_inputs(sh, 2)
        assert sha256(w) == rec["w_sha"] and sha256(x, b) == rec["x_sha"]
        kern = sc.build_csr(w, sh)
        assert sha256(kern.values, kern.colidx, kern.rowptr) == rec["csr_sha"]
        assert sha256(sc.conv_sparse(x, kern, b)) == rec["out_sha"], rec["name"]
        k16 = sc.build_csr(w.astype(np.float16), sh)
        o16 = sc.conv_sparse(x.astype(np.float16), k16, b.astype(np.float16))
        assert sha256(o16) == rec["out16_sha"], rec["name"]


# ---------------------------------------------------------------------------
# reference test_engine.py behaviour (pkg/tests/test_engine.py:20-170)
# ---------------------------------------------------------------------------

class TestEngineContract:
    def test_dense_special_case_bit_exact(self, sc, orc):
        x, wt, bias, _ = make_case(0, sparsity=0.0)
        sh = _shape(sc, x, wt, 1, 1)
        out = sc.conv_sparse(x, sc.build_csr(wt, sh), bias)
        assert beq(out, orc.conv_dense_direct(x, wt, bias, 1, 1))

    def test_all_zero_kernel_is_bias(self, sc):
        x, wt, bias, _ = make_case(1)
        sh = _shape(sc, x, wt, 1, 1)
        out = sc.conv_sparse(x, sc.build_csr(np.zeros_like(wt), sh), bias)
        assert np.array_equal(out, np.broadcast_to(bias[None, :, None, None], out.shape))

    def test_plan_invariance_and_oracle(self, sc, orc):
        x, wt, bias, _ = make_case(2, n=8, c=4, h=16, w=16, k=8, sparsity=0.9)
        sh = _shape(sc, x, wt, 1, 1)
        kern = sc.build_csr(wt, sh)
        outs = [sc.conv_sparse(x, kern, bias, sc.EnginePlan(sub_batch_size=sb)) for sb in (1, 2, 4, 8, 16)]
        for o in outs[1:]:
            assert beq(o, outs[0])
        ref = orc.conv_oracle_f64(x, wt, bias, 1, 1)
        assert orc.rel_ok(outs[0], ref, 1e-4)

    def test_worker_invariance(self, sc):
        x, wt, bias, _ = make_case(3, n=4, sparsity=0.8)
        kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
        outs = [sc.conv_sparse(x, kern, bias, sc.EnginePlan(worker_count=wc)) for wc in (1, 2, 64)]
        assert beq(outs[0], outs[1]) and beq(outs[0], outs[2])

    def test_odd_batch(self, sc):
        x, wt, bias, _ = make_case(4, n=3)
        kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
        o4 = sc.conv_sparse(x, kern, bias, sc.EnginePlan(sub_batch_size=4))
        o1 = sc.conv_sparse(x, kern, bias, sc.EnginePlan(sub_batch_size=1))
        assert o4.shape[0] == 3 and beq(o4, o1)

    def test_f16_storage(self, sc, orc):
        x, wt, bias, _ = make_case(6, dtype=np.float16, sparsity=0.5)
        kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
        out = sc.conv_sparse(x, kern, bias)
        assert out.dtype == np.float16
        assert orc.rel_ok(out, orc.conv_oracle_f64(x, wt, bias, 1, 1), 1e-2)

    def test_shape_mismatch(self, sc):
        x, wt, bias, _ = make_case(7)
        kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
        with pytest.raises(sc.ShapeError):
            sc.conv_sparse(x[:, :2], kern, bias)

    def test_bad_plan(self, sc):
        with pytest.raises(sc.ShapeError):
            sc.EnginePlan(sub_batch_size=3)
        with pytest.raises(sc.ShapeError):
            sc.EnginePlan(worker_count=0)

    def test_1d_pair_kernel(self, sc):
        x = np.full((1, 1, 1, 10), 3.0, np.float32)
        w = np.ones((1, 1, 1, 2), np.float32)
        kern = sc.build_csr(w, sc.ConvShape(n=1, c=1, h=1, w=10, k=1, r=1, s=2))
        assert np.all(sc.conv_sparse_1d(x, kern) == np.float32(6.0))

    def test_1d_requires_geometry(self, sc):
        x, wt, bias, _ = make_case(10)
        kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
        with pytest.raises(sc.ShapeError):
            sc.conv_sparse_1d(x, kern, bias)

    def test_mac_counts(self, sc):
        x, wt, bias, _ = make_case(11, sparsity=0.8)
        sh = _shape(sc, x, wt, 1, 1)
        kern = sc.build_csr(wt, sh)
        _, macs = sc.conv_sparse_reference(x, kern, bias)
        assert macs == sc.sparse_mac_count(kern, 2) == 2 * sh.k * sh.e * sh.f * kern.sparse_level
        assert sc.dense_mac_count(sh, 2) == 2 * sh.k * sh.e * sh.f * sh.c * sh.r * sh.s

    def test_tune_sub_batch(self, sc):
        x, wt, bias, _ = make_case(15, n=8)
        kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
        best, timings = sc.tune_sub_batch(x, kern, bias, candidates=(1, 2, 4), repetitions=2, warmups=1)
        assert timings[best] <= min(timings.values()) and set(timings) == {1, 2, 4}


# ---------------------------------------------------------------------------
# launch-configuration invariance (acceptance C3, tests/test_acceptance.py:127-144)
# ---------------------------------------------------------------------------

def _all_launch_outputs(sc, x, kern, bias, max_cands=None):
    import torch
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.engine import _io_dtype
    xd = torch.from_numpy(x).cuda()
    io = _io_dtype(x.dtype, kern)
    layer = device_layer(kern, 0, io)
    cands = layer.candidates(x.shape[0])
    assert cands, "no tiled variant for this geometry"
    if max_cands:
        cands = cands[:: max(1, len(cands) // max_cands)]
    outs = []
    for c in cands + [None]:
        plan = sc.EnginePlan(launch=c)
        if c is None:
            o, _ = sc.conv_sparse_reference(xd, kern, bias)
        else:
            o = sc.conv_sparse(xd, kern, bias, plan)
        outs.append((c, o.cpu().numpy()))
    return outs


def test_c3_launch_invariance(sc, orc):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((4, 8, 16, 16)).astype(np.float32)
    w = random_sparse_weights(rng, 16, 8, 3, 3, 0.9)
    b = rng.standard_normal(16).astype(np.float32)
    sh = sc.ConvShape(n=4, c=8, h=16, w=16, k=16, r=3, s=3, padding=1)
    kern = sc.build_csr(w, sh)
    v, ci, rp, _ = orc.build_csr(w, 16, 16, 1)
    ref = orc.conv_sparse(x, v, ci, rp, 16, 3, 3, 1, 1, b)
    for c, o in _all_launch_outputs(sc, x, kern, b):
        assert beq(o, ref), c


@pytest.mark.parametrize("c,hw,k,sp,n", [(64, 32, 64, 0.9, 4), (128, 16, 128, 0.9, 6),
                                         (256, 8, 256, 0.9, 10), (512, 4, 512, 0.95, 34),
                                         (512, 2, 512, 0.9, 130), (3, 32, 64, 0.9, 3)])
def test_vgg_layer_all_launches_bitwise(sc, orc, c, hw, k, sp, n):
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, sp), seed=0)
    x, b = bench_inputs(sh, n)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    for cfg, o in _all_launch_outputs(sc, x, kern, b, max_cands=24):
        assert beq(o, ref), cfg


@pytest.mark.parametrize("dtype", [np.float16])
def test_f16_all_launches_bitwise(sc, orc, dtype):
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=6, c=64, h=16, w=16, k=64, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, 0.9), seed=0).astype(dtype)
    x, b = bench_inputs(sh, 6)
    x, b = x.astype(dtype), b.astype(dtype)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 64, 3, 3, 1, 1, b)
    for cfg, o in _all_launch_outputs(sc, x, kern, b, max_cands=24):
        assert beq(o, ref), cfg


# ---------------------------------------------------------------------------
# quantised weights dequantised in registers
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("key,fmt", [("codebook16_float32", "cb4"), ("codebook16_float16", "cb4"),
                                     ("codebook4_float32", "cb4"), ("fixed16_float32", "lin16"),
                                     ("fixed8_float32", "lin16"), ("fixed16_float16", "lin16"),
                                     ("fixed8_float16", "lin16")])
def test_quantized_formats_bitwise(sc, orc, key, fmt):
    z = np.load(GOLDEN / "quant_cases.npz")
    wq = z[key]                              # reference quantize_weights_array output
    rng = np.random.default_rng(11)
    n = 6
    x = rng.standard_normal((n, 6, 12, 12)).astype(wq.dtype)
    b = rng.standard_normal(8).astype(wq.dtype)
    sh = sc.ConvShape(n=n, c=6, h=12, w=12, k=8, r=3, s=3, padding=1)
    kern = sc.build_csr(wq, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 8, 3, 3, 1, 1, b)
    native = sc.conv_sparse(x, kern, b)
    quant = sc.conv_sparse(x, kern, b, sc.EnginePlan(weight_format=fmt))
    assert beq(native, ref) and beq(quant, ref)
    # direct kernels take the quantized formats decoded on upload: every kind, bitwise
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    sh16 = sc.ConvShape(n=n, c=6, h=16, w=16, k=8, r=3, s=3, padding=1)
    x16 = rng.standard_normal((n, 6, 16, 16)).astype(wq.dtype)
    k16 = sc.build_csr(wq, sh16)
    ref16 = orc.conv_sparse(x16, k16.values, k16.colidx, k16.rowptr, 8, 3, 3, 1, 1, b)
    layer = device_layer(k16, 0, wq.dtype, fmt)
    vs = _abi.variants()
    cands = layer.candidates(n)
    kinds = {vs[cf[0]]["kind"] for cf in cands}
    assert 2 in kinds, kinds
    xd = torch.from_numpy(x16).cuda()
    for cf in [cf for cf in cands if vs[cf[0]]["kind"] == 2][::7]:
        o = sc.conv_sparse(xd, k16, b, sc.EnginePlan(weight_format=fmt, launch=cf)).cpu().numpy()
        assert beq(o, ref16), cf


def test_affine_weights_rejected_by_lin16(sc):
    z = np.load(GOLDEN / "quant_cases.npz")
    wq = z["affine16_float32"]
    sh = sc.ConvShape(n=1, c=6, h=12, w=12, k=8, r=3, s=3, padding=1)
    kern = sc.build_csr(wq, sh)
    x = np.ones((1, 6, 12, 12), np.float32)
    with pytest.raises(sc.SparseConvError):
        sc.conv_sparse(x, kern, None, sc.EnginePlan(weight_format="lin16"))


# ---------------------------------------------------------------------------
# modes and epilogues
# ---------------------------------------------------------------------------

def test_fast_math_within_north_star_tolerance(sc, orc):
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=8, c=128, h=16, w=16, k=128, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, 0.9), seed=0)
    x, b = bench_inputs(sh, 8)
    kern = sc.build_csr(w, sh)
    out = sc.conv_sparse(x, kern, b, sc.EnginePlan(fast_math=True))
    ref = orc.conv_oracle_f64(x, w, b, 1, 1)
    assert orc.rel_ok(out, ref, 1e-5)


def test_fused_relu_pool_epilogue(sc):
    import torch
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=8, c=64, h=16, w=16, k=64, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, 0.9), seed=0)
    x, b = bench_inputs(sh, 8)
    kern = sc.build_csr(w, sh)
    xd = torch.from_numpy(x).cuda()
    y = sc.conv_sparse(xd, kern, b)
    want = torch.nn.functional.max_pool2d(torch.relu(y), 2)
    got = sc.conv_sparse(xd, kern, b, relu=True, pool=True)
    assert torch.equal(got, want)
    got_relu = sc.conv_sparse(xd, kern, b, relu=True)
    assert torch.equal(got_relu, torch.relu(y))


def test_torch_input_zero_copy_path(sc):
    import torch
    x, wt, bias, _ = make_case(2, n=8, c=4, h=16, w=16, k=8, sparsity=0.9)
    kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
    a = sc.conv_sparse(x, kern, bias)
    t = sc.conv_sparse(torch.from_numpy(x).cuda(), kern, torch.from_numpy(bias).cuda())
    assert t.is_cuda and beq(t.cpu().numpy(), a)


def test_f64_generic(sc, orc):
    x, wt, bias, _ = make_case(20, dtype=np.float64, sparsity=0.6)
    kern = sc.build_csr(wt, _shape(sc, x, wt, 1, 1))
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, wt.shape[0], 3, 3, 1, 1, bias)
    assert beq(sc.conv_sparse(x, kern, bias), ref)


def test_tune_launch_picks_valid_and_identical(sc, orc):
    import torch
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    from paper_2011_06295_b200.tuner import tune_launch
    sh = sc.ConvShape(n=32, c=128, h=8, w=8, k=128, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, 0.9), seed=0)
    x, b = bench_inputs(sh, 32)
    kern = sc.build_csr(w, sh)
    best, timings = tune_launch(torch.from_numpy(x).cuda(), kern, b, repetitions=2, warmups=1,
                                max_candidates=16)
    assert best in timings and timings[best] == min(timings.values())
    out = sc.conv_sparse(x, kern, b)  # now uses the tuned launch
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 128, 3, 3, 1, 1, b)
    assert beq(out, ref)


# ---------------------------------------------------------------------------
# whole-plane kernels (plane.cuh): small spatial extents
# ---------------------------------------------------------------------------

def _plane_cands(layer, n, flags=0):
    from paper_2011_06295_b200 import _abi
    vs = _abi.variants()
    return [c for c in layer.candidates(n, flags) if vs[c[0]]["kind"] == 1]


@pytest.mark.parametrize("c,hw,k,sp,n,dtype", [(512, 2, 512, 0.9, 130, np.float32), (64, 2, 72, 0.9, 33, np.float32),
                                                (512, 4, 512, 0.95, 34, np.float32), (96, 4, 40, 0.8, 70, np.float32),
                                                (64, 2, 64, 0.9, 40, np.float16), (64, 4, 64, 0.9, 40, np.float16)])
def test_plane_kernels_bitwise(sc, orc, c, hw, k, sp, n, dtype):
    import torch
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, sp), seed=0).astype(dtype)
    x, b = bench_inputs(sh, n)
    x = x.astype(dtype)
    bq = b.astype(dtype) if dtype == np.float16 else b
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, bq)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, dtype)
    cands = _plane_cands(layer, n)
    assert cands, "no plane variant"
    for cfg in cands[:: max(1, len(cands) // 40)]:
        o = sc.conv_sparse(xd, kern, bq, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    # fused ReLU + 2x2 max-pool epilogue
    want = relu_pool_ref(ref)
    flags = 0x1 | 0x4
    for cfg in _plane_cands(layer, n, flags)[:6]:
        o = sc.conv_sparse(xd, kern, bq, sc.EnginePlan(launch=cfg), relu=True, pool=True).cpu().numpy()
        assert beq(o, want.astype(dtype)), cfg


# ---------------------------------------------------------------------------
# dispatch-free direct kernels (direct.cuh)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("c,hw,k,sp,n", [(64, 32, 64, 0.9, 3), (64, 16, 72, 0.9, 5), (256, 8, 256, 0.9, 9),
                                         (96, 8, 40, 0.5, 7), (512, 4, 512, 0.95, 17), (3, 32, 64, 0.9, 2),
                                         (64, 2, 72, 0.8, 33), (40, 4, 24, 0.6, 11)])
def test_direct_kernels_bitwise(sc, orc, c, hw, k, sp, n):
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, sp), seed=0)
    x, b = bench_inputs(sh, n)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, np.float32)
    vs = _abi.variants()
    cands = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 2]
    assert cands, "no direct variant"
    ws = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 4]
    assert ws or hw < 8, "no warp-specialised variant"
    tm = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 5]
    assert tm or hw not in (32, 16, 8, 4), "no TMEM-operand variant"
    for cfg in cands[:: max(1, len(cands) // 30)] + ws[:: max(1, len(ws) // 20)] + tm:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    want = relu_pool_ref(ref)
    pc = [cf for cf in layer.candidates(n, 0x5) if vs[cf[0]]["kind"] in (2, 4, 5)]
    for cfg in pc[:: max(1, len(pc) // 8)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg), relu=True, pool=True).cpu().numpy()
        assert beq(o, want), cfg


@pytest.mark.parametrize("c,h,w,k,r,pad,sp,n", [(64, 56, 56, 64, 3, 1, 0.9, 2), (32, 40, 36, 24, 3, 1, 0.7, 3),
                                                 (48, 28, 100, 40, 1, 0, 0.9, 2), (16, 20, 68, 16, 5, 2, 0.8, 2),
                                                 (3, 64, 64, 16, 3, 1, 0.5, 1), (64, 28, 28, 64, 3, 1, 0.9, 3),
                                                 (40, 14, 14, 48, 3, 1, 0.8, 5), (32, 7, 7, 40, 3, 1, 0.8, 9),
                                                 (96, 14, 14, 64, 1, 0, 0.875, 4), (64, 7, 7, 48, 1, 0, 0.9, 6),
                                                 (512, 2, 2, 512, 3, 1, 0.9, 37), (256, 4, 4, 96, 3, 1, 0.9, 19),
                                                 (64, 3, 3, 40, 3, 1, 0.6, 21)])
def test_wide_direct_kernels_bitwise(sc, orc, c, h, w, k, r, pad, sp, n):
    """Direct kernel on column tiles (DISPATCH_WIDE): output rows wider than
    32 or of no tile width (28, 14, 7; 8- and 4-byte row copies), the
    reference's ImageNet-size presets (pkg/src/sparseconv/bench.py:74-102)."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=h, w=w, k=k, r=r, s=r, padding=pad)
    wt = make_layer_weights(LayerSpec("l", sh, sp), seed=1)
    x, b = bench_inputs(sh, n)
    kern = sc.build_csr(wt, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, r, r, 1, pad, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, np.float32)
    vs = _abi.variants()
    cands = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 2 and vs[cf[0]]["dispatch"] == 2]
    assert cands, "no wide direct variant"
    for cfg in cands[:: max(1, len(cands) // 24)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    # the default launch picks a wide direct variant too
    o = sc.conv_sparse(xd, kern, b).cpu().numpy()
    assert beq(o, ref)
    if sh.e % 2 == 0 and sh.f % 2 == 0:
        want = relu_pool_ref(ref)
        pc = [cf for cf in layer.candidates(n, 0x5) if vs[cf[0]]["kind"] == 2 and vs[cf[0]]["dispatch"] == 2]
        assert pc
        for cfg in pc[:: max(1, len(pc) // 6)]:
            o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg), relu=True, pool=True).cpu().numpy()
            assert beq(o, want), cfg


@pytest.mark.parametrize("c,w,k,s,sp,n", [(64, 300, 100, 2, 0.77, 5), (64, 300, 100, 3, 0.875, 3),
                                          (16, 37, 24, 5, 0.5, 7), (8, 1030, 12, 4, 0.6, 2)])
def test_oned_direct_kernels_bitwise(sc, orc, c, w, k, s, sp, n):
    """1D direct kernel (DISPATCH_ONED, H = R = 1): the reference's
    conv_sparse_1d (sc/engine.py:90-106) on the cnn-non-static presets
    (pkg/src/sparseconv/bench.py:94-101) plus odd widths (4-byte row copies)."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=1, w=w, k=k, r=1, s=s)
    wt = make_layer_weights(LayerSpec("l", sh, sp), seed=2)
    x, b = bench_inputs(sh, n)
    kern = sc.build_csr(wt, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 1, s, 1, 0, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, np.float32)
    vs = _abi.variants()
    cands = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 2 and vs[cf[0]]["dispatch"] == 3]
    assert cands, "no 1D direct variant"
    for cfg in cands[:: max(1, len(cands) // 24)]:
        o = sc.conv_sparse_1d(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    o = sc.conv_sparse_1d(xd, kern, b).cpu().numpy()
    assert beq(o, ref)
    o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cands[0]), relu=True).cpu().numpy()
    assert beq(o, np.maximum(ref, 0))


@pytest.mark.parametrize("dt", [np.float32, np.float16])
@pytest.mark.parametrize("c,hw,k,sp,n", [(512, 4, 512, 0.9, 40), (96, 4, 40, 0.5, 7), (512, 2, 512, 0.9, 70),
                                         (64, 2, 72, 0.8, 33), (24, 4, 16, 0.9, 3)])
def test_image_lane_kernels_bitwise(sc, orc, c, hw, k, sp, n, dt):
    """Image-lane kernel, f32 exact and f16 storage (FHFMA, one final round)."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, sp), seed=0).astype(dt)
    x, b = bench_inputs(sh, n)
    x, b = x.astype(dt), b.astype(dt)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, dt)
    vs = _abi.variants()
    cands = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 3]
    assert cands, "no image-lane variant"
    for cfg in cands[:: max(1, len(cands) // 30)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    want = relu_pool_ref(ref)
    pc = [cf for cf in layer.candidates(n, 0x5) if vs[cf[0]]["kind"] == 3]
    for cfg in pc[:: max(1, len(pc) // 6)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg), relu=True, pool=True).cpu().numpy()
        assert beq(o, want.astype(dt)), cfg


@pytest.mark.parametrize("c,hw,k,sp,n", [(64, 32, 64, 0.9, 3), (64, 16, 72, 0.9, 5), (256, 8, 256, 0.9, 9),
                                         (96, 8, 40, 0.5, 7), (512, 4, 512, 0.9, 37), (48, 4, 40, 0.6, 19)])
def test_direct_f16_kernels_bitwise(sc, orc, c, hw, k, sp, n):
    """f16 storage, f32 accumulation with FHFMA: bit-identical to the reference's
    f16 profile (f32 compute, one final round to f16)."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, sp), seed=0).astype(np.float16)
    x, b = bench_inputs(sh, n)
    x, b = x.astype(np.float16), b.astype(np.float16)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, np.float16)
    vs = _abi.variants()
    cands = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] == 2]
    assert cands, "no f16 direct variant"
    vx1 = [cf for cf in cands if vs[cf[0]]["nbt"] == 1]  # one half per lane, no shifted copy
    assert vx1 or hw not in (32, 16, 8), "no f16 VX=1 variant"
    for cfg in cands[:: max(1, len(cands) // 20)] + vx1[:: max(1, len(vx1) // 10)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    want = relu_pool_ref(ref)
    pc = [cf for cf in layer.candidates(n, 0x5) if vs[cf[0]]["kind"] == 2]
    for cfg in pc[:: max(1, len(pc) // 6)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg), relu=True, pool=True).cpu().numpy()
        assert beq(o, want.astype(np.float16)), cfg


@pytest.mark.parametrize("c,hw,k,n", [(32, 16, 24, 5), (64, 8, 40, 9), (48, 4, 32, 33)])
def test_ragged_csr_all_kinds_bitwise(sc, orc, c, hw, k, n):
    """Non-unified CSR (build_csr(unify=False), csr.py:120-126): per-channel nnz
    differ; every kernel kind walks its own row (rowptr) and stays bitwise."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    rng = np.random.default_rng(11)
    w = random_sparse_weights(rng, k, c, 3, 3, 0.85)
    x = rng.standard_normal((n, c, hw, hw)).astype(np.float32)
    b = rng.standard_normal(k).astype(np.float32)
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    kern = sc.build_csr(w, sh, unify=False)
    assert not kern.unified and len(set(np.diff(kern.rowptr))) > 1
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, np.float32)
    vs = _abi.variants()
    cands = layer.candidates(n)
    seen = set()
    for cfg in cands:
        kind = vs[cfg[0]]["kind"]
        if kind in seen and len(seen) < 4:
            continue
        seen.add(kind)
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    assert seen >= ({0, 2} if hw >= 8 else {1, 3})


def test_builtin_launch_table_used_and_exact(sc, orc):
    """conv_sparse on a VGG-CIFAR geometry without in-process tuning takes the
    shipped B200 launch table (engine._builtin) and stays bitwise."""
    import torch
    from paper_2011_06295_b200 import engine
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import bench_inputs, make_layer_weights, vgg16_cifar
    spec = [s for s, _ in vgg16_cifar(0.95) if s.name == "conv3_2"][0]  # other sparsity: table is L-free
    sh = spec.shape.with_batch(20)
    w = make_layer_weights(spec, 3)
    x, b = bench_inputs(sh, 20)
    kern = sc.build_csr(w, sh)
    layer = device_layer(kern, 0, np.float32)
    flags = engine._flags(sc.EnginePlan(), True, False, False)
    engine.TUNED.pop((layer.signature(), 20, flags), None)
    chosen = engine._choose_launch(layer, 20, flags, sc.EnginePlan())
    assert chosen == engine._builtin()[engine._builtin_key(layer.signature(), flags)]
    got = sc.conv_sparse(torch.from_numpy(x).cuda(), kern, b, relu=True).cpu().numpy()
    ref = np.maximum(orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, sh.k, 3, 3, 1, 1, b), 0)
    assert beq(got, ref)


# ---------------------------------------------------------------------------
# activation fake-quant (quantize.py:332-338): standalone pass and fused epilogues
# ---------------------------------------------------------------------------

def test_fake_quant_kernel_bitwise(sc):
    import torch
    from paper_2011_06295_b200 import _abi
    z = np.load(GOLDEN / "fake_quant_cases.npz")
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta):
        y = torch.from_numpy(z[f"x{i}"].copy()).cuda()
        _abi.fake_quant(z[f"x{i}"].dtype, y.data_ptr(), y.numel(), m["params"],
                        torch.cuda.current_stream().cuda_stream)
        assert beq(y.cpu().numpy(), z[f"y{i}"]), (i, m)


@pytest.mark.parametrize("dt", [np.float32, np.float16])
@pytest.mark.parametrize("c,hw,k,n", [(64, 16, 48, 5), (128, 4, 96, 19), (96, 2, 64, 33), (32, 40, 24, 2)])
def test_fused_act_quant_all_kinds_bitwise(sc, orc, c, hw, k, n, dt):
    """conv -> ReLU -> fake-quant (-> pool) through every launch kind: fused in the
    direct / image-lane epilogues, a separate pass after the others."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import DeviceLayer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    aq = {"bits": 8, "clip_lo": 0.0, "clip_hi": 6.0, "mu": 0.0, "step": 6.0 / 255, "mode": "asymmetric"}
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, 0.85), seed=3).astype(dt)
    x, b = bench_inputs(sh, n)
    x, b = x.astype(dt), b.astype(dt)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    want = orc.fake_quant(np.maximum(ref, 0), aq)
    wantp = orc.fake_quant(torch.nn.functional.max_pool2d(
        torch.from_numpy(np.maximum(ref, 0).astype(np.float32)), 2).numpy().astype(dt), aq) if hw % 2 == 0 else None
    layer = DeviceLayer(kern, 0, dt)
    layer.set_act_quant(aq)
    xd = torch.from_numpy(x).cuda()
    bd = torch.from_numpy(b.astype(np.float32)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    vs = _abi.variants()
    for flags, exp in ((_abi.FLAG_RELU | _abi.FLAG_ACT_QUANT, want),
                       (_abi.FLAG_RELU | _abi.FLAG_POOL2 | _abi.FLAG_ACT_QUANT, wantp)):
        if exp is None:
            continue
        cands = layer.candidates(n, flags)
        by_kind = {}
        for cf in cands:
            by_kind.setdefault(vs[cf[0]]["kind"], []).append(cf)
        picks = [cf for lst in by_kind.values() for cf in lst[:: max(1, len(lst) // 4)]]
        if not flags & _abi.FLAG_POOL2:
            picks.append(None)  # generic kernel + fake-quant pass
        for cf in picks:
            y = torch.empty(exp.shape, dtype=xd.dtype, device="cuda")
            layer.launch(xd.data_ptr(), bd.data_ptr(), y.data_ptr(), n,
                         flags | (_abi.FLAG_GENERIC if cf is None else 0), cf, st)
            assert beq(y.cpu().numpy(), exp), (cf, flags)
    # the flag without an attached quantizer is refused
    layer.set_act_quant(None)
    with pytest.raises(Exception):
        layer.launch(xd.data_ptr(), bd.data_ptr(), xd.data_ptr(), n, _abi.FLAG_ACT_QUANT, None, st)


# ---------------------------------------------------------------------------
# API hygiene (VERDICT r1 "what's weak" 7-10)
# ---------------------------------------------------------------------------

def test_launch_requires_prepare_and_never_allocates(sc):
    """scb_conv_sparse of a tiled launch whose tables were not built by
    scb_layer_prepare fails (SCB_ERR_ARG) instead of allocating; after prepare it runs,
    also inside a CUDA graph capture."""
    import ctypes

    import torch
    from oracle import oracle as orc
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import DeviceLayer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=32, c=256, h=8, w=8, k=256, r=3, s=3, padding=1)
    kern = sc.build_csr(make_layer_weights(LayerSpec("c3", sh, 0.9), 0), sh)
    x, b = bench_inputs(sh, 32)
    layer = DeviceLayer(kern, 0, np.float32)  # fresh handle: nothing prepared
    cfg = layer.default_launch(32, 0)
    assert cfg[0] >= 0 and layer.launch_ok(32, 0, cfg)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    y = torch.empty((32, 256, 8, 8), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    lib = _abi.lib()
    args = (ctypes.c_void_p(layer.handle), ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(bd.data_ptr()),
            ctypes.c_void_p(y.data_ptr()), 32, 0, ctypes.byref(_abi.Launch.from_tuple(cfg)), ctypes.c_void_p(st))
    assert lib.scb_conv_sparse(*args) == _abi.SCB_ERR_ARG
    assert "prepare" in _abi.last_error()
    layer.prepare(32, 0, cfg)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        lib.scb_conv_sparse(*args[:7], ctypes.c_void_p(s.cuda_stream))  # warm-up outside capture
        with torch.cuda.graph(g, stream=s):
            assert lib.scb_conv_sparse(*args[:7], ctypes.c_void_p(s.cuda_stream)) == 0
    torch.cuda.current_stream().wait_stream(s)
    y.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    want = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 256, 3, 3, 1, 1, b)
    assert beq(y.cpu().numpy(), want)


@pytest.mark.parametrize("sparsity", [0.0, 0.5])
def test_dense_vgg_shapes_fall_back_from_table(sc, sparsity):
    """the shipped table is keyed on geometry; at low sparsity its launch can
    overflow shared memory -- conv_sparse falls back to a valid launch, bitwise."""
    import torch
    from oracle import oracle as orc
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    for c, hw, k in ((512, 2, 512), (512, 4, 512), (256, 8, 256)):
        sh = sc.ConvShape(n=16, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
        kern = sc.build_csr(make_layer_weights(LayerSpec("d", sh, sparsity), 0), sh)
        x, b = bench_inputs(sh, 16)
        got = sc.conv_sparse(torch.from_numpy(x).cuda(), kern, b, relu=True).cpu().numpy()
        want = np.maximum(orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b), 0)
        assert beq(got, want), (c, hw, sparsity)


def test_out_buffer_validated_and_misaligned_input(sc):
    """a caller `out` of the wrong shape / dtype / layout raises ShapeError
    (no out-of-bounds device writes); a misaligned input view still computes."""
    import torch
    from oracle import oracle as orc
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=9, c=64, h=16, w=16, k=32, r=3, s=3, padding=1)
    kern = sc.build_csr(make_layer_weights(LayerSpec("o", sh, 0.9), 0), sh)
    x, b = bench_inputs(sh, 9)
    xd = torch.from_numpy(x).cuda()
    for bad in (torch.empty((9, 32, 16, 15), device="cuda"), torch.empty((9, 32, 16, 16), device="cuda",
                dtype=torch.float16), torch.empty((9, 32, 16, 32), device="cuda")[..., ::2],
                torch.empty((9, 32, 16, 16)), np.empty((9, 32, 16, 16), np.float32)):
        with pytest.raises(sc.ShapeError):
            sc.conv_sparse(xd, kern, b, out=bad)
    good = torch.empty((9, 32, 16, 16), device="cuda")
    sc.conv_sparse(xd, kern, b, out=good)
    want = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 32, 3, 3, 1, 1, b)
    assert beq(good.cpu().numpy(), want)
    # images 1..8 as a view whose base is 64*16*16*4 bytes (+ an odd offset) into the buffer
    big = torch.empty(9 * 64 * 256 + 1, device="cuda")
    view = big[1:].view(9, 64, 16, 16)
    view.copy_(xd)
    assert view.data_ptr() % 16
    got = sc.conv_sparse(view[1:], kern, b).cpu().numpy()
    assert beq(got, want[1:])


@pytest.mark.parametrize("fmt", ["native", "cb4", "lin16", "aff16"])
def test_f16_compact_taps_in_register_decode(sc, fmt):
    """f16 direct / image-lane kernels read 4-byte taps (16-bit stage offset + f16 value
    or quantizer code) and decode the weight in registers; bitwise vs the oracle on the
    reference quantizer's outputs for every matching variant."""
    import torch
    from oracle import oracle as orc
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import (LayerSpec, affine_quantize, bench_inputs, f16_scaled,
                                             make_layer_weights, reference_quantize)
    from dataclasses import replace
    vs = _abi.variants()
    for c, hw, k, n in ((64, 32, 64, 3), (128, 8, 64, 40), (256, 4, 96, 33), (128, 2, 64, 70)):
        sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
        kern = sc.build_csr(f16_scaled(make_layer_weights(LayerSpec("q", sh, 0.9), 0)), sh)
        if fmt == "cb4":  # 16 centers spread over the values: the codebook decode path
            cents = np.quantile(kern.values.astype(np.float64), np.linspace(0.02, 0.98, 16))
            kern = replace(kern, values=reference_quantize(kern.values, "codebook", cents), _device_cache={})
        elif fmt == "lin16":
            kern = replace(kern, values=reference_quantize(kern.values, "fixed"), _device_cache={})
        elif fmt == "aff16":
            vals, step = affine_quantize(kern.values, 16)
            kern = replace(kern, values=vals, _device_cache={}, quant={"scheme": "affine", "step": step})
        x, b = bench_inputs(sh, n)
        x, b = x.astype(np.float16), b.astype(np.float16)
        want = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
        layer = device_layer(kern, 0, np.float16, fmt)
        cands = [cf for cf in layer.candidates(n) if vs[cf[0]]["kind"] in (2, 3)]
        assert cands, (fmt, hw)
        assert all(vs[cf[0]]["wf"] == {"native": 1, "cb4": 2, "lin16": 3, "aff16": 4}[fmt] for cf in cands)
        assert layer.weight_bytes(cands[0][0]) == 4 * kern.values.size + 4 * (k + 1)
        xd = torch.from_numpy(x).cuda()
        for cfg in cands[:: max(1, len(cands) // 8)]:
            o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg, weight_format=fmt)).cpu().numpy()
            assert beq(o, want), (fmt, hw, cfg)
