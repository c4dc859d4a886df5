"""Kind-7 image-lane position-class kernels (csrc/lane.cuh) against the oracle (GPU).

These kernels drop the taps that land in the zero padding (per position class) and
read / write image-minor activations; exactness rests on the -0.0 fix-up of the
epilogue (lane.cuh header).  Everything here is bitwise against the oracle, which
runs every tap like the reference (sc/_kernels.py:73-84)."""
import numpy as np
import pytest

from test_gpu_parity import beq, relu_pool_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sc():
    import paper_2011_06295_b200 as sc
    return sc


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


def _layer(sc, c, hw, k, sp, n, seed=0):
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, sp), seed=seed).astype(np.float32)
    x, b = bench_inputs(sh, n)
    return sh, w, x.astype(np.float32), b.astype(np.float32)


def _lane_cands(layer, n, flags):
    from paper_2011_06295_b200 import _abi
    vs = _abi.variants()
    cands = layer.candidates(n, flags | _abi.FLAG_IMAGE_MINOR)
    assert cands and all(vs[c[0]]["kind"] == 7 for c in cands)
    return cands


@pytest.mark.parametrize("c,hw,k,sp,n", [(512, 4, 512, 0.9, 70), (96, 4, 40, 0.5, 7), (512, 2, 512, 0.9, 70),
                                         (64, 2, 72, 0.8, 33), (24, 4, 16, 0.9, 3), (256, 4, 512, 0.9, 130),
                                         (40, 4, 24, 0.0, 5), (256, 8, 96, 0.9, 45), (40, 8, 24, 0.5, 7),
                                         # 4x4 output tiles (dispatch 4) of 16x16 / 32x32 planes
                                         (64, 16, 48, 0.9, 70), (24, 16, 20, 0.0, 5), (32, 32, 40, 0.9, 33)])
def test_lane_kernels_bitwise(sc, orc, c, hw, k, sp, n):
    """Every sampled kind-7 launch (NB, unroll, warps, stage, ring depth) through the NCHW
    API (engine.run_layer converts to image-minor and back), plain and with ReLU + pool."""
    import torch
    from paper_2011_06295_b200.device import device_layer
    sh, w, x, b = _layer(sc, c, hw, k, sp, n)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    xd = torch.from_numpy(x).cuda()
    layer = device_layer(kern, 0, np.float32)
    cands = _lane_cands(layer, n, 0)
    for cfg in cands[:: max(1, len(cands) // 24)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
    want = relu_pool_ref(ref)
    pc = _lane_cands(layer, n, 0x5)
    for cfg in pc[:: max(1, len(pc) // 6)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg), relu=True, pool=True).cpu().numpy()
        assert beq(o, want), cfg


def test_lane_image_minor_strided_subbatch(sc, orc):
    """Image-minor buffers with a row stride larger than the batch and a sub-batch that
    starts at image 8 (pointer offset, ld = full width) -- how the network runs chains."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    c, hw, k, n, ld, a = 128, 4, 96, 40, 60, 8
    sh, w, x, b = _layer(sc, c, hw, k, 0.9, n)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    layer = device_layer(kern, 0, np.float32)
    cfg = layer.default_launch(n, _abi.FLAG_IMAGE_MINOR)
    assert cfg[0] >= 0
    xm = torch.full((c * hw * hw, ld), float("nan"), device="cuda")
    xm[:, a:a + n] = torch.from_numpy(x.reshape(n, -1).T.copy()).cuda()
    ym = torch.full((k * hw * hw, ld), -7.0, device="cuda")
    bd = torch.from_numpy(b).cuda()
    st = torch.cuda.current_stream().cuda_stream
    layer.launch(xm.data_ptr() + 4 * a, bd.data_ptr(), ym.data_ptr() + 4 * a, n, _abi.FLAG_IMAGE_MINOR, cfg, st,
                 ldx=ld, ldy=ld)
    got = ym[:, a:a + n].T.contiguous().cpu().numpy().reshape(ref.shape)
    assert beq(got, ref)
    # rows outside the sub-batch untouched
    assert torch.all(ym[:, :a] == -7.0) and torch.all(ym[:, a + n:] == -7.0)
    # the layout converters are exact inverses
    back = torch.empty((n, c, hw, hw), device="cuda")
    _abi.from_image_minor(np.float32, xm.data_ptr() + 4 * a, ld, back.data_ptr(), n, c * hw * hw, st)
    assert beq(back.cpu().numpy(), x)
    xm2 = torch.zeros((c * hw * hw, ld), device="cuda")
    _abi.to_image_minor(np.float32, back.data_ptr(), xm2.data_ptr() + 4 * a, n, c * hw * hw, ld, st)
    assert torch.equal(xm2[:, a:a + n], xm[:, a:a + n])


@pytest.mark.parametrize("hw", [2, 4, 8, 16])
def test_lane_negative_zero_fixup(sc, orc, hw):
    """bias -0.0 and an all-zero input: every product is +-0, so the reference result is
    -0.0 exactly when every tap of the output -- padding taps included -- has a negative
    weight, +0.0 otherwise.  The kernel drops the padding taps and must restore the
    reference's sign from the per-class mask."""
    import torch
    from paper_2011_06295_b200.device import device_layer
    c, k, n = 8, 32, 6
    rng = np.random.default_rng(5)
    w = np.zeros((k, c, 3, 3), np.float32)
    for kk in range(k):
        idx = rng.choice(c * 9, size=7, replace=False)
        v = -rng.uniform(0.5, 1.5, size=7).astype(np.float32)
        if kk % 3 == 1:  # one positive tap somewhere (often a padding tap for edge classes)
            v[rng.integers(7)] *= -1
        w.reshape(k, -1)[kk, idx] = v
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    kern = sc.build_csr(w, sh)
    x = np.zeros((n, c, hw, hw), np.float32)
    b = np.full(k, -0.0, np.float32)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    sign = np.signbit(ref)
    assert sign.any() and (~sign).any(), "test needs both zero signs"
    layer = device_layer(kern, 0, np.float32)
    xd = torch.from_numpy(x).cuda()
    for cfg in _lane_cands(layer, n, 0)[::7]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg


def test_lane_nonfinite_weights_not_eligible(sc):
    """v*0 is NaN for an infinite weight, so dropping padding taps would be wrong: such
    layers get no kind-7 launch."""
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    sh, w, x, b = _layer(sc, 16, 4, 8, 0.5, 4)
    w[0].flat[np.flatnonzero(w[0])[0]] = np.inf
    layer = device_layer(sc.build_csr(w, sh), 0, np.float32)
    assert layer.candidates(4, _abi.FLAG_IMAGE_MINOR) == []
    assert layer.default_launch(4, _abi.FLAG_IMAGE_MINOR)[0] < 0


def test_lane_fast_mode_within_tolerance(sc, orc):
    """FFMA variants: within the north-star 1e-5 relative tolerance."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    sh, w, x, b = _layer(sc, 256, 4, 64, 0.9, 33)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 64, 3, 3, 1, 1, b)
    layer = device_layer(kern, 0, np.float32)
    cands = _lane_cands(layer, 33, _abi.FLAG_FAST)
    vs = _abi.variants()
    assert all(vs[c[0]]["mode"] == 1 for c in cands)
    xd = torch.from_numpy(x).cuda()
    for cfg in cands[::9]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg, fast_math=True)).cpu().numpy()
        assert np.all(np.abs(o - ref) <= 1e-5 * (np.abs(ref) + 1)), cfg


def test_lane_fused_act_quant_bitwise(sc, orc):
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import DeviceLayer
    aq = {"bits": 8, "clip_lo": 0.0, "clip_hi": 6.0, "mu": 0.0, "step": 6.0 / 255, "mode": "asymmetric"}
    n = 19
    sh, w, x, b = _layer(sc, 128, 4, 96, 0.85, n, seed=3)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 96, 3, 3, 1, 1, b)
    want = orc.fake_quant(np.maximum(ref, 0), aq)
    wantp = orc.fake_quant(relu_pool_ref(ref), aq)
    from paper_2011_06295_b200 import engine
    layer = DeviceLayer(kern, 0, np.float32)
    layer.set_act_quant(aq)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    for flags, exp in ((_abi.FLAG_RELU | _abi.FLAG_ACT_QUANT, want),
                       (_abi.FLAG_RELU | _abi.FLAG_POOL2 | _abi.FLAG_ACT_QUANT, wantp)):
        for cfg in _lane_cands(layer, n, flags)[::11]:
            y = torch.empty(exp.shape, device="cuda")
            engine.run_layer(layer, xd.data_ptr(), bd.data_ptr(), y, n, flags, cfg,
                             torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert beq(y.cpu().numpy(), exp), (cfg, flags)


@pytest.mark.parametrize("dt", [np.float32, np.float16])
def test_vgg_tail_network_uses_lane_layers_bitwise(sc, orc, dt):
    """conv4_1 .. conv5_3 of VGG-CIFAR (the stack's tail, pools fused) through
    SparseConvNet: the untuned plan runs them on kind-7 launches in image-minor layout
    (one conversion in, one out), 1 and 2 sub-batch chains (the second starts at image 16:
    16-byte TMA alignment in f16) and a CUDA graph replay, bit-identical to the oracle
    layer by layer."""
    import torch
    from paper_2011_06295_b200 import _abi, engine
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import f16_scaled, vgg16_cifar
    specs = vgg16_cifar(0.9)
    tail = [(s, p) for s, p in specs if s.name.startswith(("conv4", "conv5"))]
    n = 24
    net = build_net(tail, seed=0, dtype=dt, weight_fn=f16_scaled if dt == np.float16 else None)
    net.plan(n, tune=False)
    assert all(engine.launch_kind(l) == _abi.KIND_LANE for l in net.launches)
    rng = np.random.default_rng(1)
    x = np.maximum(rng.standard_normal((n, *net.in_shape)), 0).astype(dt)
    cur = x
    for L in net.layers:
        sh = L.kernel.shape
        cur = orc.conv_sparse(cur, L.kernel.values, L.kernel.colidx, L.kernel.rowptr, sh.k, 3, 3, 1, 1, L.bias)
        cur = relu_pool_ref(cur) if L.pool else np.maximum(cur, cur.dtype.type(0))
    xd = torch.from_numpy(x).cuda()
    for chains in (1, 2):
        net.set_chains(chains)
        assert beq(net.forward_device(xd).cpu().numpy(), cur), chains
    net.capture()
    assert beq(net.forward_device(xd).cpu().numpy(), cur)
    assert net.kernels_per_step() == len(tail) + 1  # input conversion; the last layer writes NCHW


@pytest.mark.parametrize("fmt", ["native", "cb4", "lin16", "aff16"])
def test_lane_f16_in_register_decode_bitwise(sc, fmt):
    """f16 storage lane kernels (FHFMA, f16 operands two images per 32-bit load) with every
    f16 weight format decoded in registers: bitwise vs the oracle on the reference
    quantizer's outputs, plain and with ReLU + pool."""
    import torch
    from dataclasses import replace
    from oracle import oracle as orc
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import (LayerSpec, affine_quantize, bench_inputs, f16_scaled,
                                             make_layer_weights, reference_quantize)
    for c, hw, k, n in ((256, 4, 96, 33), (128, 2, 64, 70), (512, 4, 512, 40), (128, 8, 64, 70), (64, 16, 48, 70)):
        sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
        kern = sc.build_csr(f16_scaled(make_layer_weights(LayerSpec("q", sh, 0.9), 0)), sh)
        if fmt == "cb4":
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
        cands = _lane_cands(layer, n, 0)
        xd = torch.from_numpy(x).cuda()
        for cfg in cands[:: max(1, len(cands) // 8)]:
            o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg, weight_format=fmt)).cpu().numpy()
            assert beq(o, want), (fmt, hw, cfg)
        wantp = relu_pool_ref(want)
        for cfg in _lane_cands(layer, n, 0x5)[::7]:
            o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg, weight_format=fmt), relu=True,
                               pool=True).cpu().numpy()
            assert beq(o, wantp), (fmt, hw, cfg)


@pytest.mark.parametrize("hw", [2, 4])
def test_lane_class_split_bitwise(sc, orc, hw):
    """Class-split lane kernels (two warps per output channel, kt = 2): plain, ReLU + pool
    (pooled windows straddle the two warps' classes: exchanged through shared memory) and
    fused fake-quant, bitwise."""
    import torch
    from paper_2011_06295_b200 import _abi, engine
    from paper_2011_06295_b200.device import DeviceLayer
    aq = {"bits": 8, "clip_lo": 0.0, "clip_hi": 6.0, "mu": 0.0, "step": 6.0 / 255, "mode": "asymmetric"}
    n, c, k = 70, 256, 60
    sh, w, x, b = _layer(sc, c, hw, k, 0.9, n, seed=7)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    layer = DeviceLayer(kern, 0, np.float32)
    layer.set_act_quant(aq)
    vs = _abi.variants()
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    st = torch.cuda.current_stream().cuda_stream
    cases = ((0, ref), (_abi.FLAG_RELU | _abi.FLAG_POOL2, relu_pool_ref(ref)),
             (_abi.FLAG_RELU | _abi.FLAG_ACT_QUANT, orc.fake_quant(np.maximum(ref, 0), aq)),
             (_abi.FLAG_RELU | _abi.FLAG_POOL2 | _abi.FLAG_ACT_QUANT, orc.fake_quant(relu_pool_ref(ref), aq)))
    for flags, exp in cases:
        all_c = _lane_cands(layer, n, flags)
        splits = sorted({vs[cf[0]]["kt"] for cf in all_c} - {1})
        assert splits == ([2, 4] if hw == 2 else [2, 3]), splits
        cands = []
        for cs in splits:
            sub = [cf for cf in all_c if vs[cf[0]]["kt"] == cs]
            cands += sub[:: max(1, len(sub) // 4)]
        for cfg in cands:
            y = torch.empty(exp.shape, device="cuda")
            engine.run_layer(layer, xd.data_ptr(), bd.data_ptr(), y, n, flags, cfg, st)
            torch.cuda.synchronize()
            assert beq(y.cpu().numpy(), exp), (cfg, flags)


def test_fused_output_layouts_bitwise(sc, orc):
    """SCB_FLAG_Y_IMAGE_MINOR (a narrow direct kernel writes an image-minor output, with pool)
    and SCB_FLAG_Y_NCHW (a kind-7 kernel writes NCHW): the layout changes at both ends of an
    image-minor run without conversion kernels, bitwise."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    vs = _abi.variants()
    st = torch.cuda.current_stream().cuda_stream
    # direct 8x8 -> image-minor pooled 4x4 output (conv3_3-like), sub-batch at image 8
    n, ld, a = 20, 40, 8
    sh, w, x, b = _layer(sc, 64, 8, 48, 0.9, n)
    kern = sc.build_csr(w, sh)
    ref = relu_pool_ref(orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 48, 3, 3, 1, 1, b))
    layer = device_layer(kern, 0, np.float32)
    fl = _abi.FLAG_RELU | _abi.FLAG_POOL2 | _abi.FLAG_Y_IMAGE_MINOR
    cands = layer.candidates(n, fl)
    assert cands and all(vs[c[0]]["kind"] == 2 and vs[c[0]]["dispatch"] == 0 for c in cands)
    xd, bd = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    for cfg in cands[:: max(1, len(cands) // 8)]:
        ym = torch.full((48 * 16, ld), -3.0, device="cuda")
        layer.launch(xd.data_ptr(), bd.data_ptr(), ym.data_ptr() + 4 * a, n, fl, cfg, st, ldy=ld)
        got = ym[:, a:a + n].T.contiguous().cpu().numpy().reshape(ref.shape)
        assert beq(got, ref), cfg
        assert torch.all(ym[:, :a] == -3.0) and torch.all(ym[:, a + n:] == -3.0)
    # kind 7 on image-minor input -> NCHW output (plain and pooled)
    sh, w, x, b = _layer(sc, 128, 2, 64, 0.9, n)
    kern = sc.build_csr(w, sh)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 64, 3, 3, 1, 1, b)
    layer = device_layer(kern, 0, np.float32)
    xm = torch.zeros((128 * 4, ld), device="cuda")
    xm[:, a:a + n] = torch.from_numpy(x.reshape(n, -1).T.copy()).cuda()
    bd = torch.from_numpy(b).cuda()
    for extra, exp in ((0, ref), (_abi.FLAG_RELU | _abi.FLAG_POOL2, relu_pool_ref(ref))):
        fl = _abi.FLAG_IMAGE_MINOR | _abi.FLAG_Y_NCHW | extra
        cands = layer.candidates(n, fl)
        assert cands
        for cfg in cands[:: max(1, len(cands) // 8)]:
            y = torch.full(exp.shape, -3.0, device="cuda")
            layer.launch(xm.data_ptr() + 4 * a, bd.data_ptr(), y.data_ptr(), n, fl, cfg, st, ldx=ld, ldy=ld)
            assert beq(y.cpu().numpy(), exp), (cfg, extra)


@pytest.mark.parametrize("c,hw,k,n", [(512, 4, 512, 40), (512, 2, 512, 70), (96, 4, 40, 7)])
def test_lane_half2_fast_mode_within_tolerance(sc, orc, c, hw, k, n):
    """The f16 opt-in fast mode (SCB_FLAG_FAST on f16 layers: half2 accumulators, one HFMA2
    per two MACs -- the north star's "half2 FMA"): within the fp16 tolerance 1e-2*(|ref|+1)
    of the reference's f16 profile; without the flag f16 layers never get these kernels."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, f16_scaled, make_layer_weights
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    kern = sc.build_csr(f16_scaled(make_layer_weights(LayerSpec("h", sh, 0.9), 0)), sh)
    x, b = bench_inputs(sh, n)
    x, b = np.maximum(x, 0).astype(np.float16), b.astype(np.float16)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b).astype(np.float64)
    layer = device_layer(kern, 0, np.float16)
    vs = _abi.variants()
    assert not any(vs[cf[0]]["mode"] == 2 for cf in layer.candidates(n, _abi.FLAG_IMAGE_MINOR))
    h2 = [cf for cf in layer.candidates(n, _abi.FLAG_IMAGE_MINOR | _abi.FLAG_FAST) if vs[cf[0]]["mode"] == 2]
    assert h2
    xd = torch.from_numpy(x).cuda()
    for cfg in h2[:: max(1, len(h2) // 6)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg, fast_math=True)).cpu().numpy().astype(np.float64)
        assert np.all(np.abs(o - ref) <= 1e-2 * (np.abs(ref) + 1)), (cfg, float(np.max(np.abs(o - ref))))


def test_layout_flag_misuse_is_refused(sc):
    """The C ABI refuses inconsistent layout requests instead of computing garbage: a row
    stride below the batch, an image-minor input without a kind-7 launch, SCB_FLAG_Y_NCHW
    without an image-minor input, SCB_FLAG_Y_IMAGE_MINOR on a kind-7 or generic launch."""
    import torch
    from paper_2011_06295_b200 import _abi
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.errors import SparseConvError
    n = 16
    sh, w, x, b = _layer(sc, 32, 4, 16, 0.9, n)
    layer = device_layer(sc.build_csr(w, sh), 0, np.float32)
    st = torch.cuda.current_stream().cuda_stream
    buf = torch.zeros(32 * 16 * 64, device="cuda")
    out = torch.zeros(16 * 16 * 64, device="cuda")
    lane = layer.default_launch(n, _abi.FLAG_IMAGE_MINOR)
    nchw = layer.default_launch(n, 0)
    assert lane[0] >= 0 and nchw[0] >= 0
    bad = [(_abi.FLAG_IMAGE_MINOR, lane, dict(ldx=8, ldy=8)),               # ld < n
           (_abi.FLAG_IMAGE_MINOR | _abi.FLAG_GENERIC, None, dict(ldx=n, ldy=n)),  # generic, image-minor
           (_abi.FLAG_Y_NCHW, nchw, dict(ldx=n, ldy=n)),                    # Y_NCHW needs minor x
           (_abi.FLAG_IMAGE_MINOR | _abi.FLAG_Y_IMAGE_MINOR, lane, dict(ldx=n, ldy=n)),
           (_abi.FLAG_Y_IMAGE_MINOR | _abi.FLAG_GENERIC, None, dict(ldx=n, ldy=n))]
    for flags, cfg, ld in bad:
        with pytest.raises(SparseConvError):
            layer.launch(buf.data_ptr(), 0, out.data_ptr(), n, flags, cfg, st, **ld)
            pytest.fail(f"accepted flags {flags:#x} launch {cfg} {ld}")
    torch.cuda.synchronize()  # no sticky error left behind


@pytest.mark.parametrize("hw", [2, 4, 8, 16])
def test_lane_ragged_csr_bitwise(sc, orc, hw):
    """Ragged (non-unified) CSR -- per-channel tap counts differ (csr.py:120-126) -- on the
    kind-7 kernels: per-(channel, stage) slots of different lengths, bitwise."""
    import torch
    from golden_gen import random_sparse_weights
    n, c, k = 21, 48, 40
    rng = np.random.default_rng(9)
    w = random_sparse_weights(rng, k, c, 3, 3, 0.85).astype(np.float32)
    sh = sc.ConvShape(n=n, c=c, h=hw, w=hw, k=k, r=3, s=3, padding=1)
    kern = sc.build_csr(w, sh, unify=False)
    assert not kern.unified and len(set(np.diff(kern.rowptr))) > 1
    x = rng.standard_normal((n, c, hw, hw)).astype(np.float32)
    b = rng.standard_normal(k).astype(np.float32)
    ref = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, k, 3, 3, 1, 1, b)
    from paper_2011_06295_b200.device import device_layer
    layer = device_layer(kern, 0, np.float32)
    xd = torch.from_numpy(x).cuda()
    cands = _lane_cands(layer, n, 0)
    for cfg in cands[:: max(1, len(cands) // 10)]:
        o = sc.conv_sparse(xd, kern, b, sc.EnginePlan(launch=cfg)).cpu().numpy()
        assert beq(o, ref), cfg
