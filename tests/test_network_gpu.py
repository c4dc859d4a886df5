"""SparseConvNet (Model.forward's conv loop on the GPU, store.py:263-286) vs
the CPU oracle run layer by layer: conv_sparse -> ReLU -> 2x2 max-pool.
Exact fp32 mode must be bit-identical, for tuned tiled launches, the generic
kernel (+ separate pool kernel) and CUDA-graph replay."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def oracle_stack(net, x):
    from oracle import oracle as orc
    a = x
    for L in net.layers:
        sh = L.kernel.shape
        z = orc.conv_sparse(a, L.kernel.values, L.kernel.colidx, L.kernel.rowptr, sh.k, sh.r, sh.s,
                            sh.stride, sh.padding, L.bias)
        a = np.maximum(z, 0) if L.relu else z
        if L.pool:
            n, k, e, f = a.shape
            a = a.reshape(n, k, e // 2, 2, f // 2, 2).max(axis=(3, 5))
    return a


@pytest.fixture(scope="module")
def vgg_small(torch):
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import vgg16_cifar
    net = build_net(vgg16_cifar(0.9), seed=0)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 3, 32, 32)).astype(np.float32)
    return net, x, oracle_stack(net, x)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def test_tuned_stack_bitwise(torch, vgg_small):
    net, x, ref = vgg_small
    net.plan(3, tune=True, repetitions=1, warmups=0, max_candidates=12)
    out = net.forward(x)
    assert out.shape == ref.shape == (3, 512, 1, 1)
    assert np.array_equal(_bits(out), _bits(ref))


def test_generic_stack_bitwise(torch, vgg_small):
    net, x, ref = vgg_small
    net.plan(3, tune=False)
    net.set_launches([None] * len(net.layers))  # generic kernel + separate max-pool kernel
    assert net.kernels_per_step() == len(net.layers) + sum(L.pool for L in net.layers)
    out = net.forward(x)
    assert np.array_equal(_bits(out), _bits(ref))


def test_graph_replay_bitwise(torch, vgg_small):
    net, x, ref = vgg_small
    net.plan(3, tune=False)
    net.capture()
    out = net.forward(x)
    assert np.array_equal(_bits(out), _bits(ref))
    x2 = np.random.default_rng(6).standard_normal(x.shape).astype(np.float32)
    out2 = net.forward(x2)  # replay reads the refreshed input buffer
    assert np.array_equal(_bits(out2), _bits(oracle_stack(net, x2)))


def test_alexnet_stack_5x5(torch):
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import alexnet_cifar
    net = build_net(alexnet_cifar(0.9), seed=0)
    x = np.random.default_rng(2).standard_normal((2, 3, 32, 32)).astype(np.float32)
    net.plan(2, tune=False)
    out = net.forward(x)
    assert np.array_equal(_bits(out), _bits(oracle_stack(net, x)))


def test_generic_pool_through_conv_sparse(torch):
    """conv_sparse(pool=True) with the generic kernel chosen (launch None in
    the tuner cache) goes through scb_maxpool2."""
    import paper_2011_06295_b200 as sc
    from paper_2011_06295_b200 import engine
    from paper_2011_06295_b200.device import device_layer
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=4, c=64, h=4, w=4, k=64, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("l", sh, 0.9), 0)
    x, b = bench_inputs(sh, 4)
    kern = sc.build_csr(w, sh)
    layer = device_layer(kern, 0, np.float32)
    flags = engine._flags(sc.EnginePlan(), True, True, False)
    engine.TUNED[(layer.signature(), 4, flags)] = None
    try:
        got = sc.conv_sparse(x, kern, b, relu=True, pool=True)
    finally:
        engine.TUNED.pop((layer.signature(), 4, flags), None)
    want = sc.conv_sparse(torch.from_numpy(x).cuda(), kern, b, relu=True, pool=True).cpu().numpy()
    assert np.array_equal(_bits(got), _bits(want))


def test_configure_network_and_apply(torch, vgg_small):
    """configure_network (bench.py:306-342 semantics) times sparse vs dense per
    layer; an applied config mixing both stays within the reference tolerance,
    an all-sparse config stays bitwise."""
    import paper_2011_06295_b200 as sc
    net, x, ref = vgg_small
    net.plan(3, tune=False)
    cfg = sc.configure_network(net, repetitions=2, warmups=1)
    assert set(cfg.choices) == {L.name for L in net.layers}
    for ch in cfg.choices.values():
        assert ch["algorithm"] in ("sparse-direct", "dense-cudnn")
        assert set(ch["median_ms"]) == {"sparse-direct", "dense-cudnn"}
    back = sc.NetworkConfig.from_json(cfg.to_json())
    assert back.choices == cfg.choices
    mixed = sc.NetworkConfig(batch=3, choices={L.name: {"algorithm": "dense-cudnn" if i % 2 else "sparse-direct"}
                                              for i, L in enumerate(net.layers)})
    net.apply_config(mixed)
    out = net.forward(x)
    # dense cuDNN sums in its own order: 13 layers of N(0,1) weights amplify
    # per-layer rounding, so compare globally (relative L2) rather than per element
    assert np.linalg.norm(out.astype(np.float64) - ref) <= 1e-4 * np.linalg.norm(ref.astype(np.float64))
    net.apply_config(sc.NetworkConfig(batch=3, choices={}))
    assert np.array_equal(_bits(net.forward(x)), _bits(ref))


def test_forward_stream_bitwise(torch, vgg_small):
    """Streaming host->device->host inference (copies overlapped) equals the
    oracle for every batch."""
    net, x, ref = vgg_small
    net.plan(3, tune=False)
    x2 = np.random.default_rng(9).standard_normal(x.shape).astype(np.float32)
    ref2 = oracle_stack(net, x2)
    xs = [torch.from_numpy(a).pin_memory() for a in (x, x2, x, x2, x)]
    outs = [torch.empty((3, 512, 1, 1)).pin_memory() for _ in xs]
    net.forward_stream(xs, outs)
    for i, o in enumerate(outs):
        assert np.array_equal(_bits(o.numpy()), _bits(ref if i % 2 == 0 else ref2)), i


@pytest.mark.parametrize("chains", [2, 3])
def test_subbatch_chains_bitwise(torch, vgg_small, chains):
    """Sub-batch chains on separate streams (set_chains): same bits as one
    stream, eager, graph-replayed and streamed."""
    net, x, ref = vgg_small
    net.plan(3, tune=False)
    net.set_chains(chains)
    try:
        assert np.array_equal(_bits(net.forward(x)), _bits(ref))
        net.capture()
        x2 = np.random.default_rng(11).standard_normal(x.shape).astype(np.float32)
        assert np.array_equal(_bits(net.forward(x2)), _bits(oracle_stack(net, x2)))
        xs = [torch.from_numpy(a).pin_memory() for a in (x, x2, x)]
        outs = [torch.empty((3, 512, 1, 1)).pin_memory() for _ in xs]
        net.forward_stream(xs, outs)
        for i, o in enumerate(outs):
            assert np.array_equal(_bits(o.numpy()), _bits(ref if i % 2 == 0 else oracle_stack(net, x2))), i
    finally:
        net.set_chains(1)


# ---------------------------------------------------------------------------
# The exact configurations bench.py times ("pin every timed
# configuration to the oracle"): full batches, shipped launch table, sub-batch
# chains and PDL as in the timed step.
# ---------------------------------------------------------------------------

def _bits16(a):
    return np.ascontiguousarray(a).view(np.uint16)


@pytest.mark.parametrize("sparsity,chains", [(0.9, 2), (0.9, 1), (0.95, 2)])
def test_config3_vgg_batch256_timed_mode_bitwise(torch, sparsity, chains):
    """BASELINE config 3: VGG-16/CIFAR, 256 images, the shipped (tuned-on-B200) launch
    table, `chains` sub-batch chains on separate streams, PDL -- vs the oracle."""
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import vgg16_cifar
    net = build_net(vgg16_cifar(sparsity), seed=0)
    net.plan(256, tune=False)
    net.set_chains(chains)
    net.pdl = True
    x = np.random.default_rng(11).standard_normal((256, 3, 32, 32)).astype(np.float32)
    got = net.forward_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(_bits(got), _bits(oracle_stack(net, x)))


@pytest.mark.parametrize("fmt", ["native", "cb4", "lin16", "aff16"])
def test_config4_vgg_f16_batch256_bitwise(torch, fmt):
    """BASELINE config 4: the same stack with f16 activations and weights -- plain f16,
    the REFERENCE's codebook:16 weights as 4-bit codes (cb4) and its fixed:16 weights as
    int16 codes (lin16), restated bit-exactly (synth.reference_quantize, pinned by
    tests/golden/quant_vgg.json) -- batch 256, in-kernel decode + FHFMA, vs the oracle."""
    from pathlib import Path
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import f16_scaled, reference_quantized_values_fn, vgg16_cifar
    fixture = Path(__file__).resolve().parent / "golden" / "quant_vgg.json"
    fn = {"native": None, "cb4": reference_quantized_values_fn("codebook", fixture),
          "lin16": reference_quantized_values_fn("fixed", fixture),
          "aff16": reference_quantized_values_fn("affine", fixture)}[fmt]
    net = build_net(vgg16_cifar(0.9), seed=0, dtype=np.float16, weight_format=fmt, weight_fn=f16_scaled,
                    values_fn=fn)
    net.plan(256, tune=False)
    x = np.random.default_rng(12).standard_normal((256, 3, 32, 32)).astype(np.float16)
    got = net.forward_device(torch.from_numpy(x).cuda()).cpu().numpy()
    want = oracle_stack(net, x)
    assert np.isfinite(want).all()  # the scaled f16 stack stays in range
    assert np.array_equal(_bits16(got), _bits16(want))


def test_config2_alexnet_batch128_bitwise(torch):
    """BASELINE config 2: AlexNet-style CIFAR stack (5x5 and 3x3), batch 128."""
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import alexnet_cifar
    net = build_net(alexnet_cifar(0.9), seed=0)
    net.plan(128, tune=False)
    x = np.random.default_rng(13).standard_normal((128, 3, 32, 32)).astype(np.float32)
    got = net.forward_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(_bits(got), _bits(oracle_stack(net, x)))


@pytest.mark.parametrize("sparsity", [0.9, 0.95, 0.99])
@pytest.mark.parametrize("dt", [np.float32, np.float16])
def test_config5_sweep_points_batch512_bitwise(torch, sparsity, dt):
    """BASELINE config 5 sweep points: 256->256 3x3 @32x32, batch 512, the launch the
    sweep times (shipped table / heuristic) -- vs the oracle."""
    import paper_2011_06295_b200 as sc
    from oracle import oracle as orc
    from paper_2011_06295_b200.synth import LayerSpec, bench_inputs, make_layer_weights
    sh = sc.ConvShape(n=512, c=256, h=32, w=32, k=256, r=3, s=3, padding=1)
    w = make_layer_weights(LayerSpec("sweep", sh, sparsity), seed=0).astype(dt)
    x, b = bench_inputs(sh, 512)
    x = x.astype(dt)
    kern = sc.build_csr(w, sh)
    got = sc.conv_sparse(torch.from_numpy(x).cuda(), kern, b).cpu().numpy()
    want = orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, 256, 3, 3, 1, 1, b)
    iv = np.uint16 if dt == np.float16 else np.uint32
    assert np.array_equal(got.view(iv), want.view(iv))


# ---------------------------------------------------------------------------
# batch-sharded runner through the real engine: two ranks on one
# GPU (gloo for the gather), each planning and running its own shard
# ---------------------------------------------------------------------------

def _sharded_worker(rank, world, port, n, q):
    import os
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.runner import BatchShardedRunner, shard_range
    from paper_2011_06295_b200.synth import vgg16_cifar
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        a, b = shard_range(n, world, rank)
        net = build_net(vgg16_cifar(0.9), seed=0, device=0)
        net.plan(b - a, tune=False)
        net.set_chains(2 if b - a >= 2 else 1)
        x = torch.from_numpy(np.random.default_rng(21).standard_normal((n, 3, 32, 32)).astype(np.float32))
        out = BatchShardedRunner(lambda xs: net.forward_device(xs.cuda())).run(x, n=n)
        if rank == 0:
            q.put(out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [64, 37])
def test_batch_sharded_runner_two_ranks_bitwise(torch, n):
    import socket

    import torch.multiprocessing as mp
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import vgg16_cifar
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    x = np.random.default_rng(21).standard_normal((n, 3, 32, 32)).astype(np.float32)
    want = oracle_stack(build_net(vgg16_cifar(0.9), seed=0), x)
    assert got.shape == want.shape and np.array_equal(_bits(got), _bits(want))
