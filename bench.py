#!/usr/bin/env python3
"""Benchmark of the B200 direct sparse convolution engine (BASELINE.json).

Metric: "Sparse conv layer us & achieved HBM GB/s vs sparsity; images/sec at
1-8 GPUs".  One *step* is one forward pass of the 13-layer VGG-16/CIFAR-10
conv stack (BASELINE config 3: 3x3 convs, 90% unified per-channel sparsity,
bias + ReLU fused, 2x2 max-pool fused at the end of each stage) over a batch
of 256 synthetic 32x32 images per GPU, fp32 in the reference's exact
arithmetic (separately rounded multiply and add, bit-identical to the CPU
reference).  ``value`` = images/s of the whole job (weak scaling: every rank
runs its own 256-image batch, no data-path collective).

Per-layer microseconds, achieved FLOP/s and HBM GB/s are reported in
``layers``; ``roofline`` describes the layer kernel with the largest share of
the step.  ``e2e`` runs the same stack through the host-facing call
(SparseConvNet.forward: pinned host batch -> H2D -> 13 kernels -> D2H).
``cpu_baseline`` times the reference algorithm's CPU restatement
(oracle/, C + OpenMP) on a bounded sample of the same workload on this box's
host cores.  ``dense_cudnn`` times torch/cuDNN dense fp32 (IEEE, no TF32)
convolutions of the same stack, the comparator the paper uses.

``--impl reference`` times only the reference's CPU path (the oracle port)
and prints the same metric with ``"impl": "reference"``.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Sparse conv layer µs & achieved HBM GB/s vs sparsity; images/sec at 1–8 GPUs"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--batch", type=int, default=256,
                    help="GLOBAL batch (BASELINE config 3: 256), split into contiguous per-GPU shards")
    ap.add_argument("--no-proxy", action="store_true", help="skip the batch-32 (8-GPU shard) proxy line")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 sparsity sweep summary")
    ap.add_argument("--sparsity", type=float, default=0.9)
    ap.add_argument("--no-tune", action="store_true", help="C heuristic launches instead of the tuner")
    ap.add_argument("--launches", default="", help="JSON of per-layer launches: loaded if present "
                    "(tuner skipped), else written after tuning")
    ap.add_argument("--cpu-images", type=int, default=8, help="images per CPU-baseline sample")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU-baseline time budget")
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="reference arm: time budget of warm-up + timed steps (bounds the per-step sample)")
    ap.add_argument("--chains", type=int, default=2, help="sub-batch chains on separate streams per GPU")
    ap.add_argument("--no-fuse-layouts", action="store_true",
                    help="separate layout-conversion kernels around the image-minor layers")
    ap.add_argument("--graph", type=int, default=0, help="1: replay the stack as one CUDA graph per step")
    ap.add_argument("--no-pdl", action="store_true", help="no programmatic dependent launch between layers")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-f16", action="store_true", help="skip the fp16 (config 4) secondary measurement")
    ap.add_argument("--no-alexnet", action="store_true", help="skip the AlexNet-style (config 2) secondary line")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(sparsity: float):
    from paper_2011_06295_b200.synth import vgg16_cifar
    return vgg16_cifar(sparsity)


def layer_work(spec, L: int, batch: int, pool: bool):
    """Algorithmic FLOPs and bytes of one layer launch:
    FLOPs = 2*N*K*E*F*L (executed MACs incl. unification padding,
    engine.py:131-136); bytes = unpadded input + output (pooled when fused)
    + values + column indices + rowptr + bias, each counted once."""
    sh = spec.shape
    flops = 2 * batch * sh.k * sh.e * sh.f * L
    e, f = (sh.e // 2, sh.f // 2) if pool else (sh.e, sh.f)
    byts = 4 * (batch * sh.c * sh.h * sh.w + batch * sh.k * e * f) + sh.k * L * (4 + 4) + 4 * (sh.k + 1) + 4 * sh.k
    return flops, byts


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md)
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = self.proc.communicate()[0]

    def summary(self):
        rows = []
        for ln in self.out.splitlines():
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append((float(p[1]), float(p[2]), p[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU legs (the oracle: reference algorithm restated in C, OpenMP threads)
# ---------------------------------------------------------------------------

def oracle_forward(x, specs, kernels, biases):
    """The conv stack through the oracle (oracle/oracle.c, the reference's
    conv_sparse_kernel restated, golden-pinned): conv_sparse -> ReLU -> 2x2
    max-pool in the activation dtype, exactly the reference's Model.forward glue
    (store.py:276-284).  Checker / CPU baseline only."""
    from oracle import oracle as orc
    a = x
    for (spec, pool), kern, b in zip(specs, kernels, biases):
        sh = spec.shape
        z = orc.conv_sparse(a, kern.values, kern.colidx, kern.rowptr, sh.k, sh.r, sh.s, sh.stride,
                            sh.padding, b)
        a = np.maximum(z, z.dtype.type(0))
        if pool:
            n, k, e, f = a.shape
            a = a.reshape(n, k, e // 2, 2, f // 2, 2).max(axis=(3, 5))
    return a


def parity_gate(name, got, want):
    """Bit-for-bit gate of a timed configuration against the oracle (the reference
    gates every timed result, bench.py:139-147)."""
    from paper_2011_06295_b200.errors import IntegrityError
    got = np.ascontiguousarray(got)
    if got.shape != want.shape or got.dtype != want.dtype:
        raise IntegrityError(f"{name}: output {got.shape}/{got.dtype} vs oracle {want.shape}/{want.dtype}")
    iv = {2: np.uint16, 4: np.uint32}[want.dtype.itemsize]
    bad = int(np.count_nonzero(got.view(iv) != want.view(iv)))
    if bad:
        raise IntegrityError(f"{name}: {bad} of {want.size} outputs differ from the oracle")
    return {"vs": "oracle (oracle/oracle.c: reference conv_sparse_kernel restated, golden-pinned)",
            "bitwise": True, "outputs": int(want.size)}


def cpu_stack_time(specs, kernels, biases, images: int, budget_s: float, seed: int = 7,
                   steps: int | None = None, warmup: int = 1):
    """Run the reference algorithm over the conv stack on `images` images
    (conv_sparse -> ReLU -> 2x2 max-pool, store.py:276-284): `warmup` untimed
    passes, then exactly `steps` timed passes, or (steps None) passes until
    `budget_s` is spent; returns (seconds per pass, passes, threads)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal((images, specs[0][0].shape.c, 32, 32)).astype(np.float32)

    def one_pass():
        return oracle_forward(x0, specs, kernels, biases)

    for _ in range(max(1, warmup)):
        one_pass()  # warm (threads, page faults)
    t0 = time.perf_counter()
    passes = 0
    while True:
        one_pass()
        passes += 1
        el = time.perf_counter() - t0
        if steps is not None:
            if passes >= steps:
                break
        elif el >= budget_s or passes >= 1000:
            break
    return el / passes, passes, orc.max_threads()


def build_kernels(specs, seed: int = 0):
    import paper_2011_06295_b200 as sc
    from paper_2011_06295_b200.synth import bench_inputs, make_layer_weights
    kernels, biases = [], []
    for spec, _ in specs:
        kernels.append(sc.build_csr(make_layer_weights(spec, seed), spec.shape))
        biases.append(bench_inputs(spec.shape, 1, seed)[1])
    return kernels, biases


def repo_libs_loaded():
    """Shared objects under this repo mapped into the process (evidence of which native code ran)."""
    try:
        maps = Path("/proc/self/maps").read_text()
    except OSError:
        return None
    root = str(ROOT.resolve())
    return sorted({ln.split()[-1][len(root) + 1:] for ln in maps.splitlines()
                   if ln.split() and ln.split()[-1].startswith(root) and ".so" in ln.split()[-1]})


def workload_name(sparsity: float) -> str:
    return (f"VGG-16 CIFAR-10, 13 sparse 3x3 convs at {sparsity:g} unified sparsity, bias+ReLU, "
            "2x2 max-pool per stage, exact fp32 (mul+add)")


# VGG-16/CIFAR conv stack (name, C, H, K, pool) = synth.VGG16_CIFAR_LAYERS, restated here so
# the reference arm imports nothing of this repo
_VGG = [("conv1_1", 3, 32, 64, 0), ("conv1_2", 64, 32, 64, 1), ("conv2_1", 64, 16, 128, 0),
        ("conv2_2", 128, 16, 128, 1), ("conv3_1", 128, 8, 256, 0), ("conv3_2", 256, 8, 256, 0),
        ("conv3_3", 256, 8, 256, 1), ("conv4_1", 256, 4, 512, 0), ("conv4_2", 512, 4, 512, 0),
        ("conv4_3", 512, 4, 512, 1), ("conv5_1", 512, 2, 512, 0), ("conv5_2", 512, 2, 512, 0),
        ("conv5_3", 512, 2, 512, 1)]


def _import_reference():
    """The UNMODIFIED reference package, pip-installed into baseline/_ref (DESIGN.md
    'reference arm'): its numba conv_sparse, build_csr and make_layer_weights."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_sparseconv_ref")
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "sparseconv").is_dir():
        raise ImportError(f"reference not installed at {ref_dir}")
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    import sparseconv
    if not str(Path(sparseconv.__file__).resolve()).startswith(str(ref_dir.resolve())):
        raise ImportError(f"sparseconv resolved to {sparseconv.__file__}, not {ref_dir}")
    return sparseconv


def run_reference(args, rank: int, world: int):
    """The reference's own CPU path for the same workload: sparseconv.conv_sparse (numba,
    sc/engine.py:68-87) with EnginePlan(sub_batch_size=8, worker_count=os.cpu_count()),
    CSR from sparseconv.build_csr, weights from sparseconv.bench.make_layer_weights, the
    Model.forward glue (ReLU, 2x2 max-pool) in numpy.  One step = one pass over
    `images` images of the 256-image batch (all 256 unless the steps would not fit the
    time budget; then a bounded sample, stated in config)."""
    if rank != 0:
        return
    ref = _import_reference()
    import numba
    specs = [(ref.LayerSpec(n, ref.ConvShape(n=1, c=c, h=h, w=h, k=k, r=3, s=3, stride=1, padding=1),
                            args.sparsity), bool(pool)) for n, c, h, k, pool in _VGG]
    kernels, biases = [], []
    for spec, _ in specs:
        kernels.append(ref.build_csr(ref.bench.make_layer_weights(spec, seed=0), spec.shape))
        brng = np.random.default_rng(1)  # = bench inputs: x (1 image) then bias, default_rng(seed+1)
        brng.standard_normal((1, spec.shape.c, spec.shape.h, spec.shape.w))
        biases.append(brng.standard_normal(spec.shape.k).astype(np.float32))
    cores = os.cpu_count() or 1
    plan = ref.EnginePlan(sub_batch_size=8, worker_count=cores)
    x_all = np.random.default_rng(7).standard_normal((args.batch, 3, 32, 32)).astype(np.float32)

    def one_pass(x):
        a = x
        for (spec, pool), kern, b in zip(specs, kernels, biases):
            a = np.maximum(ref.conv_sparse(a, kern, b, plan), 0)
            if pool:
                n, k, e, f = a.shape
                a = a.reshape(n, k, e // 2, 2, f // 2, 2).max(axis=(3, 5))
        return a

    one_pass(x_all[:8])  # numba JIT compile (the reference's own first call), untimed
    t0 = time.perf_counter()
    one_pass(x_all)
    t_full = time.perf_counter() - t0
    images = args.batch
    budget = max(60.0, args.ref_seconds)
    if t_full * (args.steps + args.warmup) > budget:
        images = max(8, int(args.batch * budget / (t_full * (args.steps + args.warmup))) // 8 * 8)
    x = x_all[:images]
    for _ in range(max(0, args.warmup - 1)):
        one_pass(x)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one_pass(x)
        ts.append(time.perf_counter() - t0)
    per_pass = sum(ts) / len(ts)
    ips = images / per_pass
    # second figure: the oracle's C restatement (oracle/, OpenMP) on the same sample, <= 3 passes
    port = None
    try:
        from oracle import oracle as orc
        okern = [orc.build_csr(w, spec.shape.h, spec.shape.w, spec.shape.padding)
                 for (spec, _), w in zip(specs, [ref.bench.make_layer_weights(sp, seed=0) for sp, _ in specs])]

        class _K:  # oracle CSR triple in the attribute form oracle_forward reads
            def __init__(self, t):
                self.values, self.colidx, self.rowptr = t[0], t[1], t[2]
        ospecs = [(type("S", (), {"shape": spec.shape})(), pool) for spec, pool in specs]
        oracle_forward(x, ospecs, [_K(t) for t in okern], biases)
        tp = []
        for _ in range(min(3, args.steps)):
            t0 = time.perf_counter()
            oracle_forward(x, ospecs, [_K(t) for t in okern], biases)
            tp.append(time.perf_counter() - t0)
        port = {"images_per_s": round(images / (sum(tp) / len(tp)), 3), "cores": orc.max_threads(),
                "passes": len(tp), "what": "oracle/oracle.c restatement of conv_sparse_kernel (C, OpenMP)"}
    except Exception as e:  # the port is a secondary figure only
        port = {"unavailable": str(e)[:200]}
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ips, 3), "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per_pass * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: sparseconv.bench.make_layer_weights (reference), N(0,1) activations",
        "config": {"workload": workload_name(args.sparsity), "global_batch": args.batch,
                   "images_per_step": images, "parallelism": "cpu",
                   "normalisation": "images/s = images per step / step time (per-image work identical "
                                    "to the 256-image batch)" if images != args.batch else "full batch per step"},
        "cpu_baseline": {"value": round(ips, 3), "unit": "images/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} passes of the 13-layer stack over {images} images through "
                                   f"the unmodified reference sparseconv.conv_sparse (numba "
                                   f"{numba.__version__}, EnginePlan(sub_batch_size=8, worker_count={cores}))"},
        "e2e": {"value": round(ips, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "port": port,
        "repo_native_libs_loaded": repo_libs_loaded(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------

def fma_peak_tflops(device: int):
    """Measured CUDA-core peaks (scb_fma_peaks): MAC/s per probe -> FLOP/s."""
    import ctypes
    from paper_2011_06295_b200 import _abi
    names = ctypes.create_string_buffer(16 * 8)
    vals = (ctypes.c_double * 8)()
    cnt = ctypes.c_int32()
    _abi.check(_abi.lib().scb_fma_peaks(device, names, vals, 8, ctypes.byref(cnt)))
    return {names.raw[16 * i:16 * i + 16].split(b"\0")[0].decode(): 2 * vals[i] / 1e12 for i in range(cnt.value)}


def integrity_gate(net, x_dev):
    """Every tuned layer launch must agree bit for bit with the independent
    generic kernel on the benchmark input (the reference gates every timed
    result, bench.py:139-147)."""
    import torch
    from paper_2011_06295_b200 import engine
    from paper_2011_06295_b200.errors import IntegrityError
    cur = x_dev
    stream = torch.cuda.current_stream().cuda_stream
    for i, L in enumerate(net.layers):
        got = torch.empty(net.out_shape(i, net.batch), dtype=net.tdtype, device=net.tdev)
        net.launch_layer(i, cur, got, stream)
        want = torch.empty_like(got)
        b = net.biases[i]
        engine.run_layer(net.dlayers[i], cur.data_ptr(), b.data_ptr() if b is not None else 0, want, net.batch,
                         net.flags(i), None, stream)
        torch.cuda.synchronize()
        if not torch.equal(got.view(torch.int32), want.view(torch.int32)):
            raise IntegrityError(f"{L.name}: tuned launch {net.launches[i]} differs from the generic kernel")
        cur = got


def dense_cudnn(specs, kernels, biases, batch: int, dev, reps: int = 10):
    """Dense torch/cuDNN fp32 (IEEE) conv + bias + ReLU (+ max-pool) stack time."""
    import torch
    import paper_2011_06295_b200 as sc
    from paper_2011_06295_b200.cudnn_mode import cudnn_fp32
    torch.backends.cudnn.benchmark = True
    with cudnn_fp32("ieee"):
        ws = [torch.from_numpy(sc.decompress(k)).to(dev) for k in kernels]
        bs = [torch.from_numpy(b).to(dev) for b in biases]
        x = torch.randn((batch, 3, 32, 32), device=dev)

        def step():
            a = x
            for (spec, pool), w, b in zip(specs, ws, bs):
                a = torch.relu(torch.nn.functional.conv2d(a, w, b, padding=spec.shape.padding))
                if pool:
                    a = torch.nn.functional.max_pool2d(a, 2)
            return a

        # per layer (the paper's comparison, sc/bench.py:199-206): the same conv + bias + ReLU
        # (+ 2x2 max-pool) in cuDNN IEEE fp32, TF32 and fp16 tensor cores (channels_last)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        per_layer = []
        for (spec, pool), w, b in zip(specs, ws, bs):
            sh = spec.shape
            e = 32 if sh.h == 32 else sh.h
            xi = torch.randn((batch, sh.c, sh.h, sh.w), device=dev)
            rec = {"layer": spec.name}
            for tag, dt, tf32, cl in (("cudnn_fp32_us", torch.float32, False, False),
                                      ("cudnn_tf32_us", torch.float32, True, False),
                                      ("cudnn_fp16_us", torch.float16, False, True)):
                xx, ww, bb = xi.to(dt), w.to(dt), b.to(dt)
                if cl:
                    xx, ww = xx.to(memory_format=torch.channels_last), ww.to(memory_format=torch.channels_last)

                def lay():
                    a = torch.relu(torch.nn.functional.conv2d(xx, ww, bb, padding=sh.padding))
                    return torch.nn.functional.max_pool2d(a, 2) if pool else a
                with cudnn_fp32("tf32" if tf32 else "ieee"):
                    for _ in range(3):
                        lay()
                    torch.cuda.synchronize()
                    tl = []
                    for _ in range(reps):
                        evs[0].record()
                        lay()
                        evs[1].record()
                        evs[1].synchronize()
                        tl.append(evs[0].elapsed_time(evs[1]))
                rec[tag] = round(statistics.median(tl) * 1e3, 2)
            per_layer.append(rec)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            evs[0].record()
            step()
            evs[1].record()
            evs[1].synchronize()
            ts.append(evs[0].elapsed_time(evs[1]))
        return {"ms_per_step": round(statistics.median(ts), 4),
                "images_per_s": round(batch / (statistics.median(ts) * 1e-3), 1),
                "precision": "fp32 ieee (torch.backends.cudnn.conv.fp32_precision='ieee'), cudnn.benchmark",
                "per_layer": per_layer}


def remap_launches(net, launches, **info):
    """The launches of a tuned net carried over to a sibling net whose kernels differ only in
    the variant fields `info` (weight format, arithmetic mode): same launch shape, the twin
    variant; a launch without a valid twin keeps its variant.  Saves re-tuning each sibling."""
    from paper_2011_06295_b200 import _abi
    vs = _abi.variants()
    index = {tuple(sorted(v.items())): i for i, v in enumerate(vs)}
    out = []
    for i, l in enumerate(launches):
        if l is None:
            out.append(None)
            continue
        twin = dict(vs[l[0]], **info)
        j = index.get(tuple(sorted(twin.items())))
        cand = (j, *l[1:]) if j is not None else tuple(l)
        flags = net.flags(i) | (_abi.FLAG_IMAGE_MINOR if vs[l[0]]["kind"] == _abi.KIND_LANE else 0)
        out.append(cand if net.dlayers[i].launch_ok(net.batch, flags, cand) else tuple(l))
    return out


def measure_f16(specs, args, dev, local_rank, reps: int = 10):
    """BASELINE config 4 (secondary): the same stack with f16 weights and
    activations (f16 storage, FHFMA f32 accumulation -- bit-identical to the
    reference's f16 profile), vs dense cuDNN fp16 tensor-core convolutions."""
    import torch
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import f16_scaled
    net = build_net(specs, seed=0, dtype=np.float16, device=local_rank, weight_fn=f16_scaled)
    net.plan(args.batch, tune=not args.no_tune)
    x = torch.randn((args.batch, 3, 32, 32), device=dev).half()
    for _ in range(3):
        net.forward_device(x)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        ev[0].record()
        net.forward_device(x)
        ev[1].record()
        ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ms = statistics.median(ts)
    gates = {"f16": parity_gate("f16 stack", net.forward_device(x).cpu().numpy(),
                                oracle_forward(x.cpu().numpy(), specs, [L.kernel for L in net.layers],
                                               [L.bias for L in net.layers]))["bitwise"]}
    # dense fp16 comparator: channels_last tensor-core convolutions
    torch.backends.cudnn.benchmark = True
    ws = [torch.from_numpy(__import__("paper_2011_06295_b200").decompress(L.kernel).astype(np.float16)).to(dev)
          .to(memory_format=torch.channels_last) for L in net.layers]
    bs = [torch.from_numpy(L.bias.astype(np.float16)).to(dev) for L in net.layers]
    xc = x.to(memory_format=torch.channels_last)

    def dense():
        a = xc
        for (spec, pool), w, b in zip(specs, ws, bs):
            a = torch.relu(torch.nn.functional.conv2d(a, w, b, padding=spec.shape.padding))
            if pool:
                a = torch.nn.functional.max_pool2d(a, 2)
        return a
    for _ in range(3):
        dense()
    torch.cuda.synchronize()
    td = []
    for _ in range(reps):
        ev[0].record()
        dense()
        ev[1].record()
        ev[1].synchronize()
        td.append(ev[0].elapsed_time(ev[1]))
    # the config-4 weight formats with the REFERENCE's quantizers (quantize_weights_array
    # codebook:16 -> 4-bit codes + f16 table, fixed:16 -> int16 codes x 2^-frac, affine:16 ->
    # int16 codes x f64 step), decoded in registers from 4-byte taps; restated
    # bit-exactly by synth.reference_quantize, pinned by tests/golden/quant_vgg.json)
    from paper_2011_06295_b200.synth import reference_quantized_values_fn
    fixture = ROOT / "tests" / "golden" / "quant_vgg.json"
    fmts = {}
    for fmt, kind in (("cb4", "codebook"), ("lin16", "fixed"), ("aff16", "affine")):
        qn = build_net(specs, seed=0, dtype=np.float16, device=local_rank, weight_format=fmt,
                       weight_fn=f16_scaled, values_fn=reference_quantized_values_fn(kind, fixture))
        qn.plan(args.batch, tune=False)  # the f16 net's tuned launches on the format's twin kernels
        qn.set_launches(remap_launches(qn, net.launches, wf={"cb4": 2, "lin16": 3, "aff16": 4}[fmt]))
        for _ in range(3):
            qn.forward_device(x)
        torch.cuda.synchronize()
        tq = []
        for _ in range(reps):
            ev[0].record()
            qn.forward_device(x)
            ev[1].record()
            ev[1].synchronize()
            tq.append(ev[0].elapsed_time(ev[1]))
        fmts[fmt] = {"ms_per_step": round(statistics.median(tq), 4),
                     "images_per_s": round(args.batch / (statistics.median(tq) * 1e-3), 1)}
        gates[fmt] = parity_gate(f"f16 stack, {fmt} weights", qn.forward_device(x).cpu().numpy(),
                                 oracle_forward(x.cpu().numpy(), specs, [L.kernel for L in qn.layers],
                                                [L.bias for L in qn.layers]))["bitwise"]
        del qn
    # opt-in fast mode (SCB_FLAG_FAST on f16): half2 accumulators within a stage (HFMA2) in the
    # image-lane layers; checked against the oracle with the fp16 tolerance 1e-2*(|ref|+1)
    hn = build_net(specs, seed=0, dtype=np.float16, device=local_rank, weight_fn=f16_scaled, fast_math=True)
    hn.plan(args.batch, tune=False)  # the f16 net's launches, image-lane layers on their half2 twins
    hn.set_launches(remap_launches(hn, net.launches, mode=2))
    for _ in range(3):
        hn.forward_device(x)
    torch.cuda.synchronize()
    th = []
    for _ in range(reps):
        ev[0].record()
        hn.forward_device(x)
        ev[1].record()
        ev[1].synchronize()
        th.append(ev[0].elapsed_time(ev[1]))
    got = hn.forward_device(x).cpu().numpy().astype(np.float64)
    want = oracle_forward(x.cpu().numpy(), specs, [L.kernel for L in hn.layers],
                          [L.bias for L in hn.layers]).astype(np.float64)
    err = float(np.max(np.abs(got - want) / (np.abs(want) + 1)))
    from paper_2011_06295_b200 import _abi as _a
    vs = _a.variants()
    half2 = {"ms_per_step": round(statistics.median(th), 4),
             "images_per_s": round(args.batch / (statistics.median(th) * 1e-3), 1),
             "max_err_over_abs_ref_plus_1": round(err, 6), "within_1e-2": err <= 1e-2,
             "half2_layers": [L.name for L, l in zip(hn.layers, hn.launches)
                              if l is not None and vs[l[0]]["mode"] == 2]}
    del hn
    return {"images_per_s": round(args.batch / (ms * 1e-3), 1), "ms_per_step": round(ms, 4),
            "weight_formats": fmts, "parity_bitwise_vs_oracle": gates, "half2_fast_mode": half2,
            "dense_cudnn_fp16_ms": round(statistics.median(td), 4),
            "arith": "f16 storage, FHFMA (f16 x f16 + f32) accumulation, bit-identical to the reference f16 profile",
            "launches": [None if l is None else list(l) for l in net.launches]}


def measure_alexnet(args, dev, local_rank, reps: int = 10):
    """BASELINE config 2 (secondary): the AlexNet-style CIFAR-10 stack (5x5 and
    3x3 convs) at 90 % unified sparsity, batch 128, exact fp32."""
    import torch
    from paper_2011_06295_b200.network import build_net
    from paper_2011_06295_b200.synth import alexnet_cifar
    net = build_net(alexnet_cifar(args.sparsity), seed=0, device=local_rank)
    batch = 128
    net.plan(batch, tune=not args.no_tune)
    x = torch.randn((batch, 3, 32, 32), device=dev)
    for _ in range(3):
        net.forward_device(x)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        ev[0].record()
        net.forward_device(x)
        ev[1].record()
        ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ms = statistics.median(ts)
    gate = parity_gate("AlexNet-style stack", net.forward_device(x).cpu().numpy(),
                       oracle_forward(x.cpu().numpy(), alexnet_cifar(args.sparsity), [L.kernel for L in net.layers],
                                      [L.bias for L in net.layers]))["bitwise"]
    macs = sum(batch * L.kernel.shape.k * L.kernel.shape.e * L.kernel.shape.f * L.kernel.sparse_level
               for L in net.layers)
    return {"images_per_s": round(batch / (ms * 1e-3), 1), "ms_per_step": round(ms, 4), "batch": batch,
            "parity_bitwise_vs_oracle": gate,
            "tflops": round(2 * macs / (ms * 1e-3) / 1e12, 3),
            "launches": [None if l is None else list(l) for l in net.launches]}


def chains_for(args, n: int) -> int:
    """Sub-batch chains for a per-GPU batch of n: --chains when each chain keeps >= 64 images
    (measured: at 32 images per GPU one chain is 25 % faster than two), else 1."""
    return args.chains if n >= 64 * args.chains else 1


def measure_shard_proxy(args, specs, local_rank, dev, rate_full: float, reps: int = 20):
    """The 8-GPU strong-scaling shard on one GPU: the same stack re-planned (tuned) for
    batch/8 = 32 images, timed like the main step.  Its per-image rate as a fraction of the
    full batch's is what 8 GPUs can at best scale to (no collective on the compute path)."""
    import torch
    from paper_2011_06295_b200.network import build_net
    nb = args.batch // 8
    net = build_net(specs, seed=0, device=local_rank)
    net.plan(nb, tune=not args.no_tune)
    net.pdl = not args.no_pdl
    net.set_chains(chains_for(args, nb))
    x = torch.randn((nb, 3, 32, 32), device=dev)
    net.x_in.copy_(x)
    if args.graph:
        net.capture()  # as the main step: forward_device replays the graph
    for _ in range(5):
        net.forward_device(x)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        net.forward_device(x)
    ev[1].record()
    ev[1].synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    rate = nb / (ms * 1e-3)
    return {"images_per_gpu": nb, "ms_per_step": round(ms, 4), "images_per_s": round(rate, 1),
            "fraction_of_full_batch_rate": round(rate / rate_full, 4),
            "implied_8gpu_images_per_s": round(8 * rate, 1),
            "chains": net.chains, "cuda_graph": bool(args.graph),
            "note": "back-to-back steps without L2 flush (the shard's working set is L2-resident on a real "
                    "8-GPU run too); launches tuned at this batch"}


def measure_sweep(args, local_rank):
    """BASELINE config 5 summary: 256->256 3x3 @32x32, batch 512, sparse (heuristic /
    shipped launches, untuned) vs cuDNN IEEE fp32 / fp16 tensor cores, every point checked
    bit for bit against the oracle on its first 8 images (benchmark.sparsity_sweep, the
    reference's sparsity_sweep semantics).  The tuned full sweep: tools/sweep.py."""
    import paper_2011_06295_b200 as sc
    from oracle import oracle as orc
    from paper_2011_06295_b200.synth import LayerSpec

    def oracle_ref(x, kern, b):
        sh = kern.shape
        return orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, sh.k, sh.r, sh.s, sh.stride,
                               sh.padding, b)
    spec = LayerSpec("sweep-256x32", sc.ConvShape(n=1, c=256, h=32, w=32, k=256, r=3, s=3, padding=1), 0.9)
    out = {"layer": "256->256 3x3 @32x32", "batch": 512, "launches": "heuristic/shipped (untuned)",
           "check": "bitwise vs oracle, first 8 images of each point"}
    for dt in ("f32", "f16"):
        r = sc.sparsity_sweep(spec, [0.5, 0.7, 0.8, 0.9, 0.95, 0.97, 0.99], batch=512, repetitions=5, warmups=2,
                              dtype=dt, device=local_rank, reference_fn=oracle_ref, check_images=8)
        out[dt] = {"sparsities": r.sparsities, "sparse_ms": [round(v, 4) for v in r.sparse_ms],
                   "dense_cudnn_ms": round(r.dense_ms, 4), "crossover": r.crossover}
    return out


def load_traffic():
    """Per-layer DRAM traffic (dram__bytes_read.sum + write.sum) from the
    committed ncu --set full capture summary, if any."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return {}
    return {}


def load_smem_pipe():
    """Per-layer shared-memory pipe utilisation (l1tex throughput % of peak, the kernels'
    real ceiling) from the committed ncu --set full stack summary, layers in order."""
    import csv
    caps = sorted((ROOT / "profiles").glob("r0*_ncu_full_stack_v*.csv"),
                  key=lambda q: (q.stem[:3], int(q.stem.rsplit("_v", 1)[1])))
    if not caps:
        return {}, None
    rows = list(csv.reader(caps[-1].open()))
    h = rows[0]
    col = "l1tex__throughput.avg.pct_of_peak_sustained_active"
    if col not in h:
        return {}, None
    kn = h.index("Kernel Name") if "Kernel Name" in h else None
    vals = [float(r[h.index(col)]) for r in rows[2:]
            if len(r) > h.index(col) and (kn is None or "k_transpose" not in r[kn])]
    from paper_2011_06295_b200.synth import VGG16_CIFAR_LAYERS
    names = [n for n, *_ in VGG16_CIFAR_LAYERS]
    return dict(zip(names, vals)), f"profiles/{caps[-1].name}"


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    from paper_2011_06295_b200.network import build_net
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    from paper_2011_06295_b200.runner import shard_range, shard_sizes
    specs = workload(args.sparsity)
    net = build_net(specs, seed=0, device=local_rank)
    net.fuse_layouts = not args.no_fuse_layouts
    # strong scaling: the global batch is split into contiguous shards, one per rank
    s0, s1 = shard_range(args.batch, world, rank)
    nloc = s1 - s0
    t0 = time.perf_counter()
    lf = Path(args.launches) if args.launches else None
    if lf is not None and lf.exists():
        net.plan(nloc, tune=False)
        net.set_launches([None if l is None else tuple(l) for l in json.loads(lf.read_text())])
    else:
        net.plan(nloc, tune=not args.no_tune)
        if lf is not None and rank == 0:
            lf.parent.mkdir(parents=True, exist_ok=True)
            lf.write_text(json.dumps([None if l is None else list(l) for l in net.launches]))
    launches = list(net.launches)
    tune_s = time.perf_counter() - t0
    chains = chains_for(args, nloc)
    net.set_chains(chains)
    net.pdl = not args.no_pdl

    g = torch.Generator(device="cpu").manual_seed(1234)
    x_global = torch.randn((args.batch, 3, 32, 32), generator=g)  # identical on every rank
    x_host = x_global[s0:s1].contiguous().pin_memory()
    x_dev = x_host.to(dev)
    integrity_gate(net, x_dev)
    # the exact timed configuration (tuned launches, sub-batch chains, PDL) against the oracle,
    # bit for bit, on this rank's shard of the step's input
    got = net.forward_device(x_dev).cpu().numpy()
    parity = parity_gate("VGG-16/CIFAR fp32 stack (timed mode)", got,
                         oracle_forward(x_host.numpy(), specs, [L.kernel for L in net.layers],
                                        [L.bias for L in net.layers]))
    parity.update({"images": nloc, "mode": f"timed launches, {chains} sub-batch chain(s), "
                                           f"pdl={not args.no_pdl}"})
    if args.graph:
        net.x_in.copy_(x_dev)
        net.capture()  # forward_device replays it (per-layer event passes stay eager)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    nl = len(net.layers)
    stream = torch.cuda.current_stream(dev)

    def step(evs=None):
        return net.forward_device(x_dev, events=evs)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # timed steps: events only around each step, so consecutive layer kernels keep their
    # programmatic-dependent-launch overlap (an event between kernels would serialise them)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local_rank) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            sev[k][0].record(stream)
            step()
            sev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in sev]
    total_s = sum(step_ms) * 1e-3
    # per-layer breakdown: separate (untimed for `value`) steps with events between layers
    nlay = max(5, args.steps // 5)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(nlay)]
    for k in range(nlay):
        flush.zero_()
        step(ev[k])
    torch.cuda.synchronize()
    layer_ms = [[ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(nlay)] for i in range(nl)]

    # e2e through the host-facing API, every step's host->device input copy and device->host
    # result inside the timed region.  N = 1: SparseConvNet.forward_stream (pinned host in and
    # out, copies of neighbouring steps overlapped with compute).  N > 1: per step each rank
    # copies its shard in, runs the stack, the outputs are gathered to rank 0 with a collective
    # (BatchShardedRunner, NCCL over NVLink) and rank 0 reads the global result back.
    out_shape_loc = net.out_shape(nl - 1, nloc)
    e_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if world == 1:
        out_host = torch.empty(out_shape_loc, dtype=torch.float32, pin_memory=True)
        xs_host = [x_host] * args.steps
        outs_host = [torch.empty_like(out_host).pin_memory() for _ in range(2)]
        outs_list = [outs_host[i % 2] for i in range(args.steps)]
        net.forward_stream(xs_host[:2], outs_list[:2])
        torch.cuda.synchronize()
        e_ev[0].record(stream)
        net.forward_stream(xs_host, outs_list)
        e_ev[1].record(stream)
        e_ev[1].synchronize()
        gather_api = "SparseConvNet.forward_stream (pinned host in/out, copies overlapped across steps)"
    else:
        from paper_2011_06295_b200.runner import BatchShardedRunner
        x_step = torch.empty_like(x_dev)
        out_host = torch.empty((args.batch, *out_shape_loc[1:]), dtype=torch.float32, pin_memory=True)

        def fwd(xh):
            x_step.copy_(xh, non_blocking=True)
            return net.forward_device(x_step)
        runner = BatchShardedRunner(fwd)

        def e2e_step():
            y = runner.run(x_host)  # x_host is this rank's shard; sizes exchanged by all_gather
            if rank == 0:
                out_host.copy_(y, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        e_ev[0].record(stream)
        for _ in range(args.steps):
            e2e_step()
        e_ev[1].record(stream)
        e_ev[1].synchronize()
        gather_api = ("BatchShardedRunner.run: per-rank H2D of the shard, SparseConvNet.forward_device, "
                      f"{dist.get_backend()} gather to rank 0, D2H of the global output on rank 0")
    e2e_s = e_ev[0].elapsed_time(e_ev[1]) * 1e-3

    # max over ranks
    t = torch.tensor([total_s, e2e_s], dtype=torch.float64,
                     device=dev if (world > 1 and dist.get_backend() == "nccl") else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # device time: max over ranks
    total_s, e2e_s = float(t[0]), float(t[1])
    proxy = None
    if world == 1 and not args.no_proxy and args.batch >= 64:
        proxy = measure_shard_proxy(args, specs, local_rank, dev, args.batch / (total_s / args.steps))
    if rank != 0:
        return

    images = args.batch * args.steps  # the global batch per step (strong scaling)
    value = images / total_s
    peaks = fma_peak_tflops(local_rank)
    peak_exact = peaks.get("fmul_fadd")
    hbm_peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    traffic = load_traffic()
    smem, smem_src = load_smem_pipe()
    layers = []
    for i, ((spec, pool), kern) in enumerate(zip(specs, [L.kernel for L in net.layers])):
        us = statistics.median(layer_ms[i]) * 1e3
        fl, by = layer_work(spec, kern.sparse_level, nloc, pool)
        layers.append({"layer": spec.name, "L": int(kern.sparse_level), "us": round(us, 2),
                       "tflops": round(fl / (us * 1e-6) / 1e12, 3), "hbm_gbs": round(by / (us * 1e-6) / 1e9, 1),
                       "fma_frac": round(fl / (us * 1e-6) / 1e12 / peak_exact, 4) if peak_exact else None,
                       "launch": list(launches[i]) if launches[i] is not None else "generic"})
    top = max(range(nl), key=lambda i: layers[i]["us"])
    fl, by = layer_work(specs[top][0], layers[top]["L"], nloc, specs[top][1])
    mean_us = statistics.mean(layer_ms[top]) * 1e3
    ach = fl / (mean_us * 1e-6) / 1e12
    roof = {"bound": "fma", "kernel": specs[top][0].name, "achieved": round(ach, 3), "peak": round(peak_exact, 3),
            "unit": "TFLOP/s", "frac": round(ach / peak_exact, 4),
            "peak_source": "measured live: scb_fma_peaks 'fmul_fadd' (exact mode = FMUL+FADD per MAC); "
                           "MEASURED_PEAKS.json has no CUDA-core peak",
            "ffma_peak_tflops": round(peaks.get("ffma", 0), 2),
            "algorithmic_flops": fl, "algorithmic_bytes": by,
            "hbm_achieved_gbs": round(by / (mean_us * 1e-6) / 1e9, 1), "hbm_peak_gbs": hbm_peak,
            "traffic": traffic.get(specs[top][0].name),
            "smem_pipe_pct": smem.get(specs[top][0].name), "smem_pipe_source": smem_src}
    # per kernel kind: the layers each kind runs and their time-weighted fraction of the peak
    from paper_2011_06295_b200 import engine as _eng
    kinds = {}
    for i, rec in enumerate(layers):
        kk = {2: "direct", 7: "image-lane position classes (kind 7)"}.get(_eng.launch_kind(launches[i]),
                                                                         f"kind {_eng.launch_kind(launches[i])}")
        kinds.setdefault(kk, []).append(rec)
    roof["per_kernel_kind"] = {
        kk: {"layers": [r["layer"] for r in recs], "us": round(sum(r["us"] for r in recs), 1),
             "frac_time_weighted": round(sum(r["fma_frac"] * r["us"] for r in recs) / sum(r["us"] for r in recs), 4),
             "frac_max": max(r["fma_frac"] for r in recs)}
        for kk, recs in kinds.items() if all(r["fma_frac"] is not None for r in recs)}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(total_s / args.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: make_layer_weights (bench.py:105-116 restated), N(0,1) activations",
        "config": {"workload": workload_name(args.sparsity),
                   "batch_per_gpu": max(shard_sizes(args.batch, world)), "global_batch": args.batch,
                   "parallelism": f"batch-sharded x{world} (strong: shards {shard_sizes(args.batch, world)}; "
                                  "no collective on the compute path, final gather in e2e)",
                   "l2": "flushed between timed steps (256 MB write, untimed)",
                   "tuned": not args.no_tune, "tune_seconds": round(tune_s, 1),
                   "streams_per_gpu": chains, "pdl": not args.no_pdl, "cuda_graph": bool(args.graph)},
        "e2e": {"value": round(args.batch * args.steps / e2e_s, 1), "unit": "images/s",
                "h2d_bytes_per_step": int(args.batch * 3 * 32 * 32 * 4),
                "d2h_bytes_per_step": int(args.batch * int(np.prod(out_shape_loc[1:])) * 4),
                "api": gather_api},
        "gpu_launches": net.kernels_per_step() * args.steps,
        "clocks": clk.summary(),
        "roofline": roof,
        "parity": parity,
        "layers": layers,
        "fma_peaks_tflops": {k: round(v, 2) for k, v in peaks.items()},
        "repo_native_libs_loaded": repo_libs_loaded(),
    }
    if proxy is not None:
        line["proxy_8gpu_shard"] = proxy
    if not args.no_f16 and world == 1:
        line["f16"] = measure_f16(specs, args, dev, local_rank)
    if not args.no_alexnet and world == 1:
        line["alexnet"] = measure_alexnet(args, dev, local_rank)
    if not args.no_dense and world == 1:
        line["dense_cudnn"] = dense_cudnn(specs, [L.kernel for L in net.layers], [L.bias for L in net.layers],
                                          args.batch, dev)
        sp_us = {l["layer"]: l["us"] for l in layers}
        for rec in line["dense_cudnn"]["per_layer"]:
            rec["sparse_us"] = sp_us.get(rec["layer"])
            rec["speedup_vs_cudnn_fp32"] = round(rec["cudnn_fp32_us"] / rec["sparse_us"], 3)
        line["dense_cudnn"]["layers_slower_than_cudnn_fp32"] = [
            r["layer"] for r in line["dense_cudnn"]["per_layer"] if r["sparse_us"] >= r["cudnn_fp32_us"]]
    if not args.no_sweep and world == 1:
        line["sweep"] = measure_sweep(args, local_rank)
    if not args.no_cpu and world == 1:
        per_pass, passes, threads = cpu_stack_time(specs, [L.kernel for L in net.layers],
                                                   [L.bias for L in net.layers], args.cpu_images,
                                                   args.cpu_seconds)
        line["cpu_baseline"] = {"value": round(args.cpu_images / per_pass, 3), "unit": "images/s",
                                "cores": threads, "kind": "port",
                                "sample": f"{passes} passes of the 13-layer stack over {args.cpu_images} images "
                                          "(oracle/oracle.c restatement of conv_sparse_kernel, OpenMP)"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        ndev = torch.cuda.device_count()
        if ndev >= world:  # one process per GPU: NCCL over NVLink
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # oversubscribed test launch (more ranks than GPUs): CPU collectives
            local_rank %= max(ndev, 1)
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
