"""Network runner: the conv loop of the reference's ``Model.forward``
(store.py:263-286) on one B200.

``Model.forward`` walks its conv layers, calling ``conv_sparse`` with the
layer's CsrKernel and bias, then ``np.maximum(z, 0)`` for ReLU layers
(store.py:276,284).  ``SparseConvNet`` does the same walk with every layer
resident on the device:

* each layer's CsrKernel is uploaded once (device.DeviceLayer) -- the
  reference rebuilds CSR on every forward for dense-stored layers
  (store.py:178-182);
* ReLU, and the 2x2/2 max-pool that the CIFAR stacks put between stages
  (the reference has no pooling: SURVEY.md 7.4 #9), are fused into the conv
  kernel's epilogue (SCB_FLAG_RELU / SCB_FLAG_POOL2), so one layer is one
  kernel launch and nothing else;
* activations live in preallocated device buffers; the whole stack can be
  captured into one CUDA graph (``capture``) so replays pay no launch cost;
* ``forward`` is the host-facing call: pinned host batch -> H2D -> layers ->
  D2H of the final activations, all on one stream.

Outputs are bit-identical to running the reference layer by layer
(conv_sparse -> maximum -> pool) in exact mode; tests/test_gpu_parity.py
checks that against the CPU oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi, engine
from .device import DeviceLayer, device_layer
from .errors import ShapeError
from .weights import CsrKernel


@dataclass
class NetLayer:
    """One conv layer of the stack (cf. ConvLayerRecord, store.py:127-181)."""

    name: str
    kernel: CsrKernel
    bias: np.ndarray | None = None
    relu: bool = True
    pool: bool = False  # fused 2x2 stride-2 max-pool after the activation
    act_quant: dict | None = None  # activation fake-quant after the ReLU (store.py:285-286)


class SparseConvNet:
    """A sequential sparse-conv stack resident on one GPU.

    ``plan(batch)`` allocates the activation buffers for a batch size and
    (optionally) runs the measured launch tuner on every layer;
    ``forward_device`` runs the stack asynchronously on the current stream;
    ``forward`` adds the host copies.  ``dtype`` is the activation dtype
    (f32, or f16 with f16 weights); ``weight_format`` selects in-register
    dequantisation ("cb4" / "lin16")."""

    def __init__(self, layers: list[NetLayer], device: int = 0, dtype=np.float32,
                 weight_format: str = "native", fast_math: bool = False):
        import torch
        if not layers:
            raise ShapeError("empty network")
        self.torch = torch
        self.layers = list(layers)
        self.device = int(device)
        self.dtype = np.dtype(dtype)
        self.weight_format = weight_format
        self.fast_math = bool(fast_math)
        self.tdev = torch.device("cuda", self.device)
        self.tdtype = engine._torch_dtype(self.dtype)
        self.batch = None
        self.graph = None
        # geometry chain check: each layer's input is the previous output
        for a, b in zip(self.layers, self.layers[1:]):
            sa, sb = a.kernel.shape, b.kernel.shape
            e, f = (sa.e // 2, sa.f // 2) if a.pool else (sa.e, sa.f)
            if (sa.k, e, f) != (sb.c, sb.h, sb.w):
                raise ShapeError(f"{a.name} -> {b.name}: output ({sa.k},{e},{f}) does not "
                                 f"match input ({sb.c},{sb.h},{sb.w})")
        self.dlayers = []
        self.biases = []
        for L in self.layers:
            if self.dtype == np.float16 and L.kernel.values.dtype != np.float16:
                raise ShapeError(f"{L.name}: f16 activations need f16 weights")
            if L.act_quant is None:
                self.dlayers.append(device_layer(L.kernel, self.device, self.dtype, weight_format))
            else:  # a private device layer: the quantizer is attached to it
                dl = DeviceLayer(L.kernel, self.device, self.dtype, weight_format)
                dl.set_act_quant(L.act_quant)
                self.dlayers.append(dl)
            if L.bias is None:
                self.biases.append(None)
            else:
                b = np.ascontiguousarray(L.bias, dtype=np.float32)
                if b.shape != (L.kernel.shape.k,):
                    raise ShapeError(f"{L.name}: bias must have shape ({L.kernel.shape.k},)")
                self.biases.append(torch.from_numpy(b).to(self.tdev))
        self.launches = [None] * len(self.layers)
        self.algorithms = ["sparse-direct"] * len(self.layers)
        self._dense = [None] * len(self.layers)
        self.chains = 1
        self.pdl = True  # programmatic dependent launch between consecutive layer kernels
        self.fuse_layouts = True  # layout changes written by the neighbouring layer kernels
        self._side_streams = []

    # ---- shapes ---------------------------------------------------------
    def flags(self, i: int) -> int:
        L = self.layers[i]
        f = 0
        if L.relu:
            f |= _abi.FLAG_RELU
        if L.pool:
            f |= _abi.FLAG_POOL2
        if self.fast_math:
            f |= _abi.FLAG_FAST
        if L.act_quant is not None:
            f |= _abi.FLAG_ACT_QUANT
        return f

    def out_shape(self, i: int, n: int):
        sh = self.layers[i].kernel.shape
        e, f = (sh.e // 2, sh.f // 2) if self.layers[i].pool else (sh.e, sh.f)
        return (n, sh.k, e, f)

    @property
    def in_shape(self):
        sh = self.layers[0].kernel.shape
        return (sh.c, sh.h, sh.w)

    # ---- planning -------------------------------------------------------
    def plan(self, batch: int, tune: bool = True, repetitions: int = 3, warmups: int = 1,
             max_candidates: int | None = None) -> list:
        """Allocate activations for `batch` images and pick every layer's
        launch (measured when `tune`, else the C heuristic)."""
        torch = self.torch
        self.batch = int(batch)
        self.graph = None
        self.x_in = torch.zeros((self.batch, *self.in_shape), dtype=self.tdtype, device=self.tdev)
        self.acts = [None] * len(self.layers)  # allocated per layout by set_launches
        self.scratch = [None] * len(self.layers)
        if tune:
            from .tuner import tune_launch
            gen = torch.Generator(device="cpu").manual_seed(0)
            x = torch.randn((self.batch, *self.in_shape), generator=gen).to(self.tdev, self.tdtype)
            plan = engine.EnginePlan(fast_math=self.fast_math, weight_format=self.weight_format,
                                     device=self.device)
            opts = []  # per layer: (NCHW launch, seconds, image-minor launch, seconds)
            with torch.cuda.device(self.device):
                for i, L in enumerate(self.layers):
                    best, tim = tune_launch(x, L.kernel, L.bias, plan, relu=L.relu, pool=L.pool,
                                            repetitions=repetitions, warmups=warmups,
                                            max_candidates=max_candidates, include_generic=True)
                    # image-minor kernels (kind 7), timed on their own layout
                    bm, tm = tune_launch(x, L.kernel, L.bias, plan, relu=L.relu, pool=L.pool,
                                         repetitions=repetitions, warmups=warmups,
                                         max_candidates=max_candidates, layout="minor")
                    opts.append((best, tim[best], bm, tm[bm] if bm is not None else float("inf")))
                    x = torch.relu(torch.randn(self.out_shape(i, self.batch), generator=gen)).to(
                        self.tdev, self.tdtype)
            self.launches = self._pick_layouts(opts)
        else:
            self.launches = []
            for i in range(len(self.layers)):
                l = self.dlayers[i].default_launch(self.batch, self.flags(i))
                # measured (profiles/r02_lane_*): the image-minor kernels win where they apply
                lm = self.dlayers[i].default_launch(self.batch, self.flags(i) | _abi.FLAG_IMAGE_MINOR)
                if lm[0] >= 0:
                    l = lm
                self.launches.append(None if l[0] < 0 else l)
        self.set_launches(self.launches)
        return list(self.launches)

    def _layout_change_s(self, i: int) -> float:
        """Estimated seconds to change the layout of layer i's output (-1: the stack input):
        one transpose kernel, read + write at ~5 TB/s."""
        shp = (self.batch, *self.in_shape) if i < 0 else self.out_shape(i, self.batch)
        return 2.0 * float(np.prod(shp)) * np.dtype(self.dtype).itemsize / 5.0e12

    def _pick_layouts(self, opts) -> list:
        """Per-layer layout choice over the measured kernel times plus the layout changes
        between consecutive layers (two-state shortest path: NCHW / image-minor)."""
        inf = float("inf")
        nl = len(opts)
        cost = [opts[0][1], opts[0][3] + self._layout_change_s(-1)]  # ends in NCHW / minor
        back = []
        for i in range(1, nl):
            ch = self._layout_change_s(i - 1)
            cn = [cost[0], cost[1] + ch]
            cm = [cost[0] + ch, cost[1]]
            back.append((int(cn[1] < cn[0]), int(cm[1] < cm[0])))
            cost = [min(cn) + opts[i][1], min(cm) + opts[i][3]]
        cost[1] += self._layout_change_s(nl - 1)  # the NCHW result
        state = int(cost[1] < cost[0] and cost[1] < inf)
        pick = [state]
        for i in range(nl - 2, -1, -1):
            state = back[i][state]
            pick.append(state)
        pick.reverse()
        return [opts[i][2] if m else opts[i][0] for i, m in enumerate(pick)]

    def set_launches(self, launches) -> None:
        """Install explicit per-layer launches (tuple, or None = generic)."""
        if len(launches) != len(self.layers):
            raise ShapeError("one launch per layer")
        self.launches = list(launches)
        self.graph = None
        torch = self.torch
        ld = engine.minor_ld(self.batch)
        self.ld = ld
        self.minor = [a == "sparse-direct" and engine.launch_kind(l) == _abi.KIND_LANE
                      for l, a in zip(self.launches, self.algorithms)]
        nl = len(self.layers)
        # fused layout changes: a narrow direct layer feeding an image-minor run writes its output
        # image-minor (SCB_FLAG_Y_IMAGE_MINOR), and the last layer of an image-minor run writes
        # NCHW (SCB_FLAG_Y_NCHW) -- no conversion kernel at either end when the launch allows it.
        # Only for small output planes (<= 16 positions): those stores scatter one element per
        # 32-byte sector (measured on a 32x32 plane: 141 us in place of 32 us + a 20 us transpose)
        self.yflag = [0] * nl
        vs = _abi.variants()
        for i in range(nl):
            l = self.launches[i]
            if self.algorithms[i] != "sparse-direct" or l is None or not self.fuse_layouts:
                continue
            nxt_minor = i + 1 < nl and self.minor[i + 1]
            _, _, e, f = self.out_shape(i, 1)
            if e * f > 16:
                continue
            if not self.minor[i] and nxt_minor and vs[l[0]]["kind"] == 2 and vs[l[0]]["dispatch"] == 0:
                f = self.flags(i) | _abi.FLAG_Y_IMAGE_MINOR
                if self.dlayers[i].launch_ok(self.batch, f, l):
                    self.yflag[i] = _abi.FLAG_Y_IMAGE_MINOR
            elif self.minor[i] and not nxt_minor:
                f = self.flags(i) | _abi.FLAG_IMAGE_MINOR | _abi.FLAG_Y_NCHW
                if self.dlayers[i].launch_ok(self.batch, f, l):
                    self.yflag[i] = _abi.FLAG_Y_NCHW
        # output layout of each layer, and a conversion buffer where a layer's input differs
        self.out_minor = [(m and self.yflag[i] != _abi.FLAG_Y_NCHW) or self.yflag[i] == _abi.FLAG_Y_IMAGE_MINOR
                          for i, m in enumerate(self.minor)]
        self.acts = []
        self.xconv = []
        for i in range(nl):
            n, k, e, f = self.out_shape(i, self.batch)
            if self.out_minor[i]:
                self.acts.append(torch.empty((k * e * f, ld), dtype=self.tdtype, device=self.tdev))
            else:
                self.acts.append(torch.empty((n, k, e, f), dtype=self.tdtype, device=self.tdev))
            sh = self.layers[i].kernel.shape
            in_minor = i > 0 and self.out_minor[i - 1]
            if self.minor[i] and not in_minor:
                self.xconv.append(torch.empty((sh.c * sh.h * sh.w, ld), dtype=self.tdtype, device=self.tdev))
            elif in_minor and not self.minor[i]:
                self.xconv.append(torch.empty((self.batch, sh.c, sh.h, sh.w), dtype=self.tdtype, device=self.tdev))
            else:
                self.xconv.append(None)
        # NCHW result of the stack (the last layer's output, converted when image-minor)
        self.result = torch.empty(self.out_shape(nl - 1, self.batch), dtype=self.tdtype,
                                  device=self.tdev) if self.out_minor[-1] else self.acts[-1]
        for i, L in enumerate(self.layers):
            self.scratch[i] = None
            if self.launches[i] is None and L.pool:
                sh = L.kernel.shape
                self.scratch[i] = self.torch.empty((self.batch, sh.k, sh.e, sh.f), dtype=self.tdtype,
                                                   device=self.tdev)
        self._prepare_all()

    def _prepare_all(self) -> None:
        """Build every layer's launch tables for the batch and each sub-batch chain size
        (scb_layer_prepare) up front: the step itself then never allocates, which also
        keeps it capturable into a CUDA graph."""
        if self.batch is None:
            return
        sizes = {e - a for a, e in self._chain_bounds()} | {self.batch}
        for i, L in enumerate(self.layers):
            if self.launches[i] is None or self.algorithms[i] != "sparse-direct":
                continue
            for n in sizes:
                for pdl in (0, _abi.FLAG_NO_PDL):
                    self.dlayers[i].prepare(n, self.flags(i) | pdl | self._layout_flag(i) | self.yflag[i],
                                            self.launches[i])

    def set_chains(self, chains: int) -> None:
        """Run the batch as `chains` independent sub-batch chains on their own
        streams (images are independent, so this changes no result bit): the
        last partial wave of one chain's layer kernel overlaps the other
        chains' kernels instead of leaving SMs idle.  1 = one stream."""
        chains = int(chains)
        if chains < 1 or (self.batch is not None and chains > self.batch):
            raise ShapeError(f"chains must be in [1, batch], got {chains}")
        self.chains = chains
        self.graph = None
        if self.batch is not None and len(self.launches) == len(self.layers):
            self._prepare_all()

    def _chain_bounds(self):
        from .runner import shard_range
        b = [shard_range(self.batch, self.chains, j) for j in range(self.chains)]
        if any(getattr(self, "minor", None) or []):
            # image-minor sub-batches start at a multiple of 8 images (16-byte aligned TMA
            # rows in f32 and f16)
            cuts = sorted({min(self.batch, (a + 7) // 8 * 8) for a, _ in b} | {self.batch})
            b = [(a, e) for a, e in zip([0] + cuts[:-1], cuts) if e > a]
        return b

    # ---- execution ------------------------------------------------------
    def _layout_flag(self, i: int) -> int:
        return _abi.FLAG_IMAGE_MINOR if getattr(self, "minor", None) and self.minor[i] else 0

    def launch_layer(self, i: int, x_dev, y_dev, stream: int, rows: tuple | None = None) -> None:
        """Layer i on images rows[0]:rows[1] (default: the whole batch) of NCHW buffers
        (a kind-7 launch converts through temporary image-minor buffers: engine.run_layer)."""
        b = self.biases[i]
        a, e = rows if rows is not None else (0, self.batch)
        sc = self.scratch[i]
        engine.run_layer(self.dlayers[i], x_dev[a:e].data_ptr(), b.data_ptr() if b is not None else 0,
                         y_dev[a:e], e - a, self.flags(i) | (0 if self.pdl else _abi.FLAG_NO_PDL),
                         self.launches[i], stream,
                         scratch=None if sc is None else sc[a:e])

    def _minor_ptr(self, buf, a: int) -> int:
        return buf.data_ptr() + a * buf.element_size()

    def _step(self, i: int, cur, cur_minor: bool, stream, rows):
        """Layer i of one chain: converts the input layout when the producer's differs,
        runs the layer into self.acts[i]; returns (output buffer, output is image-minor)."""
        a, e = rows
        n = e - a
        s = stream.cuda_stream
        if self.algorithms[i] == "dense-cudnn":
            if cur_minor:
                cur = self._to_nchw(i, cur, rows, s)
            with self.torch.cuda.stream(stream):
                self.dense_layer(i)(cur[a:e], self.acts[i][a:e])
            self._dense_quant(i, self.acts[i][a:e], s)
            return self.acts[i], False
        pdl = 0 if self.pdl else _abi.FLAG_NO_PDL
        b = self.biases[i]
        bptr = b.data_ptr() if b is not None else 0
        if self.minor[i]:
            if not cur_minor:
                sh = self.layers[i].kernel.shape
                xc = self.xconv[i]
                _abi.to_image_minor(self.dtype, cur[a:e].data_ptr(), self._minor_ptr(xc, a), n,
                                    sh.c * sh.h * sh.w, self.ld, s)
                cur = xc
            y = self._minor_ptr(self.acts[i], a) if self.out_minor[i] else self.acts[i][a:e].data_ptr()
            self.dlayers[i].launch(self._minor_ptr(cur, a), bptr, y, n,
                                   self.flags(i) | _abi.FLAG_IMAGE_MINOR | self.yflag[i] | pdl,
                                   self.launches[i], s, ldx=self.ld, ldy=self.ld)
            return self.acts[i], self.out_minor[i]
        if cur_minor:
            cur = self._to_nchw(i, cur, rows, s)
        if self.yflag[i] == _abi.FLAG_Y_IMAGE_MINOR:  # writes the next layer's image-minor input
            self.dlayers[i].launch(cur[a:e].data_ptr(), bptr, self._minor_ptr(self.acts[i], a), n,
                                   self.flags(i) | _abi.FLAG_Y_IMAGE_MINOR | pdl, self.launches[i], s,
                                   ldy=self.ld)
            return self.acts[i], True
        self.launch_layer(i, cur, self.acts[i], s, rows)
        return self.acts[i], False

    def _to_nchw(self, i: int, cur, rows, s: int):
        a, e = rows
        xc = self.xconv[i]
        _abi.from_image_minor(self.dtype, self._minor_ptr(cur, a), self.ld, xc[a:e].data_ptr(), e - a,
                              int(np.prod(xc.shape[1:])), s)
        return xc

    def _finish(self, cur, cur_minor: bool, stream, rows) -> None:
        """The NCHW result: convert the last (image-minor) output into self.result."""
        if cur_minor:
            a, e = rows
            _abi.from_image_minor(self.dtype, self._minor_ptr(cur, a), self.ld, self.result[a:e].data_ptr(),
                                  e - a, int(np.prod(self.result.shape[1:])), stream.cuda_stream)

    def _run_chain(self, x, stream, rows, on_first=None) -> None:
        cur, cur_minor = x, False
        for i in range(len(self.layers)):
            cur, cur_minor = self._step(i, cur, cur_minor, stream, rows)
            if i == 0 and on_first is not None:
                on_first(stream)
        self._finish(cur, cur_minor, stream, rows)

    def _run_stack(self, x, stream, on_first=None) -> None:
        """The whole stack on `stream`, forked over the sub-batch chains."""
        torch = self.torch
        if self.chains == 1:
            self._run_chain(x, stream, (0, self.batch), on_first)
            return
        while len(self._side_streams) < self.chains - 1:
            self._side_streams.append(torch.cuda.Stream(self.device))
        streams = [stream] + self._side_streams[:self.chains - 1]
        for s in streams[1:]:
            s.wait_stream(stream)
        for s, rows in zip(streams, self._chain_bounds()):
            self._run_chain(x, s, rows)
        for s in streams[1:]:
            stream.wait_stream(s)
        if on_first is not None:
            on_first(stream)  # (joined: every chain is past its first layer)

    def dense_layer(self, i: int):
        """Dense cuDNN equivalent of layer i (IEEE fp32 / fp16, TF32 off):
        conv2d + bias, ReLU, 2x2 max-pool; the "dense-cudnn" algorithm of a
        NetworkConfig (configure.py)."""
        if self._dense[i] is None:
            import torch
            from .weights import decompress
            L = self.layers[i]
            sh = L.kernel.shape
            w = torch.from_numpy(decompress(L.kernel).astype(self.dtype)).to(self.tdev)
            b = None if L.bias is None else torch.from_numpy(
                np.asarray(L.bias, dtype=self.dtype)).to(self.tdev)

            def run(x, out=None):
                from .cudnn_mode import cudnn_fp32
                with cudnn_fp32("ieee"):
                    a = torch.nn.functional.conv2d(x, w, b, stride=sh.stride, padding=sh.padding)
                if L.relu:
                    a = torch.relu(a)
                if L.pool:
                    a = torch.nn.functional.max_pool2d(a, 2)
                if out is not None:
                    out.copy_(a)
                    return out
                return a
            self._dense[i] = run
        return self._dense[i]

    def apply_config(self, config) -> None:
        """Install a NetworkConfig (configure.py): per-layer algorithm and, for
        sparse layers, the recorded launch."""
        if self.batch is None or config.batch != self.batch:
            self.plan(config.batch, tune=False)
        launches = list(self.launches)
        for i, L in enumerate(self.layers):
            ch = config.choices.get(L.name, {})
            algo = ch.get("algorithm", "sparse-direct")
            # a config written by the reference names its CPU dense baselines (bench.py:238,
            # ALGORITHMS): on the GPU the dense path of either is the cuDNN convolution
            algo = {"dense-direct": "dense-cudnn", "dense-gemm": "dense-cudnn"}.get(algo, algo)
            if algo not in ("sparse-direct", "dense-cudnn"):
                raise ShapeError(f"unknown algorithm {algo!r} for layer {L.name}")
            self.algorithms[i] = algo
            if algo == "sparse-direct" and "launch" in ch:
                launches[i] = None if ch["launch"] is None else tuple(ch["launch"])
        self.set_launches(launches)

    def _dense_quant(self, i: int, out, stream: int) -> None:
        """Activation fake-quant after a dense (cuDNN) layer (store.py:285-286)."""
        aq = self.layers[i].act_quant
        if aq is not None:
            _abi.fake_quant(self.dtype, out.data_ptr(), out.numel(), aq, stream)

    def kernels_per_step(self) -> int:
        """Our kernel launches in one forward: one per sparse layer, +1 for a generic
        layer's separate pool, +1 for a fake-quant pass the layer's kernel does not fuse
        (only the direct and image-lane epilogues do), +1 after a dense layer with one."""
        vs = _abi.variants()
        n = 0
        prev_out_minor = False
        for i, (l, L, a) in enumerate(zip(self.launches, self.layers, self.algorithms)):
            aq = L.act_quant is not None
            n += 1 if self.minor[i] != prev_out_minor else 0  # layout conversion of the input
            prev_out_minor = self.out_minor[i]
            if a == "dense-cudnn":
                n += 1 if aq else 0
                continue
            n += 2 if (l is None and L.pool) else 1
            if aq and (l is None or vs[l[0]]["kind"] not in (2, 3, 7)):
                n += 1
        return n + (1 if prev_out_minor else 0)

    def forward_device(self, x_dev=None, events=None):
        """Run the stack on the current stream of the device; returns the last
        activation buffer (no synchronisation).  ``events``: optional list of
        len(layers)+1 CUDA events recorded between layers."""
        torch = self.torch
        if self.batch is None:
            raise ShapeError("call plan(batch) first")
        if x_dev is not None and x_dev is not self.x_in:
            self.x_in.copy_(x_dev)
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            if self.graph is not None and events is None:
                self.graph.replay()
                return self.result
            if events is None:
                self._run_stack(self.x_in, stream)
                return self.result
            # per-layer events: one chain, an event between layers (a layout conversion
            # is timed with the layer that needs it)
            rows = (0, self.batch)
            cur, cur_minor = self.x_in, False
            events[0].record(stream)
            for i in range(len(self.layers)):
                cur, cur_minor = self._step(i, cur, cur_minor, stream, rows)
                if i == len(self.layers) - 1:
                    self._finish(cur, cur_minor, stream, rows)
                events[i + 1].record(stream)
        return self.result

    def capture(self) -> None:
        """Capture the whole stack into one CUDA graph (replayed by
        forward_device when no per-layer events are requested)."""
        torch = self.torch
        with torch.cuda.device(self.device):
            self.graph = None
            s = torch.cuda.Stream(self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                self.forward_device()  # warm (lazy attribute setup outside capture)
            torch.cuda.current_stream(self.device).wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.forward_device()
            self.graph = g

    def forward(self, x_host, out_host=None):
        """Host batch in, host activations out (the call a user makes):
        H2D of `x_host` (pinned for an async copy), the stack, D2H."""
        torch = self.torch
        xt = x_host if isinstance(x_host, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x_host))
        if xt.dtype != self.tdtype:
            # the reference computes in the input's dtype (store.py:263-286): a silent cast
            # would change the arithmetic, so a mismatch is an error
            raise ShapeError(f"input dtype {xt.dtype} != the network's activation dtype {self.tdtype}")
        if tuple(xt.shape) != (self.batch, *self.in_shape):
            raise ShapeError(f"input {tuple(xt.shape)} != planned {(self.batch, *self.in_shape)}")
        with torch.cuda.device(self.device):
            self.x_in.copy_(xt, non_blocking=True)
            y = self.forward_device()
            if out_host is None:
                out_host = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            out_host.copy_(y, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
        return out_host if isinstance(x_host, torch.Tensor) else out_host.numpy()

    def forward_stream(self, x_hosts, out_hosts) -> None:
        """Streaming inference over many pinned host batches: the H2D copy of
        batch i+1 and the D2H copy of batch i-1 run on a copy stream while the
        stack computes batch i (two device input buffers).  Synchronous on return;
        every batch's copies and compute happen inside the call."""
        torch = self.torch
        if len(x_hosts) != len(out_hosts):
            raise ShapeError("one output buffer per input batch")
        with torch.cuda.device(self.device):
            comp = torch.cuda.current_stream(self.device)
            copy = getattr(self, "_copy_stream", None) or torch.cuda.Stream(self.device)
            self._copy_stream = copy
            if getattr(self, "_x2", None) is None or self._x2.shape != self.x_in.shape:
                self._x2 = torch.empty_like(self.x_in)
            bufs = (self.x_in, self._x2)
            loaded = [torch.cuda.Event() for _ in x_hosts]
            done = [torch.cuda.Event() for _ in x_hosts]
            freed = [torch.cuda.Event() for _ in x_hosts]
            with torch.cuda.stream(copy):
                bufs[0].copy_(x_hosts[0], non_blocking=True)
                loaded[0].record(copy)
            for i in range(len(x_hosts)):
                xb = bufs[i % 2]
                if i + 1 < len(x_hosts):
                    with torch.cuda.stream(copy):
                        if i >= 1:
                            copy.wait_event(freed[i - 1])  # batch i-1 no longer reads that buffer
                        bufs[(i + 1) % 2].copy_(x_hosts[i + 1], non_blocking=True)
                        loaded[i + 1].record(copy)
                comp.wait_event(loaded[i])
                self._run_stack(xb, comp, on_first=lambda st, ev=freed[i]: ev.record(st))
                cur = self.result
                done[i].record(comp)
                with torch.cuda.stream(copy):
                    copy.wait_event(done[i])
                    out_hosts[i].copy_(cur, non_blocking=True)
                # the next batch overwrites the activations only after this D2H read them
                comp.wait_stream(copy)
            copy.synchronize()
            comp.synchronize()


def build_net(specs_pools, seed: int = 0, dtype=np.float32, device: int = 0,
              weight_format: str = "native", fast_math: bool = False, weight_fn=None, values_fn=None):
    """SparseConvNet of synthetic unified-sparsity layers
    (synth.make_layer_weights / bench_inputs, bench.py:105-116,175-177).
    `weight_fn(w) -> w` post-processes each layer's dense weights (e.g. synth.codebook16);
    `values_fn(name, values) -> values` replaces each layer's CSR values (e.g. the
    reference quantizer, synth.reference_quantized_values_fn)."""
    from .synth import bench_inputs, make_layer_weights
    from .weights import build_csr
    layers = []
    for spec, pool in specs_pools:
        w = make_layer_weights(spec, seed).astype(dtype)
        if weight_fn is not None:
            w = weight_fn(w)
        _, b = bench_inputs(spec.shape, 1, seed)
        kern = build_csr(w, spec.shape)
        if values_fn is not None:
            from dataclasses import replace
            res = values_fn(spec.name, kern.values)
            vals, quant = res if isinstance(res, tuple) else (res, None)
            kern = replace(kern, values=np.ascontiguousarray(vals), _device_cache={}, quant=quant)
        layers.append(NetLayer(spec.name, kern, b, relu=True, pool=pool))
    return SparseConvNet(layers, device=device, dtype=dtype, weight_format=weight_format,
                         fast_math=fast_math)
