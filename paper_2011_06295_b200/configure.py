"""Per-layer algorithm choice for a network (the reference's NetworkConfig /
configure_network, sc/bench.py:281-342; the paper's Algorithm 2,
PAPER.md:274-287).

For every conv layer of a SparseConvNet the sparse engine (with its tuned
launch) and the dense cuDNN convolution are timed at the network's batch on
the GPU; the faster one is recorded, ties broken toward dense as in the
reference (bench.py:282).  The JSON layout keeps the reference's
``{"batch", "choices": {layer: {"algorithm", "sub_batch_size", "median_ms"}}}``
and adds the sparse launch.  ``SparseConvNet.apply_config`` installs a
config: layers set to "dense-cudnn" run torch/cuDNN convolutions (IEEE fp32,
TF32 off), everything else the sm_100a kernels.
"""
from __future__ import annotations

import json
import statistics
from dataclasses import dataclass, field
from pathlib import Path

ALGORITHMS = ("sparse-direct", "dense-cudnn")


@dataclass
class NetworkConfig:
    """Per-layer execution plan: algorithm = argmin of measured medians."""

    batch: int
    choices: dict = field(default_factory=dict)

    def to_json(self) -> str:
        return json.dumps({"batch": self.batch, "choices": self.choices}, indent=2, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "NetworkConfig":
        doc = json.loads(text)
        return cls(batch=doc["batch"], choices=doc["choices"])

    def save(self, path) -> None:
        Path(path).write_text(self.to_json())

    @classmethod
    def load(cls, path) -> "NetworkConfig":
        return cls.from_json(Path(path).read_text())


def _median_ms(fn, repetitions: int, warmups: int) -> float:
    import torch
    for _ in range(warmups):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(repetitions):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def configure_network(net, batch: int | None = None, repetitions: int = 5, warmups: int = 2,
                      tune: bool = True) -> NetworkConfig:
    """Time sparse vs dense per layer of `net` (a SparseConvNet) and return the
    NetworkConfig (the net is planned for `batch` if it is not already)."""
    import torch
    if batch is not None and net.batch != batch:
        net.plan(batch, tune=tune)
    elif net.batch is None:
        net.plan(batch or 32, tune=tune)
    config = NetworkConfig(batch=net.batch)
    stream = torch.cuda.current_stream(net.device).cuda_stream
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn((net.batch, *net.in_shape), generator=g).to(net.tdev, net.tdtype)
    with torch.cuda.device(net.device):
        for i, L in enumerate(net.layers):
            y = torch.empty(net.out_shape(i, net.batch), dtype=net.tdtype, device=net.tdev)
            t_sparse = _median_ms(lambda: net.launch_layer(i, x, y, stream), repetitions, warmups)
            dense = net.dense_layer(i)
            t_dense = _median_ms(lambda: dense(x), repetitions, warmups)
            chosen = "sparse-direct" if t_sparse < t_dense else "dense-cudnn"
            launch = net.launches[i]
            config.choices[L.name] = {
                "algorithm": chosen,
                "sub_batch_size": (launch[2] if launch is not None else 1) if chosen == "sparse-direct" else None,
                "launch": None if launch is None else list(launch),
                "median_ms": {"sparse-direct": round(t_sparse, 5), "dense-cudnn": round(t_dense, 5)},
            }
            x = torch.relu(torch.randn(net.out_shape(i, net.batch), generator=g)).to(net.tdev, net.tdtype)
    return config
