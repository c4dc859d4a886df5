"""Per-layer times of the VGG-CIFAR stack at a small per-GPU shard (the 8-GPU proxy):
tuned plan at --batch, one chain, CUDA events between layers (median of --reps passes).
Usage: python tools/probe_shard.py [--batch 32]"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2011_06295_b200 import engine  # noqa: E402
from paper_2011_06295_b200.network import build_net  # noqa: E402
from paper_2011_06295_b200.synth import vgg16_cifar  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
net = build_net(vgg16_cifar(0.9))
net.plan(a.batch, tune=True)
x = torch.randn((a.batch, 3, 32, 32), device="cuda")
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(net.layers) + 1)]
per = [[] for _ in net.layers]
for _ in range(a.reps):
    net.forward_device(x, events=evs)
    evs[-1].synchronize()
    for i in range(len(net.layers)):
        per[i].append(evs[i].elapsed_time(evs[i + 1]) * 1e3)
rows = [{"layer": L.name, "us": round(statistics.median(t), 2), "kind": engine.launch_kind(l), "launch": l}
        for L, t, l in zip(net.layers, per, net.launches)]
print(json.dumps({"batch": a.batch, "sum_us": round(sum(r["us"] for r in rows), 1), "layers": rows}))
# whole-step time: eager launches vs one CUDA graph replay (launch overhead at small shards)
for graph in (False, True):
    if graph:
        net.capture()
    for _ in range(5):
        net.forward_device(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(a_reps := 50):
        net.forward_device(x)
    b.record()
    b.synchronize()
    print(json.dumps({"batch": int(x.shape[0]),
                      "cuda_graph": graph, "ms_per_step": round(a.elapsed_time(b) / a_reps, 4)}))
