"""Layer-benchmark API (benchmark.py = the reference's bench_layer /
sparsity_sweep / emit_report, sc/bench.py:153-397): report layout and sweep
crossover on CPU, timed and checked layers on the GPU."""
import csv
import json

import numpy as np
import pytest

from paper_2011_06295_b200.benchmark import REPORT_COLUMNS, BenchRecord, crossover, emit_report


def _records():
    return [BenchRecord("conv3_2", "sparse-direct", "f32", 8, 0.167, 0.001, 0.168, 5, 100, 0.9, (1, 2, 8, 8, 8, 32, 2)),
            BenchRecord("conv3_2", "dense-cudnn", "f32", None, 0.2, 0.001, 0.2, 5, 1000, 0.9),
            BenchRecord("conv3_2", "dense-cudnn-tf32", "f32", None, 0.05, 0.001, 0.05, 5, 1000, 0.9),
            BenchRecord("conv3_2", "sparse-direct", "f16", 16, 0.12, 0.001, 0.12, 5, 100, 0.9),
            BenchRecord("conv3_2", "dense-cudnn", "f16", None, 0.04, 0.001, 0.04, 5, 1000, 0.9),
            BenchRecord("conv1_2", "sparse-direct", "f32", 1, 0.158, 0.001, 0.16, 5, 100, 0.95)]


def test_report_layout_matches_reference_columns(tmp_path):
    """Same columns and pivot as sc/bench.py:349-371: one row per (layer, sparsity%),
    dense = the IEEE dense baseline (TF32 is not an fp32 result and stays out)."""
    emit_report(_records(), "json", tmp_path / "r.json")
    rows = json.loads((tmp_path / "r.json").read_text())
    assert [r["layer"] for r in rows] == ["conv1_2", "conv3_2"]
    r = rows[1]
    assert r["sparsity"] == 90.0 and r["subBatchSize"] == 8
    assert r["sparse-f32"] == 0.167 and r["dense-f32"] == 0.2 and r["sparse-f16"] == 0.12 and r["dense-f16"] == 0.04
    assert rows[0]["dense-f32"] == "" and rows[0]["sparsity"] == 95.0
    emit_report(_records(), "csv", tmp_path / "r.csv")
    assert tuple(next(csv.reader(open(tmp_path / "r.csv")))) == REPORT_COLUMNS
    emit_report(_records(), "markdown", tmp_path / "r.md")
    assert (tmp_path / "r.md").read_text().splitlines()[0] == "| " + " | ".join(REPORT_COLUMNS) + " |"


def test_crossover_interpolation():
    sp = [0.5, 0.7, 0.9, 0.99]
    assert crossover(sp, [4.0, 3.0, 1.0, 0.5], 2.0) == pytest.approx(0.8)
    assert crossover(sp, [1.0, 0.9, 0.5, 0.1], 2.0) == 0.5
    assert crossover(sp, [9.0, 8.0, 7.0, 6.0], 2.0) is None


@pytest.mark.gpu
def test_bench_layer_and_sweep_on_gpu():
    """bench_layer times sparse + cuDNN (IEEE, TF32, f16) after checking them -- the
    sparse engine bit for bit against the oracle -- and sparsity_sweep reports the
    crossover against cuDNN IEEE fp32."""
    from oracle import oracle as orc

    import paper_2011_06295_b200 as sc
    from paper_2011_06295_b200.synth import LayerSpec

    def oracle_ref(x, kern, b):
        sh = kern.shape
        return orc.conv_sparse(x, kern.values, kern.colidx, kern.rowptr, sh.k, sh.r, sh.s, sh.stride, sh.padding, b)

    spec = LayerSpec("conv3_2", sc.ConvShape(n=1, c=256, h=8, w=8, k=256, r=3, s=3, padding=1), 0.9)
    recs = sc.bench_layer(spec, batch=32, tune=False, repetitions=3, warmups=1, reference_fn=oracle_ref)
    got = {(r.algorithm, r.dtype) for r in recs}
    assert got == {("sparse-direct", "f32"), ("dense-cudnn", "f32"), ("dense-cudnn-tf32", "f32"),
                   ("sparse-direct", "f16"), ("dense-cudnn", "f16")}
    assert all(r.median_ms > 0 for r in recs)
    sp = next(r for r in recs if r.algorithm == "sparse-direct" and r.dtype == "f32")
    assert sp.mac_count == 32 * 256 * 64 * 230  # N*K*E*F*L, L = 2304 - round(0.9*2304) (engine.py:131-136)
    # default checker: dense IEEE cuDNN at the reference tolerance
    assert sc.bench_layer(spec, batch=16, profiles=("f32",), tune=False, repetitions=2, warmups=1)
    sw = sc.sparsity_sweep(spec, [0.5, 0.9, 0.99], batch=64, repetitions=3, warmups=1, reference_fn=oracle_ref)
    assert len(sw.sparse_ms) == 3 and sw.dense_ms > 0 and sw.sparse_ms[0] > sw.sparse_ms[2]
    assert sw.crossover is None or 0.5 <= sw.crossover <= 0.99
