"""Model-store loader vs the reference: the fixture in tests/golden/store_small
was written by the reference's save_model and its expected arrays by the
reference's load_model + conv_sparse (tests/golden/make_store.py)."""
import json
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

STORE = GOLDEN / "store_small"


def _expected():
    return np.load(GOLDEN / "store_small_expected.npz")


def test_fnv1a64_known_answers():
    from paper_2011_06295_b200.store import fnv1a64
    assert fnv1a64(b"") == 0xCBF29CE484222325
    assert fnv1a64(b"a") == 0xAF63DC4C8601EC8C  # standard FNV-1a 64 test vector
    assert fnv1a64(b"foobar") == 0x85944171F73967E8


def test_loaded_kernels_match_reference_load():
    from paper_2011_06295_b200.store import load_conv_layers
    exp = _expected()
    layers = load_conv_layers(STORE)
    assert [L.name for L in layers] == ["conv0", "conv1", "conv2"]
    for L in layers:
        assert np.array_equal(L.kernel.values.view(np.uint32), exp[f"{L.name}.values"].view(np.uint32))
        assert np.array_equal(L.kernel.colidx, exp[f"{L.name}.colidx"])
        assert np.array_equal(L.kernel.rowptr, exp[f"{L.name}.rowptr"])
        assert np.array_equal(L.bias, exp[f"{L.name}.bias"])
    assert not layers[2].kernel.unified


def test_corrupt_blob_rejected(tmp_path):
    from paper_2011_06295_b200.errors import FormatError
    from paper_2011_06295_b200.store import load_conv_layers
    d = tmp_path / "m"
    shutil.copytree(STORE, d)
    b = bytearray((d / "conv0.values.bin").read_bytes())
    b[70] ^= 0x1
    (d / "conv0.values.bin").write_bytes(bytes(b))
    with pytest.raises(FormatError, match="checksum"):
        load_conv_layers(d)
    shutil.copytree(STORE, tmp_path / "v")
    m = json.loads((tmp_path / "v" / "manifest.json").read_text())
    m["format_version"] = 2
    (tmp_path / "v" / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(FormatError, match="version"):
        load_conv_layers(tmp_path / "v")


@pytest.mark.gpu
def test_loaded_net_forward_bitwise():
    from paper_2011_06295_b200.store import load_net
    exp = _expected()
    net = load_net(STORE)
    net.plan(exp["x"].shape[0], tune=False)
    out = net.forward(exp["x"])
    assert np.array_equal(out.view(np.uint32), exp["conv_out"].view(np.uint32))
    # the same weights re-encoded as 4-bit codebook indices (the stored codebook has 16 entries)
    net16 = load_net(STORE, weight_format="cb4")
    net16.plan(exp["x"].shape[0], tune=False)
    assert np.array_equal(net16.forward(exp["x"]).view(np.uint32), exp["conv_out"].view(np.uint32))


STORE_AQ = GOLDEN / "store_aq"


def test_act_quant_loaded_from_manifest():
    """Layers carry the manifest's act_quant (quantize.py:324-326, store.py:339,411)."""
    from paper_2011_06295_b200.store import load_conv_layers
    layers = load_conv_layers(STORE_AQ)
    m = json.loads((STORE_AQ / "manifest.json").read_text())
    want = {r["name"]: r.get("act_quant") for r in m["layers"] if r["type"] == "conv"}
    assert [L.name for L in layers] == list(want)
    for L in layers:
        assert L.act_quant == want[L.name] and L.act_quant["bits"] == 8


@pytest.mark.gpu
def test_act_quant_net_forward_bitwise():
    """Model.forward with activation quantizers (conv -> ReLU -> fake_quant per layer,
    store.py:276-286): fused epilogue, generic kernel + fake-quant pass, bit-identical
    to the reference's own output."""
    from paper_2011_06295_b200.store import load_net
    exp = np.load(GOLDEN / "store_aq_expected.npz")
    net = load_net(STORE_AQ)
    net.plan(exp["x"].shape[0], tune=False)
    out = net.forward(exp["x"])
    assert np.array_equal(out.view(np.uint32), exp["conv_out"].view(np.uint32))
    net.set_launches([None] * len(net.layers))  # generic kernels: separate fake-quant pass
    assert np.array_equal(net.forward(exp["x"]).view(np.uint32), exp["conv_out"].view(np.uint32))


@pytest.mark.gpu
def test_loaded_net_refuses_other_input_dtype():
    """the device net has a fixed activation dtype; an input of another dtype is
    refused instead of silently cast (the reference computes in the input's dtype)."""
    from paper_2011_06295_b200.errors import ShapeError
    from paper_2011_06295_b200.store import load_net
    exp = _expected()
    net = load_net(STORE, dtype=np.float32)
    net.plan(exp["x"].shape[0], tune=False)
    with pytest.raises(ShapeError, match="dtype"):
        net.forward(exp["x"].astype(np.float64))
