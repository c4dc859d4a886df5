"""Per-layer layout choice of the tuned network plan (network.py SparseConvNet._pick_layouts):
a two-state shortest path over the measured NCHW / image-minor kernel times plus the
estimated layout changes between consecutive layers.  Host logic only (CPU)."""
from paper_2011_06295_b200.network import SparseConvNet


class _Stub:
    _pick_layouts = SparseConvNet._pick_layouts

    def __init__(self, change):
        self.change = change

    def _layout_change_s(self, i):
        return 0.0 if i < 0 else self.change  # the stack input: free here


def _opts(times):
    return [(("n", i), tn, ("m", i) if tm is not None else None, tm if tm is not None else float("inf"))
            for i, (tn, tm) in enumerate(times)]


def test_free_changes_pick_the_faster_kernel_per_layer():
    got = _Stub(0.0)._pick_layouts(_opts([(1.0, 2.0), (3.0, 1.0), (1.0, None), (5.0, 4.0)]))
    assert got == [("n", 0), ("m", 1), ("n", 2), ("m", 3)]


def test_expensive_changes_keep_one_layout():
    # minor saves 0.5 on layer 1 but costs two changes of 1.0 each
    got = _Stub(1.0)._pick_layouts(_opts([(1.0, 1.2), (3.0, 2.5), (1.0, 1.1)]))
    assert got == [("n", 0), ("n", 1), ("n", 2)]


def test_a_slower_layer_joins_the_minor_run_to_save_a_change():
    # layer 0 is 0.1 slower image-minor, but staying minor saves the change (0.5) before layer 1
    got = _Stub(0.5)._pick_layouts(_opts([(1.0, 1.1), (5.0, 2.0), (1.0, 0.9)]))
    assert got == [("m", 0), ("m", 1), ("m", 2)]


def test_no_minor_kernels_anywhere():
    got = _Stub(0.0)._pick_layouts(_opts([(1.0, None), (2.0, None)]))
    assert got == [("n", 0), ("n", 1)]
