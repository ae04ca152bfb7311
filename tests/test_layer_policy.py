"""Host-side path selection of MoELayer (no GPU needed): which kernels a step of
T tokens runs, and the launch counts bench.py reports for it."""
import pytest
import torch

from paper_2605_17889_b200.layer import MoELayer
from paper_2605_17889_b200.synthetic import make_layer_weights


@pytest.fixture(scope="module")
def c4_layer():
    wts = make_layer_weights(64, 256, 128, seed=0, device="cpu", shared_ff=256)
    return MoELayer(wts, 6, "deepseek")


def test_small_path_needs_few_rows_per_expert():
    """Mixtral-shaped (E=8, k=2): the weight-streaming kernel only while an expert
    averages <= 32 rows (T <= 128); measured slower than the prefill kernels
    (M = 128 pair tiles) at 48."""
    wts = make_layer_weights(8, 256, 128, seed=0, device="cpu")
    L = MoELayer(wts, 2, "mixtral")
    assert L.uses_small_path(128) and not L.uses_small_path(129) and not L.uses_small_path(192)


def test_decode_path_selection(c4_layer):
    L = c4_layer
    # weight-streaming decode kernel up to SMALL_T_MAX tokens, prefill kernels above
    assert L.uses_small_path(1) and L.uses_small_path(256) and not L.uses_small_path(257)
    assert not L.uses_small_path(0)
    # dense single launch only where (almost) every expert is touched and T <= 48
    assert not L.uses_dense_decode(8)       # (1 - 6/64)^8 = 0.45 of the experts untouched
    assert L.uses_dense_decode(24) and L.uses_dense_decode(48)
    assert not L.uses_dense_decode(64)      # measured slower than the routed path
    assert L.launches_per_step(32) == 1
    assert L.launches_per_step(64) == 2  # router, then FFN + combine straight from the router's idx
    assert L.launches_per_step(65) == 1 + 2 + 1  # router, permute (index kernel + row copy), one FFN launch
    # prefill: router, permute (hist, scan, scatter, row copy), K3, K4, combine, shared x2
    assert L.launches_per_step(262144) == 1 + 3 + 1 + 2 + 1 + 2
    G = MoELayer(L.wts, L.k, L.mode_name, gather_a=True)
    assert G.launches_per_step(262144) == 1 + 3 + 2 + 1 + 2  # K3 gathers the rows: no copy launch


def test_dense_decode_needs_bf16_router_and_output():
    wts = make_layer_weights(8, 256, 128, seed=1, device="cpu")
    wts.wg = wts.wg + 1e-3  # no longer bf16-exact: the router keeps fp32 weights
    L = MoELayer(wts, 2, "mixtral")
    assert L.wg_router.dtype == torch.float32
    assert not L.uses_dense_decode(32) and L.uses_small_path(32)
    L2 = MoELayer(make_layer_weights(8, 256, 128, seed=1, device="cpu"), 2, "mixtral", out_dtype=torch.float32)
    assert not L2.uses_dense_decode(32)


def test_small_path_shape_limits():
    L = MoELayer(make_layer_weights(4, 192, 128, seed=2, device="cpu"), 2)  # d % 128 != 0
    assert not L.uses_small_path(8)
