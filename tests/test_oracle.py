"""CPU oracle vs golden vectors (no GPU).  Pins the oracle before it is trusted:
  * canonical fp32 router order: bit-exact against an exact-rational replay;
  * top-k indices: against float64 + exact-replay goldens (C2 and C4 shapes);
  * whole expert stage: against float64 numpy on small ragged cases;
  * permutation / combine properties the reference's conventions imply."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import oracle as O
from tests.golden.inputs import ROUTING_CASES, layer_micro_inputs, routing_inputs

GOLD = __import__("pathlib").Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", sorted(ROUTING_CASES))
def test_canonical_logits_bitexact(name):
    g = np.load(GOLD / f"routing_{name}.npz")
    x, wg, k = routing_inputs(name)
    near = g["near"]
    _, _, _, lg = O.router_topk(x[near], wg, k, want_logits=True)
    ex = g["exact_logits"]
    mask = ~np.isnan(ex)
    assert mask.sum() > 100
    assert np.array_equal(lg[mask].view(np.uint32), ex[mask].view(np.uint32))


@pytest.mark.parametrize("name", sorted(ROUTING_CASES))
def test_topk_indices_match_golden(name):
    g = np.load(GOLD / f"routing_{name}.npz")
    x, wg, k = routing_inputs(name)
    idx, w, counts = O.router_topk(x, wg, k, mode=0 if "mixtral" in name else 1)
    assert np.array_equal(idx, g["idx"].astype(np.int32))
    assert np.array_equal(counts, np.bincount(idx.ravel(), minlength=wg.shape[0]))


@pytest.mark.parametrize("case", ["a", "b", "c"])
def test_layer_micro_vs_float64(case):
    g = np.load(GOLD / "layer_micro.npz")
    x, wg, w1, w3, w2, k, mode = layer_micro_inputs()[case]
    r = O.moe_layer(x, wg, w1, w3, w2, k, mode)
    assert np.array_equal(r["idx"], g[f"{case}_idx"])
    assert np.array_equal(r["counts"], g[f"{case}_counts"])
    np.testing.assert_allclose(r["w"], g[f"{case}_w"], rtol=1e-6, atol=1e-7)
    ref = g[f"{case}_out"]
    assert np.linalg.norm(r["out"] - ref) / np.linalg.norm(ref) < 1e-5
    if case == "b":
        assert r["counts"][3] == 0  # empty expert handled


def test_tie_goes_to_lower_index():
    x = np.ones((3, 16), np.float32)
    wg = np.zeros((6, 16), np.float32)
    wg[2] = wg[4] = 0.5
    idx, w, _ = O.router_topk(x, wg, 2)
    assert (idx == [2, 4]).all()
    np.testing.assert_allclose(w, 0.5)
    idx, _, _ = O.router_topk(x, np.zeros((6, 16), np.float32), 3)
    assert (idx == [0, 1, 2]).all()


@settings(max_examples=60, deadline=None)
@given(T=st.integers(0, 60), E=st.integers(1, 12), k=st.integers(1, 4), tile=st.sampled_from([1, 2, 8, 128]),
       seed=st.integers(0, 2**31 - 1))
def test_permute_properties(T, E, k, tile, seed):
    k = min(k, E)
    rng = np.random.default_rng(seed)
    idx = np.array([rng.choice(E, size=k, replace=False) for _ in range(T)], dtype=np.int32).reshape(T, k)
    offsets, dst = O.permute(idx, E, tile)
    counts = np.bincount(idx.ravel(), minlength=E)
    seg = np.diff(offsets)
    assert (seg % tile == 0).all() and (seg >= counts).all() and (seg - counts < tile).all()
    flat = dst.ravel()
    assert len(set(flat.tolist())) == flat.size  # a permutation into distinct rows
    for e in range(E):  # stable: expert e's rows in ascending token order, contiguous from offsets[e]
        rows = dst[idx == e]
        toks = np.nonzero((idx == e).any(axis=1))[0]
        assert np.array_equal(np.sort(rows), offsets[e] + np.arange(len(toks)))
        assert np.array_equal(dst[toks][idx[toks] == e], offsets[e] + np.arange(len(toks)))


def test_combine_fixed_order_and_shared():
    rng = np.random.default_rng(0)
    y = rng.standard_normal((10, 16)).astype(np.float32)
    dst = np.array([[0, 5], [9, 1], [2, 3]], np.int32)
    w = rng.random((3, 2)).astype(np.float32)
    sh = rng.standard_normal((3, 16)).astype(np.float32)
    out = O.combine(y, dst, w, sh)
    exp = np.zeros((3, 16), np.float32)
    for t in range(3):
        acc = np.zeros(16, np.float32)
        for j in range(2):
            acc = (acc + np.float32(w[t, j]) * y[dst[t, j]]).astype(np.float32)
        exp[t] = acc + sh[t]
    assert np.array_equal(out, exp)


def test_oracle_rejects_bad_shapes():
    with pytest.raises(ValueError):
        O.router_topk(np.zeros((2, 12), np.float32), np.zeros((4, 12), np.float32), 2)  # d % 8
    with pytest.raises(ValueError):
        O.router_topk(np.zeros((2, 16), np.float32), np.zeros((4, 16), np.float32), 5)  # k > E
