"""cox_decode_moe_routed (router in the expert kernel's prologue, one launch)
== router launch + cox_small_expert_ffn_idx, bit for bit (idx, w, counts, dst,
offsets, out), and == the oracle; repeated launches / graph replays reuse the
self-resetting histogram counters."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2605_17889_b200.layer import MoELayer
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _pair(E, d, ff, k, mode, sff, seed=0):
    wts = make_layer_weights(E, d, ff, seed=seed, device=DEV, shared_ff=sff, keep_split=True)
    a = MoELayer(wts, k, mode)
    a.DECODE_ROUTE_IN = True
    b = MoELayer(wts, k, mode)
    b.DECODE_ROUTE_IN = False
    b.DENSE_T_MAX = 0
    a.DENSE_T_MAX = 0
    a.SMALL_GATHER_T_MAX = b.SMALL_GATHER_T_MAX = 256  # the idx paths gather rows at every T here
    return wts, a, b


@pytest.mark.parametrize("T,d,ff,E,k,mode,sff", [
    (64, 2048, 1408, 64, 6, "deepseek", 2816),  # C4 decode shape
    (1, 512, 256, 8, 2, "mixtral", 0),
    (7, 256, 128, 16, 4, "deepseek", 256),
    (200, 512, 256, 32, 8, "mixtral", 0),
    (256, 1024, 384, 64, 6, "deepseek", 512),
    (33, 4096, 1024, 8, 2, "mixtral", 0),
])
def test_routed_one_launch_identical_to_two_launches(T, d, ff, E, k, mode, sff):
    wts, a, b = _pair(E, d, ff, k, mode, sff)
    assert a.uses_routed_one_launch(T) and not b.uses_routed_one_launch(T)
    x = make_tokens(T, d, seed=5, device=DEV)
    oa = a(x).clone()
    ob = b(x).clone()
    torch.cuda.synchronize()
    ba, bb = a.buffers(T, DEV), b.buffers(T, DEV)
    assert torch.equal(ba.idx, bb.idx)
    assert torch.equal(ba.w, bb.w)
    assert torch.equal(ba.counts[:E], bb.counts[:E])
    assert torch.equal(ba.dst, bb.dst)
    assert torch.equal(ba.offsets[:E + 1], bb.offsets[:E + 1])
    assert torch.equal(oa, ob)


@pytest.mark.parametrize("mode", ["mixtral", "deepseek"])
def test_routed_one_launch_vs_oracle_and_replays(mode):
    from oracle import oracle as O
    T, d, ff, E, k, sff = 48, 512, 256, 16, 4, (256 if mode == "deepseek" else 0)
    wts, a, _ = _pair(E, d, ff, k, mode, sff, seed=2)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    shared = (f(wts.shared_w1), f(wts.shared_w3), f(wts.shared_w2)) if sff else None
    x = make_tokens(T, d, seed=6, device=DEV)
    replay, out = a.capture(x)
    for s in range(3):  # fresh tokens each replay: counters must have been reset
        x.copy_(make_tokens(T, d, seed=10 + s, device=DEV))
        replay()
        torch.cuda.synchronize()
        ref = O.moe_layer(f(x), f(wts.wg), f(wts.w1), f(wts.w3), f(wts.w2), k, 0 if mode == "mixtral" else 1,
                          shared=shared)
        bb = a.buffers(T, DEV)
        assert np.array_equal(bb.idx.cpu().numpy(), ref["idx"])
        assert np.array_equal(bb.dst.cpu().numpy(), ref["dst"])
        assert np.array_equal(bb.offsets.cpu().numpy()[:E + 1], ref["offsets"][:E + 1])
        got = f(out)
        err = np.linalg.norm(got - ref["out"]) / np.linalg.norm(ref["out"])
        assert err < 1e-2, err


@pytest.mark.parametrize("route_in", [True, False])
def test_decode_routing_exact_ties_vs_oracle(route_in):
    """Duplicated router rows give exactly tied logits: the lower expert index
    wins, in the decode router kernel and the in-kernel (prologue) router."""
    from oracle import oracle as O
    T, d, ff, E, k = 64, 256, 128, 64, 6
    wts = make_layer_weights(E, d, ff, seed=7, device=DEV, keep_split=True)
    wg = wts.wg.clone()
    wg[1::2] = wg[0::2]  # experts 2i and 2i+1 tie on every token
    wg[60:] = 0.0        # logits exactly +0
    wts.wg = wg
    layer = MoELayer(wts, k, "deepseek")
    layer.DECODE_ROUTE_IN = route_in
    layer.DENSE_T_MAX = 0
    x = make_tokens(T, d, seed=8, device=DEV)
    out = layer(x)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    ref = O.moe_layer(f(x), f(wg), f(wts.w1), f(wts.w3), f(wts.w2), k, 1)
    b = layer.buffers(T, DEV)
    assert np.array_equal(b.idx.cpu().numpy(), ref["idx"])
    assert np.array_equal(b.w.cpu().numpy(), ref["w"]) or np.allclose(b.w.cpu().numpy(), ref["w"], rtol=1e-6)
    err = np.linalg.norm(f(out) - ref["out"]) / np.linalg.norm(ref["out"])
    assert err < 1e-2
