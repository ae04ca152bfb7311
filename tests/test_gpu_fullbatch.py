"""Full-batch, bit-exact routing: EVERY token of the BASELINE-sized batches.

The router's indices, the per-expert counts, and the permutation (offsets and
dst) of the CUDA path are compared with the CPU oracle (oracle/oracle_router.c,
OpenMP over tokens) for all 262,144 tokens of C2, C3L and C4 (C4 runs the
tensor-core screen + exact re-scoring router), on the very tokens and router
weights bench.py uses (seeds 1 and 0).  The adversarial "tie" batches make a
large share of the decisions depend on fp32 rounding alone (router rows
2m+1 = chunk_reverse(row 2m), chunk-reverse-symmetric tokens: the pair's logits are
equal in real arithmetic), so only a router that replays the canonical
summation order bit for bit passes them.  Semantics: PAPER.md:67 (top-k over
the expert pool), eas.py:364-374 (ties -> lower index).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (test infrastructure)
from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.synthetic import make_router_weight, make_tie_batch, make_tokens  # noqa: E402

DEV = "cuda"
T_FULL = 64 * 4096
# name: (d, E, k, mode) — bench.py's C2, C3L (C3/C5 layer) and C4 layers
CASES = {"C2": (4096, 8, 2, 0), "C3L": (6144, 8, 2, 0), "C4": (2048, 64, 6, 1)}


def _bits(x: torch.Tensor) -> np.ndarray:
    return x.view(torch.int16).cpu().numpy().view(np.uint16)


def _route_and_check(x, wg, k, mode, wtol):
    T, d = x.shape
    E = wg.shape[0]
    wgb = wg.to(torch.bfloat16)  # MoELayer routes with the bf16 copy (exact for these weights)
    assert torch.equal(wgb.float(), wg)
    idx, w, counts = ops.router_topk(x, wgb, k, mode)
    offsets = torch.empty((E + 1,), dtype=torch.int32, device=DEV)
    dst = torch.empty((T, k), dtype=torch.int32, device=DEV)
    ops.permute(idx, x, E, out=(offsets, dst, None))
    torch.cuda.synchronize()
    oi, ow, oc = O.router_topk_bf16(_bits(x), wg.cpu().numpy(), k, mode)
    gi = idx.cpu().numpy()
    bad = np.nonzero((gi != oi).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} of {T} tokens routed differently, first {bad[:5]}"
    assert np.array_equal(counts.cpu().numpy(), oc)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=wtol, atol=1e-7)
    oo, od = O.permute(oi, E, 1)
    assert np.array_equal(offsets.cpu().numpy(), oo)
    assert np.array_equal(dst.cpu().numpy(), od)
    return oi


@pytest.mark.parametrize("name", list(CASES))
def test_full_batch_routing_bitexact(name):
    d, E, k, mode = CASES[name]
    x = make_tokens(T_FULL, d, seed=1, device=DEV)
    wg = make_router_weight(E, d, seed=0, device=DEV)
    _route_and_check(x, wg, k, mode, 2e-6 if mode == 0 else 1e-5)


@pytest.mark.parametrize("name", list(CASES))
def test_full_batch_routing_bitexact_near_ties(name):
    d, E, k, mode = CASES[name]
    x, wg, pair = make_tie_batch(T_FULL, d, E, seed=3, device=DEV, lead_k=k - 1)
    oi = _route_and_check(x, wg, k, mode, 2e-6 if mode == 0 else 1e-5)
    # the adversarial tokens really are decided by rounding: count the tie tokens
    # whose pair is split by the selection or ordered inside it, and those whose
    # pair's fp32 logits are exactly equal (resolved by the lower-index rule)
    n = 16384
    lo = np.nonzero(pair[:n].cpu().numpy() >= 0)[0]
    _, _, _, lg = O.router_topk(x[:n].float().cpu().numpy(), wg.cpu().numpy(), k, mode, want_logits=True)
    p = pair[:n].cpu().numpy()[lo]
    a, b = lg[lo, 2 * p], lg[lo, 2 * p + 1]
    sel = oi[:n][lo]
    in_a = (sel == (2 * p)[:, None]).any(1)
    in_b = (sel == (2 * p + 1)[:, None]).any(1)
    split = int((in_a ^ in_b).sum())           # exactly one of the pair selected: membership at stake
    rounded = int(((a != b) & (in_a | in_b)).sum())   # fp32 values differ: rounding decides
    exact_ties = int(((a == b) & (in_a | in_b)).sum())  # fp32 values equal: lower index wins
    assert split > 500, split
    assert rounded > 300, rounded
    assert exact_ties > 300, exact_ties
