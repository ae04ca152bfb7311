"""Robustness of the routing kernels to non-finite activations and invalid ids.

A deep stack without normalisation can overflow (NaN/inf activations); the
router must still return valid, distinct expert ids (NaN logits rank below
every number, like -inf, in the oracle too) and the permute / combine kernels
must stay in bounds for invalid ids supplied through the C ABI."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (test infrastructure)
from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.synthetic import make_tokens  # noqa: E402

DEV = "cuda"


@pytest.mark.parametrize("T,d,E,k,mode", [
    (300, 512, 8, 2, 0),
    (300, 2048, 64, 6, 1),
    (148 * 128 + 5, 2048, 64, 6, 1),   # tensor-core screening path
    (40, 1024, 64, 6, 1),              # decode-size kernel
])
def test_router_nan_tokens_give_valid_ids(T, d, E, k, mode):
    x = make_tokens(T, d, seed=3, device=DEV)
    x[7] = float("nan")
    x[11, :5] = float("inf")
    x[13, 100] = float("-inf")
    g = torch.Generator(device=DEV).manual_seed(4)
    wg = ((torch.rand((E, d), generator=g, device=DEV) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    idx, w, counts = ops.router_topk(x, wg, k, mode)
    torch.cuda.synchronize()
    gi = idx.cpu().numpy()
    assert ((gi >= 0) & (gi < E)).all()
    assert all(len(set(r)) == k for r in gi)
    oi, _, oc = O.router_topk(x.float().cpu().numpy(), wg.float().cpu().numpy(), k, mode)
    assert np.array_equal(gi, oi)
    assert np.array_equal(counts.cpu().numpy(), oc)


def test_permute_and_combine_ignore_invalid_ids():
    T, d, E, k = 64, 256, 8, 2
    x = make_tokens(T, d, seed=5, device=DEV)
    idx = torch.stack([torch.arange(T) % E, (torch.arange(T) + 3) % E], 1).to(torch.int32).to(DEV)
    idx[5, 1] = -1
    idx[9, 0] = E
    offsets, dst, x_perm = ops.permute(idx, x, E)
    torch.cuda.synchronize()
    dd = dst.cpu().numpy()
    assert dd[5, 1] == -1 and dd[9, 0] == -1
    valid = dd[dd >= 0]
    assert sorted(valid.tolist()) == list(range(T * k - 2))
    assert int(offsets[-1]) == T * k - 2
    y = torch.randn((x_perm.shape[0], d), device=DEV).to(torch.bfloat16)
    w = torch.full((T, k), 0.5, device=DEV)
    out = ops.combine(y, dst, w)
    torch.cuda.synchronize()
    ref = 0.5 * y[dst[5, 0].long()].float()
    assert torch.allclose(out[5].float(), ref, atol=1e-2)
