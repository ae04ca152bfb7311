"""cox_shared_down_combine (shared-expert down projection with the top-k combine
in its epilogue) == cox_grouped_down(shared) + cox_combine, bit for bit, and
the DeepSeek-style prefill layer that uses it == the oracle."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2605_17889_b200 import ops
from paper_2605_17889_b200.layer import MoELayer
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _unfused(h_s, offs, w2s, y, dst, w):
    ys = ops.grouped_down(h_s, offs, [0], [w2s], w2s.shape[0])
    return ops.combine(y, dst, w, ys[: dst.shape[0]])


@pytest.mark.parametrize("T,d,ffs,k,rows", [(1000, 512, 256, 6, 6400), (4096, 2048, 2816, 6, 24576),
                                            (257, 256, 128, 2, 600), (3000, 1024, 512, 8, 24000),
                                            (300, 768, 192, 1, 300)])
def test_fused_equals_separate(T, d, ffs, k, rows):
    g = torch.Generator(device=DEV).manual_seed(T + d + k)
    h_s = (torch.randn((T, ffs), device=DEV, generator=g) * 0.5).to(torch.bfloat16)
    w2s = (torch.randn((d, ffs), device=DEV, generator=g) / ffs ** 0.5).to(torch.bfloat16)
    y = torch.randn((rows, d), device=DEV, generator=g).to(torch.bfloat16)
    dst = torch.randint(0, rows, (T, k), device=DEV, generator=g, dtype=torch.int32)
    dst[::7, 0] = -1  # invalid expert id: no contribution (as cox_combine)
    w = torch.rand((T, k), device=DEV, generator=g)
    offs = torch.tensor([0, T], dtype=torch.int32, device=DEV)
    ref = _unfused(h_s, offs, w2s, y, dst, w)
    out = ops.shared_down_combine(h_s, offs, w2s, y, dst, w)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_layer_fused_vs_unfused_and_oracle():
    """T*k > SHARED_SIDE_MAX_ROWS: the prefill layer takes the fused path."""
    from oracle import oracle as O
    T, d, ff, E, k, sff = 3000, 512, 256, 16, 4, 512
    wts = make_layer_weights(E, d, ff, seed=3, device=DEV, shared_ff=sff, keep_split=True)
    x = make_tokens(T, d, seed=4, device=DEV)
    a = MoELayer(wts, k, "deepseek")
    a.SHARED_FUSED_COMBINE = True
    assert T * k > a.SHARED_SIDE_MAX_ROWS
    out_f = a(x).clone()
    b = MoELayer(wts, k, "deepseek")
    b.SHARED_FUSED_COMBINE = False
    out_u = b(x).clone()
    torch.cuda.synchronize()
    assert torch.equal(out_f, out_u)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    ref = O.moe_layer(f(x), f(wts.wg), f(wts.w1), f(wts.w3), f(wts.w2), k, 1,
                      shared=(f(wts.shared_w1), f(wts.shared_w3), f(wts.shared_w2)))
    got = f(out_f)
    err = np.linalg.norm(got - ref["out"]) / np.linalg.norm(ref["out"])
    assert err < 1e-2, err
    assert np.array_equal(a.buffers(T, DEV).idx.cpu().numpy(), ref["idx"])
