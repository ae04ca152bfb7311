"""K3 with the permuted rows gathered from x by cp.async (cox_grouped_swiglu_gather):
h must be bit-identical to K3 on the materialised x_perm (same A bits, same MMA
order), for ragged segments incl. empty experts and partial 256-row tiles, and a
layer running the gather path must equal the x_perm path bit for bit."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

DEV = "cuda"


def _route(T, d, E, k, mode, seed):
    wts = make_layer_weights(E, d, 256, seed=seed, device=DEV)
    x = make_tokens(T, d, seed=seed + 1, device=DEV)
    idx, w, counts = ops.router_topk(x, wts.wg, k, mode)
    return x, idx, counts


@pytest.mark.parametrize("T,d,ff,E,k,mode", [
    (3000, 512, 256, 8, 2, 0),
    (2500, 2048, 1408, 64, 6, 1),     # C4 shapes (64 groups, many partial tiles)
    (700, 1024, 512, 16, 4, 1),
    (5000, 4096, 384, 8, 2, 0),       # C2 d (K = 4096: 32 stages of the ring)
])
def test_gather_swiglu_bitexact_vs_x_perm(T, d, ff, E, k, mode):
    x, idx, _ = _route(T, d, E, k, mode, seed=11)
    wts = make_layer_weights(E, d, ff, seed=5, device=DEV)
    w13 = [wts.w13[e] for e in range(E)]
    offs, dst, x_perm = ops.permute(idx, x, E)
    cap = x_perm.shape[0]
    rt = torch.full((cap,), -1, dtype=torch.int32, device=DEV)
    offs2, dst2, _ = ops.permute(idx, x, E, copy_rows=False, row_tokens=rt)
    assert torch.equal(offs, offs2) and torch.equal(dst, dst2)
    rows = int(offs[-1].item())
    assert torch.equal(x_perm[:rows], x[rt[:rows].long()])
    h_ref = ops.grouped_swiglu(x_perm, offs, list(range(E)), w13, ff)
    h_g = torch.full_like(h_ref, 3.0)
    ops.grouped_swiglu_gather(x, rt, offs, list(range(E)), w13, ff, h_g)
    torch.cuda.synchronize()
    assert torch.equal(h_g[:rows], h_ref[:rows])


def test_gather_subset_groups_and_empty_experts():
    T, d, ff, E, k = 1500, 512, 256, 8, 2
    x = make_tokens(T, d, seed=4, device=DEV)
    # k distinct experts per token (top-k never repeats one), none of them expert 5
    g = torch.Generator().manual_seed(0)
    pool = torch.tensor([0, 1, 2, 3, 4, 6, 7])
    idx = torch.stack([pool[torch.randperm(7, generator=g)[:k]] for _ in range(T)]).to(torch.int32).to(DEV)
    wts = make_layer_weights(E, d, ff, seed=9, device=DEV)
    rt = torch.empty((T * k,), dtype=torch.int32, device=DEV)
    offs, dst, x_perm = ops.permute(idx, x, E, row_tokens=rt)
    assert int((offs[6] - offs[5]).item()) == 0
    groups = [1, 5, 6]
    h_ref = torch.full((T * k, ff), 7.0, dtype=torch.bfloat16, device=DEV)
    h_g = h_ref.clone()
    ops.grouped_swiglu(x_perm, offs, groups, [wts.w13[g] for g in groups], ff, h=h_ref)
    ops.grouped_swiglu_gather(x, rt, offs, groups, [wts.w13[g] for g in groups], ff, h_g)
    torch.cuda.synchronize()
    assert torch.equal(h_g, h_ref)   # same rows written, the rest untouched (7.0)


@pytest.mark.parametrize("T,d,ff,E,k,mode,shared_ff", [
    (20000, 1024, 512, 8, 2, "mixtral", 0),
    (9000, 2048, 1408, 64, 6, "deepseek", 2816),
])
def test_layer_gather_equals_x_perm_path(T, d, ff, E, k, mode, shared_ff):
    wts = make_layer_weights(E, d, ff, seed=0, device=DEV, shared_ff=shared_ff)
    x = make_tokens(T, d, seed=1, device=DEV)
    a = MoELayer(wts, k, mode, gather_a=False)(x).clone()
    b = MoELayer(wts, k, mode, gather_a=True)(x)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
