"""GPU parity of the decode-size expert FFN (csrc/small_gemm.cu, cox_small_expert_ffn).

One weight-streaming launch computes K3 (SwiGLU) and K4 (down) of every
group, plus the shared experts: checked per expert against a torch fp32
reference (rel-L2 <= 1e-2, the bar of the prefill GEMMs), against the prefill
kernels on the same operands, and through MoELayer (which takes this path for
T <= SMALL_T_MAX) against the fp32 CPU oracle with routing bit-exact.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (test infrastructure)
from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens, split_w13  # noqa: E402

DEV = "cuda"


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _swiglu_ref(xe, w13e, w2e):
    w1, w3 = split_w13(w13e[None])
    h = torch.nn.functional.silu(xe @ w1[0].float().T) * (xe @ w3[0].float().T)
    return h, h.to(torch.bfloat16).float() @ w2e.float().T


@pytest.mark.parametrize("E,d,ff,counts,shared_ff", [
    (4, 256, 256, [0, 1, 16, 17], 0),
    (3, 512, 384, [64, 65, 150], 256),        # 65 and 150 rows: 64-row chunks
    (8, 1024, 512, [6, 0, 9, 3, 12, 5, 1, 30], 0),
    (64, 2048, 1408, None, 2816),             # C4 decode shape, T = 64 tokens x top-6
])
def test_small_ffn_vs_torch_fp32(E, d, ff, counts, shared_ff):
    if counts is None:
        counts = np.random.default_rng(0).multinomial(64 * 6, np.ones(E) / E).tolist()
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    rows = int(offs[-1])
    wts = make_layer_weights(E, d, ff, seed=3, device=DEV, shared_ff=shared_ff)
    x = make_tokens(max(rows, 1), d, seed=4, device=DEV)
    offs_t = torch.from_numpy(offs).to(DEV)
    h = torch.full((max(rows, 1), ff), 3.0, dtype=torch.bfloat16, device=DEV)
    y = torch.full((max(rows, 1), d), 3.0, dtype=torch.bfloat16, device=DEV)
    shared = None
    Ts = 40
    xs = make_tokens(Ts, d, seed=5, device=DEV)  # the step's tokens: shared-expert input
    if shared_ff:
        shared = (wts.shared_w13, wts.shared_w2, torch.empty((Ts, shared_ff), dtype=torch.bfloat16, device=DEV),
                  torch.empty((Ts, d), dtype=torch.bfloat16, device=DEV))
    ops.small_expert_ffn(xs, offs_t, list(range(E)), [wts.w13[e] for e in range(E)],
                         [wts.w2[e] for e in range(E)], h, y, x_perm=x, shared=shared)
    torch.cuda.synchronize()
    for e in range(E):
        r0, r1 = int(offs[e]), int(offs[e + 1])
        if r1 == r0:
            continue
        href, yref = _swiglu_ref(x[r0:r1].float(), wts.w13[e], wts.w2[e])
        assert rel_l2(h[r0:r1].float().cpu(), href.cpu()) < 1e-2, f"h expert {e}"
        assert rel_l2(y[r0:r1].float().cpu(), yref.cpu()) < 1e-2, f"y expert {e}"
    if rows == 0:
        assert (h == 3).all() and (y == 3).all()
    if shared_ff:
        href, yref = _swiglu_ref(xs.float(), wts.shared_w13, wts.shared_w2)
        assert rel_l2(shared[2].float().cpu(), href.cpu()) < 1e-2
        assert rel_l2(shared[3].float().cpu(), yref.cpu()) < 1e-2


def test_small_ffn_close_to_prefill_kernels():
    """Same operands through the prefill kernels (M=256 x N=256 tiles): the two
    paths differ only in fp32 summation order, so the bf16 outputs agree to a
    few bf16 ulps."""
    E, d, ff = 8, 1024, 1024
    counts = [5, 0, 33, 64, 70, 1, 9, 2]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    rows = int(offs[-1])
    wts = make_layer_weights(E, d, ff, seed=6, device=DEV)
    x = make_tokens(rows, d, seed=7, device=DEV)
    offs_t = torch.from_numpy(offs).to(DEV)
    g = list(range(E))
    w13 = [wts.w13[e] for e in g]
    w2 = [wts.w2[e] for e in g]
    h1 = ops.grouped_swiglu(x, offs_t, g, w13, ff)
    y1 = ops.grouped_down(h1, offs_t, g, w2, d)
    h2 = torch.empty_like(h1)
    y2 = torch.empty_like(y1)
    ops.small_expert_ffn(x, offs_t, g, w13, w2, h2, y2, x_perm=x)
    torch.cuda.synchronize()
    assert rel_l2(h2.float().cpu(), h1.float().cpu()) < 4e-3
    assert rel_l2(y2.float().cpu(), y1.float().cpu()) < 4e-3


@pytest.mark.parametrize("T,d,ff,E,k,mode,shared_ff", [
    (64, 2048, 1408, 64, 6, "deepseek", 2816),
    (200, 1024, 512, 16, 4, "deepseek", 256),
    (5, 512, 256, 8, 2, "mixtral", 0),
    (65, 1024, 512, 16, 4, "deepseek", 256),
    (256, 1024, 512, 16, 4, "deepseek", 256),
])
def test_decode_from_idx_matches_permute_path(T, d, ff, E, k, mode, shared_ff):
    """The expert launch that reads the router's idx/counts directly (no permute
    kernel, rows gathered from x) produces the permute's offsets and dst and the
    same output bits as router + permute (x_perm materialised) + tiled-B launch."""
    wts = make_layer_weights(E, d, ff, seed=9, device=DEV, shared_ff=shared_ff)
    x = make_tokens(T, d, seed=10, device=DEV)
    a_l = MoELayer(wts, k, mode)
    b_l = MoELayer(wts, k, mode)
    a_l.DENSE_T_MAX = b_l.DENSE_T_MAX = 0
    a_l.SMALL_ROWS_PER_EXPERT_MAX = b_l.SMALL_ROWS_PER_EXPERT_MAX = 1 << 30  # kernel equivalence at any rows/expert
    a_l.SMALL_GATHER_T_MAX = 256  # idx path at every T here
    b_l.SMALL_GATHER_T_MAX = 0    # router + permute + x_perm launch at every T
    assert a_l.uses_idx_decode(T) and not b_l.uses_idx_decode(T)
    assert a_l.launches_per_step(T) == 2 and b_l.launches_per_step(T) == 4
    a = a_l(x).clone()
    bo = b_l(x).clone()
    torch.cuda.synchronize()
    ba, bb = a_l.buffers(T, DEV), b_l.buffers(T, DEV)
    assert torch.equal(ba.idx, bb.idx)
    assert torch.equal(ba.offsets, bb.offsets)
    assert torch.equal(ba.dst, bb.dst)
    assert torch.equal(a, bo)


@pytest.mark.parametrize("seed", range(10))
def test_random_decode_configs_vs_oracle(seed):
    """Seeded random decode-size layers through MoELayer (whichever decode path
    it picks: routed from idx, dense single launch): routing bit-exact and
    rel-L2 <= 1e-2 against the fp32 oracle; skewed routing included."""
    rng = np.random.default_rng(2000 + seed)
    d = 128 * int(rng.integers(1, 9))
    ff = 128 * int(rng.integers(1, 6))
    E = int(rng.choice([2, 4, 8, 16, 32, 64]))
    k = int(rng.integers(1, min(E, 8) + 1))
    T = int(rng.integers(1, 257))
    mode = "mixtral" if rng.random() < 0.5 else "deepseek"
    sff = 128 * int(rng.integers(1, 4)) if rng.random() < 0.4 else 0
    wts = make_layer_weights(E, d, ff, seed=seed, device=DEV, shared_ff=sff, keep_split=True)
    x = make_tokens(T, d, seed=seed + 11, device=DEV).float()
    if rng.random() < 0.4:  # skew toward one expert
        x += 2.0 * d ** 0.5 * wts.wg[int(rng.integers(0, E))]
    x = x.to(torch.bfloat16)
    layer = MoELayer(wts, k, mode)
    layer.SMALL_ROWS_PER_EXPERT_MAX = 1 << 30  # exercise the weight-streaming kernel at any rows/expert
    assert layer.uses_small_path(T)
    out = layer(x)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    shared = (f(wts.shared_w1), f(wts.shared_w3), f(wts.shared_w2)) if sff else None
    ref = O.moe_layer(f(x), f(wts.wg), f(wts.w1), f(wts.w3), f(wts.w2), k, 0 if mode == "mixtral" else 1,
                      shared=shared)
    b = layer.buffers(T, DEV)
    assert np.array_equal(b.idx.cpu().numpy(), ref["idx"])
    if not layer.uses_dense_decode(T):
        assert np.array_equal(b.dst.cpu().numpy(), ref["dst"])
        assert np.array_equal(b.offsets.cpu().numpy(), ref["offsets"])
    assert rel_l2(f(out), ref["out"]) <= 1e-2


def test_captured_graph_survives_other_batch_sizes():
    """A CUDA graph captured at one batch size keeps its buffers (pinned per T):
    forwards at other batch sizes in between must not reallocate them, so the
    replay still produces the eager result (graph replay into freed
    memory)."""
    d, ff, E, k, sff = 1024, 512, 16, 4, 256
    wts = make_layer_weights(E, d, ff, seed=13, device=DEV, shared_ff=sff)
    layer = MoELayer(wts, k, "deepseek")
    xs = make_tokens(64, d, seed=14, device=DEV)
    replay, out = layer.capture(xs)
    for T in (200, 5000, 37, 3000):  # other paths and batch sizes, fresh allocations
        layer(make_tokens(T, d, seed=T, device=DEV))
    junk = [torch.full((1 << 20,), 7.0, device=DEV) for _ in range(64)]  # reuse freed blocks
    xs.copy_(make_tokens(64, d, seed=15, device=DEV))
    replay()
    torch.cuda.synchronize()
    ref = MoELayer(wts, k, "deepseek")(xs)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    del junk
