"""GPU parity of the tensor-core screening router (csrc/router_tc.cu).

Batches of >= 148*128 tokens with bf16 x and router weights and E >= 32
experts take the tcgen05 screen + exact canonical re-scoring path.  Bars (same as the CUDA-core
router): indices and counts BIT-EXACT vs the CPU oracle; Mixtral-mode weights
within 2e-6 (expf of CUDA vs glibc); DeepSeek-mode weights within 1e-5 (the
full-softmax denominator uses tensor-core logits for the experts outside the
candidate set).  Near-tie stress: duplicated and 1-ulp-perturbed router rows.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (test infrastructure)
from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.synthetic import make_tokens  # noqa: E402

DEV = "cuda"
T_TC = 148 * 128 + 77  # above the screening threshold, ragged last tile


def _wg(E, d, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return ((torch.rand((E, d), generator=g, device=DEV) * 2 - 1) / d ** 0.5).to(torch.bfloat16)


def _check(x, wg, k, mode, wtol):
    idx, w, counts = ops.router_topk(x, wg, k, mode)
    torch.cuda.synchronize()
    oi, ow, oc = O.router_topk(x.float().cpu().numpy(), wg.float().cpu().numpy(), k, mode)
    gi = idx.cpu().numpy()
    bad = np.nonzero((gi != oi).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} tokens differ, first {bad[:5]}: gpu {gi[bad[:3]]} oracle {oi[bad[:3]]}"
    assert np.array_equal(counts.cpu().numpy(), oc)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=wtol, atol=1e-7)


@pytest.mark.parametrize("d,E,k,mode", [
    (2048, 64, 6, 1),    # C4 shape (DeepSeek softmax)
    (2048, 64, 6, 0),
    (4096, 40, 2, 0),    # E not a multiple of 16, C2-sized rows
    (1024, 36, 3, 1),
    (512, 160, 8, 0),
    (1024, 96, 4, 1),    # the screen's largest ring footprint (E in (80, 96])
    (768, 256, 8, 1),    # widest E: 32-column router tiles, 4-stage ring
    (4096, 32, 2, 1),    # narrowest E: 8-stage ring, NCH = 16 re-score
])
def test_tc_router_bitexact_indices(d, E, k, mode):
    x = make_tokens(T_TC, d, seed=11, device=DEV)
    _check(x, _wg(E, d, 12), k, mode, 2e-6 if mode == 0 else 1e-5)


def test_tc_router_near_ties():
    """Rows that are exact duplicates (ties -> lower index) and rows that differ
    in one element by one bf16 ulp: the logits differ by far less than the
    tensor-core error, so only the exact re-scoring can order them."""
    d, E, k = 2048, 64, 6
    wg = _wg(E, d, 13)
    wg[5] = wg[9]                          # exact duplicate
    wg[17] = wg[3]
    v = wg[3, 100].float()
    wg[17, 100] = (v * (1 + 2 ** -7)).to(torch.bfloat16)   # one ulp-ish apart in one element
    wg[40] = wg[41]
    x = make_tokens(T_TC, d, seed=14, device=DEV)
    # bias tokens towards the tied rows so that they are often in the top-k
    x += 0.05 * (wg[9] + wg[3] + wg[41]).float().to(torch.bfloat16) * d ** 0.5
    x = x.to(torch.bfloat16)
    _check(x, wg, k, 1, 1e-5)
    _check(x, wg, k, 0, 2e-6)


def test_tc_router_matches_cuda_core_router(monkeypatch):
    """Same indices and (Mixtral) bit-identical weights as the all-CUDA-core
    kernels, which are selected below the screening threshold: compare the
    first 4096 tokens routed inside a large batch with the same tokens routed
    alone."""
    d, E, k = 4096, 32, 2
    wg = _wg(E, d, 15)
    x = make_tokens(T_TC, d, seed=16, device=DEV)
    idx_big, w_big, _ = ops.router_topk(x, wg, k, 0)
    idx_small, w_small, _ = ops.router_topk(x[:4096].contiguous(), wg, k, 0)
    torch.cuda.synchronize()
    assert torch.equal(idx_big[:4096], idx_small)
    assert torch.equal(w_big[:4096], w_small)


@pytest.mark.parametrize("seed", range(6))
def test_tc_router_random_configs(seed):
    rng = np.random.default_rng(3000 + seed)
    d = 64 * int(rng.integers(2, 49))        # 128 .. 3072
    E = int(rng.integers(32, 257))
    k = int(rng.integers(1, 9))
    mode = int(rng.integers(0, 2))
    x = make_tokens(T_TC, d, seed=seed + 20, device=DEV)
    if rng.random() < 0.5:  # skewed, near-tie-rich routing: scaled-down tokens
        x = (x.float() * 0.05).to(torch.bfloat16)
    _check(x, _wg(E, d, seed + 30), k, mode, 2e-6 if mode == 0 else 1e-5)
