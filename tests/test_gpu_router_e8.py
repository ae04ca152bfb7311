"""GPU parity of the TMA-fed router for E <= 8 (csrc/router_e8.cu), taken for
bf16 tokens with T >= 148*64 and d % 256 == 0.  Bars: indices and counts
BIT-EXACT vs the CPU oracle (canonical order; ties -> lower index), routing
weights within 2e-6 (CUDA vs glibc expf), and the permutation built from them
bit-exact."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (test infrastructure)
from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.synthetic import make_router_weight, make_tie_batch, make_tokens  # noqa: E402

DEV = "cuda"


def _check(x, wg, k, mode):
    idx, w, counts = ops.router_topk(x, wg, k, mode)
    torch.cuda.synchronize()
    bits = x.view(torch.int16).cpu().numpy().view(np.uint16)
    oi, ow, oc = O.router_topk_bf16(bits, wg.float().cpu().numpy(), k, mode)
    gi = idx.cpu().numpy()
    bad = np.nonzero((gi != oi).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} tokens differ, first {bad[:5]}: gpu {gi[bad[:3]]} oracle {oi[bad[:3]]}"
    assert np.array_equal(counts.cpu().numpy(), oc)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("T,d,E,k,mode,wdt", [
    (148 * 64, 4096, 8, 2, 0, torch.bfloat16),       # exactly one tile per SM
    (148 * 64 * 3 + 37, 1024, 8, 2, 0, torch.bfloat16),  # ragged last tile (TMA zero fill)
    (20011, 6144, 8, 2, 1, torch.bfloat16),          # C3-sized rows, DeepSeek weights
    (12345, 2048, 6, 3, 0, torch.bfloat16),          # E < 8: padded router rows never win
    (10007, 512, 2, 1, 1, torch.float32),            # fp32 router weights in shared memory
    (9999, 4096, 8, 8, 0, torch.float32),            # k = E
])
def test_e8_router_bitexact(T, d, E, k, mode, wdt):
    x = make_tokens(T, d, seed=21, device=DEV)
    wg = make_router_weight(E, d, seed=22, device=DEV)
    if wdt == torch.float32:
        wg = wg + torch.rand_like(wg) * 1e-4  # not bf16-exact: the fp32 copy is routed
    _check(x, wg.to(wdt) if wdt == torch.bfloat16 else wg, k, mode)


def test_e8_router_near_ties():
    """Chunk-reverse-paired router rows and symmetric tokens: the pairs' logits
    are equal in real arithmetic and decided by fp32 rounding or by the
    lower-index rule (synthetic.make_tie_batch)."""
    x, wg, _ = make_tie_batch(40000, 2048, 8, seed=5, device=DEV, lead_k=1)
    _check(x, wg.to(torch.bfloat16), 2, 0)


def test_e8_router_nan_and_inf_tokens():
    """Non-finite logits rank like -inf (ties -> lower index), as in the oracle."""
    T, d = 148 * 64, 1024
    x = make_tokens(T, d, seed=23, device=DEV)
    x[5, :] = float("nan")
    x[77, 3] = float("inf")
    x[901, :8] = float("-inf")
    wg = make_router_weight(8, d, seed=24, device=DEV).to(torch.bfloat16)
    _check(x, wg, 2, 0)
