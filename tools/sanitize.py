"""Small-shape run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for (T, d, ff, E, k, mode, shared) in [(300, 256, 256, 8, 2, "mixtral", 0), (97, 512, 128, 16, 6, "deepseek", 256),
                                           (5000, 256, 128, 64, 6, "deepseek", 0)]:
        wts = make_layer_weights(E, d, ff, seed=0, device=dev, shared_ff=shared)
        x = make_tokens(T, d, seed=1, device=dev)
        out = MoELayer(wts, k, mode)(x)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
    # small-T router paths (fp32 input, 1-token warp tiles) and the staged router (E > 8, T >= 148*32)
    from paper_2605_17889_b200 import ops
    wg = torch.randn(64, 256, device=dev) / 16
    ops.router_topk(make_tokens(5000, 256, device=dev), wg, 6, 1)
    ops.router_topk(make_tokens(33, 256, device=dev, dtype=torch.float32), wg[:8].contiguous(), 2, 0)
    torch.cuda.synchronize()
    # decode-size paths: routed weight-streaming launch straight from idx (T=64,
    # E=64), the dense single launch (T=40, E=16), and the x_perm / row-gather
    # variants of cox_small_expert_ffn
    for (T, d, ff, E, k, mode, shared) in [(64, 256, 128, 64, 6, "deepseek", 256), (40, 256, 128, 16, 4, "deepseek", 128),
                                           (150, 256, 128, 8, 2, "mixtral", 0)]:
        wts = make_layer_weights(E, d, ff, seed=2, device=dev, shared_ff=shared)
        x = make_tokens(T, d, seed=3, device=dev)
        layer = MoELayer(wts, k, mode)
        out = layer(x)
        layer.SMALL_GATHER_T_MAX = 0  # router + permute + x_perm launch
        out2 = layer(x)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all() and torch.isfinite(out2.float()).all()
    # split-expert decode router (T <= 64, E = 64 / 8 / 160) with one workspace reused
    for E in (64, 8, 160):
        wgd = (torch.rand(E, 512, device=dev) * 2 - 1).to(torch.bfloat16) / 16
        ws = ops.router_workspace(37, E, dev)
        for _ in range(2):
            ops.router_topk(make_tokens(37, 512, device=dev), wgd, 6, 1, workspace=ws)
    torch.cuda.synchronize()
    # prefill layer with shared experts on the side stream
    wts = make_layer_weights(16, 256, 128, seed=6, device=dev, shared_ff=256)
    layer = MoELayer(wts, 4, "deepseek")
    out = layer(make_tokens(3000, 256, seed=7, device=dev))
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    # TMA-fed E <= 8 router (T >= 148*64, d % 256 == 0) with bf16 and fp32 router rows
    from paper_2605_17889_b200.synthetic import make_router_weight
    wg8 = make_router_weight(8, 512, seed=3, device=dev)
    ops.router_topk(make_tokens(148 * 64 + 5, 512, device=dev), wg8.to(torch.bfloat16), 2, 0)
    ops.router_topk(make_tokens(148 * 64 + 5, 512, device=dev), wg8 + 1e-4, 2, 1)
    # device-side cold-expert fetch (touched / untouched entries)
    host = [torch.randn(4096 + 8 * i).to(torch.bfloat16).pin_memory() for i in range(4)]
    dst = [torch.empty_like(h, device=dev) for h in host]
    counts = torch.tensor([1, 0, 3, 0], dtype=torch.int32, device=dev)
    fetched = torch.empty(4, dtype=torch.int32, device=dev)
    ops.fetch_experts(counts, [0, 1, 2, 3], host, dst, fetched=fetched)
    torch.cuda.synchronize()
    assert torch.equal(dst[2].cpu(), host[2]) and fetched.tolist() == [1, 0, 1, 0]
    # stratified stack: streamed and touched-only cold experts
    from paper_2605_17889_b200.config import ResidencyPlan
    from paper_2605_17889_b200.executor import StratifiedMoEStack, make_pool, make_router_weights
    st = StratifiedMoEStack(3, make_router_weights(3, 8, 256, device=dev), make_pool(5, 256, 256, device=dev), 2,
                            ResidencyPlan(tuple((0, 1) for _ in range(3)), 2))
    xs = make_tokens(200, 256, seed=8, device=dev)
    st(xs, fetch="stream")
    st(xs, fetch="touched")
    torch.cuda.synchronize()
    # tensor-core screening router (E >= 32, T >= 148*128)
    wg64 = (torch.rand(64, 256, device=dev) * 2 - 1).to(torch.bfloat16) / 16
    ops.router_topk(make_tokens(148 * 128 + 9, 256, device=dev), wg64, 6, 1)
    torch.cuda.synchronize()
    # K3 gather mode (A rows by cp.async from x), incl. partial tiles and shared experts
    for (T, d, ff, E, k, mode, shared) in [(3000, 256, 128, 8, 2, "mixtral", 0), (2500, 512, 256, 16, 4, "deepseek", 256)]:
        wts = make_layer_weights(E, d, ff, seed=4, device=dev, shared_ff=shared)
        x = make_tokens(T, d, seed=5, device=dev)
        a = MoELayer(wts, k, mode, gather_a=True)(x)
        b = MoELayer(wts, k, mode, gather_a=False)(x)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    print("sanitize run ok")


if __name__ == "__main__":
    main()
