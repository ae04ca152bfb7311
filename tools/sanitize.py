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
    # tensor-core screening router (E >= 32, T >= 148*128)
    wg64 = (torch.rand(64, 256, device=dev) * 2 - 1).to(torch.bfloat16) / 16
    ops.router_topk(make_tokens(148 * 128 + 9, 256, device=dev), wg64, 6, 1)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
