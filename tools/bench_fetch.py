"""PCIe rate of the device-side cold-expert fetch (cox_fetch_experts: SM loads
of mapped pinned host memory) against copy-engine cudaMemcpyAsync, for C3-sized
experts (604 MB: W13 + W2).  Run under gpurun."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2605_17889_b200 import ops  # noqa: E402


def main():
    d, ff, n = 6144, 16384, 4
    host = [torch.empty((2 * ff * d,), dtype=torch.bfloat16).pin_memory() for _ in range(n)]
    host2 = [torch.empty((d * ff,), dtype=torch.bfloat16).pin_memory() for _ in range(n)]
    dev = [torch.empty_like(h, device="cuda") for h in host]
    dev2 = [torch.empty_like(h, device="cuda") for h in host2]
    counts = torch.ones((8,), dtype=torch.int32, device="cuda")
    nbytes = sum(h.numel() * 2 for h in host + host2)
    for ctas in (32, 74, 148, 296):
        for rep in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ops.fetch_experts(counts, [i for i in range(n)] * 2, host + host2, dev + dev2, max_ctas=ctas)
            b.record()
            torch.cuda.synchronize()
        print(f"fetch kernel {ctas:3d} CTAs: {nbytes / (a.elapsed_time(b) / 1e3) / 1e9:6.1f} GB/s", flush=True)
    counts.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ops.fetch_experts(counts, [i for i in range(n)] * 2, host + host2, dev + dev2)
    b.record()
    torch.cuda.synchronize()
    print(f"fetch kernel, all untouched: {a.elapsed_time(b) * 1e3:.1f} us", flush=True)
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for h, dd in zip(host + host2, dev + dev2):
            dd.copy_(h, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
    print(f"copy engine (cudaMemcpyAsync): {nbytes / (a.elapsed_time(b) / 1e3) / 1e9:6.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
