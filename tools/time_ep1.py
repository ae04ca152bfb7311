"""Time MoELayer vs FusedEPMoELayer vs EPMoELayer (NCCL) at world size 1 on C2 (overhead check)."""
import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_17889_b200.ep import EPMoELayer, FusedEPMoELayer  # noqa: E402
from paper_2605_17889_b200.layer import MoELayer  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
wts = make_layer_weights(8, 4096, 14336, seed=0, device="cuda")
x = make_tokens(64 * 4096, 4096, seed=1, device="cuda")
for name, lay in [("MoELayer", MoELayer(wts, 2)), ("FusedEP", FusedEPMoELayer(wts, 2)), ("NcclEP", EPMoELayer(wts, 2)),
                  ("MoELayer", MoELayer(wts, 2))]:
    for _ in range(3):
        lay(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        lay(x)
    b.record()
    torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 5, 2), "ms")
dist.destroy_process_group()
