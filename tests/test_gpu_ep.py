"""EP with the REAL CUDA stage at world size 2 on one GPU (gloo backend, rows
staged through host memory): every rank's output must be bit-identical to
the single-GPU MoELayer on that rank's batch."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2605_17889_b200.ep import EPMoELayer
        from paper_2605_17889_b200.layer import MoELayer
        from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens
        E, d, ff, k = 8, 512, 256, 2
        wts = make_layer_weights(E, d, ff, seed=0, device="cuda")
        x = make_tokens(1500 + 77 * rank, d, seed=10 + rank, device="cuda")
        ref = MoELayer(wts, k)(x).clone()
        out = EPMoELayer(wts, k, "mixtral")(x)
        torch.cuda.synchronize()
        q.put((rank, bool(torch.equal(ref, out))))
    except Exception as exc:  # surface the error to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_ep_world2_real_kernels_bitexact():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
