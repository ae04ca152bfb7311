"""EP with the REAL CUDA stage at world size 2 on one GPU: the NCCL-style path
(gloo, rows staged through host memory) and the fused peer-memory path
(buffers mapped across the two processes by CUDA IPC).  Every rank's output
must be bit-identical to the single-GPU MoELayer on that rank's batch."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


class IpcTransport:
    """Test transport for several ranks on ONE GPU (symmetric memory refuses
    that): buffers are exchanged between the processes as CUDA IPC handles
    (torch.multiprocessing queues), the barrier is a device sync + gloo barrier."""

    def __init__(self, rank, inboxes):
        self.rank, self.inboxes = rank, inboxes
        self._keep = []

    def alloc(self, spec, dev):
        mine = {n: torch.zeros(shape, dtype=dt, device=dev) for n, (shape, dt) in spec.items()}
        for r, box in enumerate(self.inboxes):
            if r != self.rank:
                box.put((self.rank, mine))
        peers = {self.rank: mine}
        for _ in range(len(self.inboxes) - 1):
            r, t = self.inboxes[self.rank].get(timeout=120)
            peers[r] = t
        self._keep.append(peers)  # every allocation's peer mappings stay alive
        out = {}
        for n in spec:
            ptrs = [peers[r][n].data_ptr() for r in range(len(self.inboxes))]
            out[n] = (mine[n], torch.tensor(ptrs, dtype=torch.int64, device=dev))
        return out

    def barrier(self):
        torch.cuda.synchronize()
        dist.barrier()


def _worker(rank, ws, port, q, fused=False, inboxes=None, cap_factor=1.25, check_capacity=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2605_17889_b200.ep import EPMoELayer, FusedEPMoELayer
        from paper_2605_17889_b200.layer import MoELayer
        from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens
        E, d, ff, k = 8, 512, 256, 2
        wts = make_layer_weights(E, d, ff, seed=0, device="cuda")
        x = make_tokens(1500 + 77 * rank, d, seed=10 + rank, device="cuda")
        ref = MoELayer(wts, k)(x).clone()
        if fused and not check_capacity:
            # capacity overflow without the host check: rows beyond cap are dropped
            # by the kernels (no out-of-bounds access) and check() raises
            lay = FusedEPMoELayer(wts, k, "mixtral", transport=IpcTransport(rank, inboxes),
                                  capacity_factor=cap_factor, check_capacity=False)
            lay(x)
            torch.cuda.synchronize()
            try:
                lay.check()
                q.put((rank, "overflow not reported"))
            except RuntimeError:
                q.put((rank, True))
            return
        if fused:
            lay = FusedEPMoELayer(wts, k, "mixtral", transport=IpcTransport(rank, inboxes),
                                  capacity_factor=cap_factor)
            out = lay(x).clone()
            out2 = lay(x)
            torch.cuda.synchronize()
            lay.check()
            if not torch.equal(out, out2):
                q.put((rank, "second step differs"))
                return
            if cap_factor < 0.1 and lay.regrows != 1:
                q.put((rank, f"expected one capacity regrow, got {lay.regrows}"))
                return
        else:
            out = EPMoELayer(wts, k, "mixtral")(x)
        torch.cuda.synchronize()
        q.put((rank, bool(torch.equal(ref, out))))
    except Exception as exc:  # surface the error to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused,cap_factor,check_capacity", [
    (False, 1.25, True),
    (True, 1.25, True),
    (True, 0.01, True),    # receive buffers far too small: grown collectively, still bit-exact
    (True, 0.01, False),   # no host check: dropped rows, no out-of-bounds access, check() raises
])
def test_ep_world2_real_kernels_bitexact(fused, cap_factor, check_capacity):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    inboxes = [ctx.Queue() for _ in range(2)]
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, fused, inboxes, cap_factor, check_capacity))
          for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
