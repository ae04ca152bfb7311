"""Expert-parallel dispatch/combine logic on CPU: world_size 2 and 4 over gloo,
with the CPU oracle standing in for the CUDA kernels (the communication and
layout code is exactly the product's ep.EPMoELayer).  The EP result must be
BIT-identical to the single-rank oracle on every rank's batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleStage:
    def __init__(self, wg, w1, w3, w2, k, mode, local):
        self.wg, self.w1, self.w3, self.w2 = wg, w1, w3, w2
        self.k, self.mode, self.local = k, mode, list(local)
        self.E = wg.shape[0]

    def route_and_permute(self, x):
        xn = x.numpy()
        idx, w, counts = O.router_topk(xn, self.wg, self.k, self.mode)
        offsets, dst = O.permute(idx, self.E, 1)
        x_perm = O.gather(xn, dst, int(offsets[-1]))
        t = torch.from_numpy
        return t(idx), t(w), t(counts), t(dst), t(x_perm)

    def experts(self, rows, seg_offsets, n_src, out=None):
        L = len(self.local)
        seg = seg_offsets.numpy()
        y = out if out is not None else torch.empty_like(rows)
        for g in range(n_src * L):
            r0, r1 = int(seg[g]), int(seg[g + 1])
            if r1 > r0:
                e = self.local[g % L]
                y[r0:r1] = torch.from_numpy(O.expert_ffn(rows[r0:r1].numpy(), self.w1[e], self.w3[e], self.w2[e]))
        return y

    def combine(self, yback, dst, w):
        return torch.from_numpy(O.combine(yback.numpy(), dst.numpy(), w.numpy()))

    def empty_rows(self, n, like):
        return torch.empty((max(n, 1), like.shape[1]), dtype=like.dtype)


def _weights(E, d, ff, seed=0):
    rng = np.random.default_rng(seed)
    u = lambda *s, fan: (rng.random(s, dtype=np.float32) * 2 - 1) / np.float32(np.sqrt(fan))  # noqa: E731
    return u(E, d, fan=d), u(E, ff, d, fan=d), u(E, ff, d, fan=d), u(E, d, ff, fan=ff)


def _tokens(rank, T, d):
    return np.random.default_rng(100 + rank).standard_normal((T, d), dtype=np.float32)


def _worker(rank, ws, port, E, d, ff, k, mode, T, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2605_17889_b200.ep import EPMoELayer
        wg, w1, w3, w2 = _weights(E, d, ff)
        L = E // ws
        stage = OracleStage(wg, w1, w3, w2, k, mode, range(rank * L, (rank + 1) * L))
        layer = EPMoELayer({"E": E}, k, "mixtral" if mode == 0 else "deepseek", stage=stage)
        Tr = T + 7 * rank  # ragged batches per rank
        x = _tokens(rank, Tr, d)
        out = layer(torch.from_numpy(x)).numpy()
        ref = O.moe_layer(x, wg, w1, w3, w2, k, mode)["out"]
        ok = np.array_equal(out, ref)
        q.put((rank, ok, float(np.abs(out - ref).max()), layer.last_split))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ws,E,k,mode", [(2, 4, 2, 0), (4, 8, 2, 0), (2, 16, 6, 1)])
def test_ep_bitexact_vs_single_rank(ws, E, k, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, PORTS[(ws, E)], E, 64, 96, k, mode, 37, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, err, split in sorted(res):
        assert ok, f"rank {rank}: EP output differs from single-rank oracle (max |err| {err})"
        send, recv = split
        assert len(send) == ws and sum(send) == (37 + 7 * rank) * k


PORTS = {(2, 4): _free_port(), (4, 8): _free_port(), (2, 16): _free_port()}
