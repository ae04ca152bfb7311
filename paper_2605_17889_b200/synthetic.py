"""Synthetic, seeded inputs and random-init weights (no checkpoints, no datasets).

Weights follow nn.Linear's default U(-1/sqrt(fan_in), +1/sqrt(fan_in)) and are
rounded to bf16; x ~ N(0, 1) rounded to bf16.  Generation uses a seeded
torch.Generator on the target device; whoever needs the same bits on the CPU
(the oracle) copies the generated tensors, so both sides see identical values.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class LayerWeights:
    wg: torch.Tensor                 # [E, d] fp32 (bf16-representable values)
    w1: torch.Tensor | None          # [E, ff, d] bf16 (kept only if keep_split)
    w3: torch.Tensor | None          # [E, ff, d] bf16
    w13: torch.Tensor                # [E, 2ff, d] bf16, K3 interleaved layout
    w2: torch.Tensor                 # [E, d, ff] bf16
    shared_w1: torch.Tensor | None = None   # [ffs, d]
    shared_w3: torch.Tensor | None = None
    shared_w13: torch.Tensor | None = None  # [2ffs, d]
    shared_w2: torch.Tensor | None = None   # [d, ffs]

    @property
    def num_experts(self) -> int:
        return self.w13.shape[0]

    @property
    def hidden_dim(self) -> int:
        return self.w13.shape[2]

    @property
    def expert_dim(self) -> int:
        return self.w2.shape[2]


def _uniform(shape, fan_in, g, device):
    t = torch.empty(shape, dtype=torch.float32, device=device)
    t.uniform_(-1.0, 1.0, generator=g)
    t.mul_(fan_in ** -0.5)
    return t.to(torch.bfloat16)


def interleave_w13_torch(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[.., ff, d] x2 -> [.., 2ff, d]: 128-row blocks (gate_i, up_i, ...). Layout helper."""
    *lead, ff, d = w1.shape
    a = w1.reshape(*lead, ff // 128, 128, d)
    b = w3.reshape(*lead, ff // 128, 128, d)
    return torch.stack([a, b], dim=-3).reshape(*lead, 2 * ff, d).contiguous()


def make_router_weight(E: int, d: int, seed: int = 0, device="cuda") -> torch.Tensor:
    """The router weight of make_layer_weights(E, d, ff, seed) alone (its first
    draw from the seeded generator): fp32 [E, d] with bf16-representable values."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return _uniform((E, d), d, g, device).float()


def make_layer_weights(E: int, d: int, ff: int, seed: int = 0, device="cuda", shared_ff: int = 0,
                       keep_split: bool = False) -> LayerWeights:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    wg = _uniform((E, d), d, g, device).float()  # == make_router_weight(E, d, seed)
    w13 = torch.empty((E, 2 * ff, d), dtype=torch.bfloat16, device=device)
    w2 = torch.empty((E, d, ff), dtype=torch.bfloat16, device=device)
    w1s, w3s = [], []
    for e in range(E):
        w1 = _uniform((ff, d), d, g, device)
        w3 = _uniform((ff, d), d, g, device)
        w13[e] = interleave_w13_torch(w1, w3)
        w2[e] = _uniform((d, ff), ff, g, device)
        if keep_split:
            w1s.append(w1)
            w3s.append(w3)
    lw = LayerWeights(wg=wg, w1=torch.stack(w1s) if keep_split else None,
                      w3=torch.stack(w3s) if keep_split else None, w13=w13, w2=w2)
    if shared_ff:
        sw1 = _uniform((shared_ff, d), d, g, device)
        sw3 = _uniform((shared_ff, d), d, g, device)
        lw.shared_w13 = interleave_w13_torch(sw1, sw3)
        lw.shared_w2 = _uniform((d, shared_ff), shared_ff, g, device)
        if keep_split:
            lw.shared_w1, lw.shared_w3 = sw1, sw3
    return lw


def make_tokens(T: int, d: int, seed: int = 1, device="cuda", dtype=torch.bfloat16) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.empty((T, d), dtype=torch.float32, device=device)
    x.normal_(0.0, 1.0, generator=g)
    return x.to(dtype)


def split_w13(w13: torch.Tensor):
    """Inverse of interleave: [.., 2ff, d] -> (w1, w3) [.., ff, d]."""
    *lead, two_ff, d = w13.shape
    ff = two_ff // 2
    v = w13.reshape(*lead, ff // 128, 2, 128, d)
    return (v[..., 0, :, :].reshape(*lead, ff, d), v[..., 1, :, :].reshape(*lead, ff, d))


def chunk_reverse(v: torch.Tensor) -> torch.Tensor:
    """The involution pi that reverses the 8 elements of every chunk of the last
    dimension (d % 8 == 0).  In the router's canonical order a chunk is one
    sequential fma chain, so the products x_i w_i of x.pi(w) enter that chain
    in the opposite order: with pi(x) == x the logit x.pi(w) equals x.w in real
    arithmetic, but the fp32 results may differ in the last bits."""
    *lead, d = v.shape
    return v.reshape(*lead, d // 8, 8).flip(-1).reshape(*lead, d)


def make_tie_batch(T: int, d: int, E: int, seed: int = 3, device="cuda", tie_fraction: float = 0.5,
                   boost: float = 2.0, lead_k: int = 0):
    """Adversarial routing batch: router rows 2m+1 = chunk_reverse(row 2m) for
    the first half of the experts (pairs m < E/4), and a `tie_fraction` of the
    tokens are chunk-reverse symmetric (x == pi(x) bit
    for bit) and pushed toward one pair (2m, 2m+1), so the pair's two logits are
    EQUAL in real arithmetic and differ only by fp32 rounding of the canonical
    summation order — the top-k decision (membership and order) of those tokens
    is decided by rounding alone, or by the lower-index rule when the fp32
    values coincide.  lead_k > 0: half of the tie tokens also get lead_k other
    experts pushed above the pair, so with top_k = lead_k + 1 only one of the
    pair is selected (membership decided by rounding).  Returns (x bf16 [T, d], wg fp32 [E, d] with bf16-exact
    values, pair index per token or -1)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    wg = _uniform((E, d), d, g, device).float()
    npair = max(1, E // 4)
    for m in range(npair):
        wg[2 * m + 1] = chunk_reverse(wg[2 * m])
    x = torch.empty((T, d), dtype=torch.float32, device=device)
    x.normal_(0.0, 1.0, generator=g)
    u = torch.rand((T,), generator=g, device=device)
    pair = torch.randint(0, npair, (T,), generator=g, device=device)
    tie = u < tie_fraction
    dirs = wg[2 * pair] + wg[2 * pair + 1]                      # pi-symmetric direction of the pair
    scale = boost / (wg[0] * wg[0]).sum().clamp_min(1e-12)      # ~boost added to the pair's logits
    xt = 0.5 * (x + chunk_reverse(x)) + scale * dirs
    lead = torch.rand((T,), generator=g, device=device) < 0.5
    for _ in range(lead_k):
        e = torch.randint(2 * npair, E, (T,), generator=g, device=device)  # an unpaired expert
        push = wg[e] + chunk_reverse(wg[e])                     # pi-symmetric push toward expert e
        xt = xt + torch.where(lead[:, None], 2.0 * scale * push, torch.zeros_like(push))
    x = torch.where(tie[:, None], xt, x).to(torch.bfloat16)
    xs = x.reshape(T, d // 8, 8)
    mirrored = xs[:, :, :4].flip(-1)                            # exact symmetry in bf16: q -> 7 - q
    xs[:, :, 4:] = torch.where(tie[:, None, None], mirrored, xs[:, :, 4:])
    return xs.reshape(T, d), wg, torch.where(tie, pair, torch.full_like(pair, -1))


@dataclass
class TopicWorkload:
    """Topic-structured routing for a deep MoE stack (the GPU counterpart of
    eas.generate_synthetic_trace, eas.py:180-240): every sequence belongs to
    one of K latent topics (topic sizes skewed ~ 1/rank), its tokens carry the
    topic's unit direction u_topic (x = noise + amp * u_topic; the residual
    stream keeps it from layer to layer), and each layer's router rows hold a
    per-(topic, layer) Zipf preference over a random expert permutation:
    wg_l[e] = base_l[e] + sum_topic beta * log(E * pref[topic, l, e]) * u_topic / amp,
    so a topic's tokens prefer that topic's hot experts in every layer.
    Calibrating on prototype sequences (eas.cluster / select_prototypes on
    sequence embeddings) therefore predicts which experts are hot."""
    dirs: torch.Tensor          # [K, d] fp32 unit vectors
    topic_weights: list         # [K] sampling probabilities
    amp: float

    @property
    def num_topics(self) -> int:
        return self.dirs.shape[0]


def make_topic_workload(d: int, num_topics: int = 8, amp: float = 8.0, seed: int = 31, device="cuda") -> TopicWorkload:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.empty((num_topics, d), dtype=torch.float32, device=device)
    u.normal_(0.0, 1.0, generator=g)
    u /= u.norm(dim=1, keepdim=True)
    w = [1.0 / (i + 1) for i in range(num_topics)]
    s = sum(w)
    return TopicWorkload(dirs=u, topic_weights=[v / s for v in w], amp=amp)


def make_topic_router(N: int, E: int, d: int, wl: TopicWorkload, zipf: float = 1.2, beta: float = 1.0,
                      seed: int = 7, device="cuda") -> torch.Tensor:
    """Router weights [N, E, d] fp32 (bf16-exact values) with the topic preferences."""
    import numpy as np
    rng = np.random.default_rng(seed)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    wg = torch.empty((N, E, d), dtype=torch.float32, device=device)
    wg.uniform_(-d ** -0.5, d ** -0.5, generator=g)
    rank_w = 1.0 / np.arange(1, E + 1, dtype=float) ** zipf
    rank_w /= rank_w.sum()
    K = wl.num_topics
    bias = np.empty((K, N, E))
    for t in range(K):
        for layer in range(N):
            pref = np.empty(E)
            pref[rng.permutation(E)] = rank_w
            bias[t, layer] = beta * np.log(E * pref)
    b = torch.from_numpy(bias).to(device=device, dtype=torch.float32)       # [K, N, E]
    wg += torch.einsum("kne,kd->ned", b, wl.dirs) / wl.amp
    return wg.to(torch.bfloat16).float()


def make_topic_tokens(wl: TopicWorkload, n_seq: int, seq_len: int, seed: int, device="cuda"):
    """x [n_seq * seq_len, d] bf16 (sequence-major) and the topic of every sequence."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    w = torch.tensor(wl.topic_weights, device=device)
    topics = torch.multinomial(w, n_seq, replacement=True, generator=g)
    d = wl.dirs.shape[1]
    x = torch.empty((n_seq, seq_len, d), dtype=torch.float32, device=device)
    x.normal_(0.0, 1.0, generator=g)
    x += wl.amp * wl.dirs[topics][:, None, :]
    return x.reshape(n_seq * seq_len, d).to(torch.bfloat16), topics


def sequence_embeddings(x: torch.Tensor, n_seq: int, proj_dim: int = 32, seed: int = 5):
    """Per-sequence embedding for prototype clustering: the mean token, randomly
    projected to proj_dim dims (numpy float64 [n_seq, proj_dim])."""
    d = x.shape[1]
    g = torch.Generator(device=x.device)
    g.manual_seed(seed)
    P = torch.empty((d, proj_dim), dtype=torch.float32, device=x.device)
    P.normal_(0.0, d ** -0.5, generator=g)
    m = x.float().reshape(n_seq, -1, d).mean(dim=1)
    return (m @ P).double().cpu().numpy()
