"""Generate the numeric golden vectors (run once in the build container; the
outputs are committed, this script is kept for provenance).

    python tests/golden/make_numeric_golden.py

The reference (moeplan) contains no router/permute/FFN code, so these vectors
come from restatements INDEPENDENT of the C oracle:
  * routing_<case>.npz : expected top-k indices for a seeded batch.  Tokens
    whose float64 top-k is well separated (gap > 1e-3 between the k-th and
    (k+1)-th logits) take the float64 answer; for the near-tie tokens the
    canonical fp32 summation order (oracle_router.c header) is replayed with
    EXACT rational arithmetic (fractions.Fraction, correctly rounded to fp32 at
    every fma/add), and the golden stores those fp32 logits bit-for-bit.
  * layer_micro.npz : small ragged cases (E=4, d=64, ff=96, T=37, incl. an
    empty expert) with float64 numpy outputs of the whole expert stage.
Inputs are regenerated from the seeds by tests/golden/inputs.py (no large
arrays committed).
"""
from __future__ import annotations

import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from inputs import ROUTING_CASES, layer_micro_inputs, routing_inputs  # noqa: E402

_HALF = Fraction(1, 2)


def f32_round(fr: Fraction) -> np.float32:
    """Round a rational to the nearest fp32 (ties to even); normal range only."""
    if fr == 0:
        return np.float32(0.0)
    sign = -1 if fr < 0 else 1
    a = abs(fr)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    scale = Fraction(2) ** (e - 23)
    q = a / scale
    n = q.numerator // q.denominator
    rem = q - n
    if rem > _HALF or (rem == _HALF and n % 2 == 1):
        n += 1
    return np.float32(float(sign * n * scale))


def canonical_logit_exact(x: np.ndarray, w: np.ndarray) -> np.float32:
    """The canonical order of oracle_router.c, with exact rational fma/add."""
    d = x.shape[0]
    xs = [Fraction(float(v)) for v in x]
    ws = [Fraction(float(v)) for v in w]
    p = []
    for l in range(32):
        acc = np.float32(0.0)
        j = 0
        while True:
            s = 8 * (32 * j + l)
            if s >= d:
                break
            for q in range(8):
                acc = f32_round(xs[s + q] * ws[s + q] + Fraction(float(acc)))
            j += 1
        p.append(acc)
    for off in (16, 8, 4, 2, 1):
        p = [f32_round(Fraction(float(p[l])) + Fraction(float(p[l ^ off]))) for l in range(32)]
    return p[0]


def make_routing(name: str):
    x, wg, k = routing_inputs(name)
    lg64 = x.astype(np.float64) @ wg.astype(np.float64).T
    T, E = lg64.shape
    order = np.argsort(-lg64, axis=1, kind="stable")
    srt = np.take_along_axis(lg64, order, axis=1)
    # a token is "near-tie" if any adjacent pair among the top k+1 is within 1e-3
    gaps = np.abs(np.diff(srt[:, : k + 1], axis=1)).min(axis=1)
    near = np.nonzero(gaps < 1e-3)[0]
    idx = order[:, :k].astype(np.int32)
    exact_logits = np.full((len(near), E), np.nan, np.float32)
    for i, t in enumerate(near):
        # Only experts that can enter the top-k are replayed exactly: the top
        # k+4 by float64, provided the rest lie > 1e-3 below the (k+1)-th.
        cand = list(order[t, : k + 4]) if E > k + 4 and srt[t, k + 3] < srt[t, k] - 1e-3 else list(range(E))
        for e in cand:
            exact_logits[i, e] = canonical_logit_exact(x[t], wg[e])
        lg = exact_logits[i]
        taken = []
        for _ in range(k):
            best = -1
            for e in sorted(cand):
                if e in taken:
                    continue
                if best < 0 or lg[e] > lg[best]:
                    best = e
            taken.append(best)
        idx[t] = taken
    np.savez_compressed(HERE / f"routing_{name}.npz", idx=idx.astype(np.int8), near=near.astype(np.int32),
                        exact_logits=exact_logits)
    flips = sum(int((order[t, :k] != idx[t]).any()) for t in near)
    print(f"routing_{name}: T={T} near-ties={len(near)} fp64-vs-fp32 flips={flips}")


def silu(g):
    return g / (1.0 + np.exp(-g))


def make_layer_micro():
    out = {}
    for case, (x, wg, w1, w3, w2, k, mode) in layer_micro_inputs().items():
        xd = x.astype(np.float64)
        lg = xd @ wg.astype(np.float64).T
        T, E = lg.shape
        idx = np.argsort(-lg, axis=1, kind="stable")[:, :k]
        sel = np.take_along_axis(lg, idx, axis=1)
        if mode == 0:
            p = np.exp(sel - sel.max(axis=1, keepdims=True))
            wts = p / p.sum(axis=1, keepdims=True)
        else:
            p = np.exp(lg - lg.max(axis=1, keepdims=True))
            wts = np.take_along_axis(p / p.sum(axis=1, keepdims=True), idx, axis=1)
        res = np.zeros((T, x.shape[1]))
        for t in range(T):
            for j in range(k):
                e = idx[t, j]
                h = silu(w1[e].astype(np.float64) @ xd[t]) * (w3[e].astype(np.float64) @ xd[t])
                res[t] += wts[t, j] * (w2[e].astype(np.float64) @ h)
        counts = np.bincount(idx.ravel(), minlength=E)
        out[f"{case}_idx"] = idx.astype(np.int32)
        out[f"{case}_w"] = wts
        out[f"{case}_counts"] = counts.astype(np.int32)
        out[f"{case}_out"] = res
    np.savez_compressed(HERE / "layer_micro.npz", **out)
    print("layer_micro:", sorted({k.split('_')[0] for k in out}))


if __name__ == "__main__":
    for name in ROUTING_CASES:
        make_routing(name)
    make_layer_micro()
