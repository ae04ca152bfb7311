"""Grouped SwiGLU + down GEMMs over ragged segments (some leaving <= 128 rows
in their last m-tile); prints md5 digests of h and y.  Run once with
COX_GEMM_HALF=0 and once with COX_GEMM_HALF=1: the M = 128 half tiles must
give the same bits as full 256-row tiles (tests/test_gpu_parity.py)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_17889_b200 import ops  # noqa: E402
from paper_2605_17889_b200.synthetic import make_layer_weights, make_tokens  # noqa: E402

E, d, ff = 8, 512, 384
counts = [40, 0, 300, 1, 50, 129, 17, 270]
offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]).astype(np.int32), device="cuda")
wts = make_layer_weights(E, d, ff, seed=0, device="cuda")
x = make_tokens(int(sum(counts)), d, seed=1, device="cuda")
h = ops.grouped_swiglu(x, offs, list(range(E)), [wts.w13[e] for e in range(E)], ff)
y = ops.grouped_down(h, offs, list(range(E)), [wts.w2[e] for e in range(E)], d)
torch.cuda.synchronize()
md5 = lambda t: hashlib.md5(t.cpu().view(torch.int16).numpy().tobytes()).hexdigest()  # noqa: E731
print(md5(h), md5(y))
