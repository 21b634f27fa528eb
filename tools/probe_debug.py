"""Probe-GEMM experiment: cfg3-shaped coarse quantizer (K=65536, d=128,
mixture-sampled centroids), 4096..10000 queries; prints timing and (with
PQS_PROBE_DEBUG=1) candidate statistics.  Checks a sample against the oracle."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02912_b200 as P  # noqa: E402
from oracle import pqscan_oracle as O  # noqa: E402
from tests.helpers import mixture  # noqa: E402

K = int(os.environ.get("K", 65536))
NQ = int(os.environ.get("NQ", 10000))
MA = int(os.environ.get("MA", 64))
rng = np.random.default_rng(3)
x = mixture(rng, K + NQ, 128)
coarse, qs = x[:K], x[K:] + 0.5
books = rng.normal(0, 1, (8, 256, 16)).astype(np.float32)
pq = P.ProductQuantizer(8, 8, 128, books)
sizes = np.zeros(K, np.int64)
sizes[0] = 1
ivf = P.DeviceIvf.from_arrays(pq, coarse, sizes, np.zeros((1, 8), np.uint8), np.zeros(1, np.int64))
qd = torch.from_numpy(qs).cuda()
for _ in range(2):
    ivf.probe(qd, MA)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cells, dist = ivf.probe(qd, MA)
e1.record()
torch.cuda.synchronize()
print(f"probe {NQ} queries x K={K} ma={MA}: {e0.elapsed_time(e1):.3f} ms")
cells, dist = cells.cpu().numpy(), dist.cpu().numpy()
for qi in range(0, NQ, NQ // 8):
    oc, od = O.nearest_k(qs[qi:qi + 1].astype(np.float64), coarse.astype(np.float64), MA)
    assert np.array_equal(cells[qi], oc[0]) and np.array_equal(dist[qi], od[0]), qi
print("sample == oracle")
