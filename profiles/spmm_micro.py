"""SpMM microbenchmark: one partition-sized CSR (306k rows, ~50 nnz/row) with
controlled neighbour locality, D = 100 / 256, through the production fp32 path.
Prints effective gathered TB/s (nnz * D * 4 / t) and compulsory GB/s."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01381_b200 import ops  # noqa: E402


def make_csr(n, deg, window, rs):
    # each row: `deg` neighbours at uniform offset within +-window (wrapping), sorted
    off = rs.integers(1, window + 1, size=(n, deg)) * rs.choice([-1, 1], size=(n, deg))
    col = (np.arange(n)[:, None] + off) % n
    col.sort(axis=1)
    ptr = np.arange(0, n * deg + 1, deg, dtype=np.int64)
    return ptr, col.reshape(-1).astype(np.int32)


def bench(ptr, col, n, d, reps=10):
    dev = "cuda"
    x = torch.randn(n, d, device=dev)
    out = torch.empty(n, d, device=dev)
    p = torch.as_tensor(ptr, device=dev)
    c = torch.as_tensor(col, device=dev)
    a = torch.full((len(col),), 0.02, device=dev)
    sa = torch.full((n,), 0.5, device=dev)
    for _ in range(3):
        ops.csr_aggregate(x, p, c, a, out, self_alpha=sa)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.csr_aggregate(x, p, c, a, out, self_alpha=sa)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    nnz = len(col)
    gathered = nnz * d * 4
    compulsory = 2 * n * d * 4 + nnz * 8
    return t, gathered / t / 1e12, compulsory / t / 1e9


def main():
    rs = np.random.default_rng(0)
    n, deg = 306_000, 50
    for window in (32, 1024, 16_384, 150_000):
        ptr, col = make_csr(n, deg, window, rs)
        for d in (100, 256):
            t, g, c = bench(ptr, col, n, d)
            print(f"window={window:7d} D={d:3d}  {t*1e3:7.3f} ms  gathered {g:5.2f} TB/s  "
                  f"compulsory {c:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
