"""tcgen05 GEMM microbenchmark (z = relu(A W), A: M x K fp32, W: K x N) through the
C-ABI dense_forward, with QGNN_GEMM_DEBUG masks that remove one component at a time
(1 = MMAs, 2 = output stores, 4 = lo split; results invalid under a mask) to see
which one bounds the kernel.  Prints ms and algorithmic GB/s (A read + C write)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01381_b200 import ops  # noqa: E402


def run(M, K, N, reps=20):
    a = torch.randn(M, (K + 3) // 4 * 4, device="cuda")[:, :K]
    w = torch.randn(K, N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    for _ in range(3):
        ops.dense_forward(a, w, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.dense_forward(a, w, out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    gb = (M * a.stride(0) * 4 + M * N * 4) / 1e9
    return t, gb / t * 1e3


DBG = os.environ.get("DBG", "0,1,2,4,3,7").split(",")


def main():
    M = int(os.environ.get("M", 300_000))
    shapes = [tuple(int(v) for v in x.split("x")) for x in
              os.environ.get("SHAPES", "100x256,256x256,256x48").split(",")]
    for K, N in shapes:
        for cl in os.environ.get("CLUSTERS", "1,2").split(","):
            for dbg in DBG:
                os.environ["QGNN_GEMM_DEBUG"] = dbg
                os.environ["QGNN_GEMM_CLUSTER"] = cl
                t, gbs = run(M, K, N)
                print(f"K={K:3d} N={N:3d} cluster={cl} dbg={dbg}  {t*1e3:8.1f} us  {gbs:7.0f} GB/s",
                      flush=True)
    os.environ["QGNN_GEMM_DEBUG"] = "0"


if __name__ == "__main__":
    main()
