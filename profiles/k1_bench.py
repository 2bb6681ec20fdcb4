"""K1 microbenchmark: qgnn_quantize_pack (fp32 rows, GPU wire layout) at the
bench's message shapes, timed with CUDA events on the launching stream.

    QGNN_K1_GRP=0|1 python profiles/k1_bench.py [n_messages]

Prints one line per (dim, bits): µs per launch, elements/s, algorithmic GB/s
(rows read D*4 B per message + wire chunk + 19 B metadata) and a
digest of the wire bytes, so two kernel variants can be compared bit for bit
across processes.
"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01381_b200 import ops  # noqa: E402
from paper_2306_01381_b200._lib import WIRE_GPU  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
    torch.cuda.set_device(0)
    torch.manual_seed(0)
    rs = np.random.default_rng(0)
    n_rows = 306_000
    for d in (100, 256):
        ld = (d + 7) // 8 * 8
        x = torch.randn((n_rows, ld), device="cuda")
        x[::3] = torch.relu(x[::3])
        rows = torch.as_tensor(rs.integers(0, n_rows, n).astype(np.int32), device="cuda")
        ids = torch.as_tensor(np.arange(n, dtype=np.int32) * 3, device="cuda")
        sets = torch.as_tensor((np.arange(n) * 8 // n).astype(np.int16), device="cuda")
        keys = torch.as_tensor(rs.integers(0, 2**62, 8).astype(np.int64), device="cuda")
        for b in (8, 4, 2):
            cb = ops.chunk_wire_bytes(d, b)
            off = torch.as_tensor(np.arange(n, dtype=np.int64) * cb, device="cuda")
            bits = torch.full((n,), b, dtype=torch.uint8, device="cuda")
            out = torch.zeros(n * cb, dtype=torch.uint8, device="cuda")
            xv = x[:, :d]
            args = dict(layout=WIRE_GPU, set_of=sets, check_errors=False)
            for _ in range(3):
                ops.quantize_pack(xv, rows, ids, bits, off, keys, out, **args)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record()
            for _ in range(reps):
                ops.quantize_pack(xv, rows, ids, bits, off, keys, out, **args)
            e1.record()
            torch.cuda.synchronize()
            ops.sync_check()
            us = e0.elapsed_time(e1) / reps * 1e3
            byts = n * (d * 4 + cb + 19)
            dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
            print(f"K1 grp={os.environ.get('QGNN_K1_GRP', '1')} D={d} b={b} n={n}: "
                  f"{us:8.1f} us  {n * d / us / 1e3:7.1f} Gelem/s  {byts / us / 1e3:7.1f} GB/s  "
                  f"sha={dig}", flush=True)


if __name__ == "__main__":
    main()
