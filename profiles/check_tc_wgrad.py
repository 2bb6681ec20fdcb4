# debug: MN-major tcgen05 weight-gradient variants (run under gpurun)
import os, sys, subprocess
import numpy as np
if len(sys.argv) == 1:
    for v in range(4):
        env = dict(os.environ, QGNN_TC_MN=str(v))
        r = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print("variant", v, "->", (r.stdout + r.stderr).strip()[-600:], flush=True)
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_01381_b200 import ops
rs = np.random.default_rng(0)
for (n, m, k) in [(64, 32, 32), (1000, 100, 256), (5000, 256, 47)]:
    a = rs.standard_normal((n, m)).astype(np.float32)
    b = rs.standard_normal((n, k)).astype(np.float32)
    am = np.zeros((n, (m + 7) // 8 * 8), np.float32); am[:, :m] = a
    bm = np.zeros((n, (k + 7) // 8 * 8), np.float32); bm[:, :k] = b
    at = torch.as_tensor(am, device="cuda")[:, :m]
    bt = torch.as_tensor(bm, device="cuda")[:, :k]
    out = torch.zeros((m, k), device="cuda")
    ops.dense_weight_grad(at, bt, out)
    torch.cuda.synchronize()
    ref = a.astype(np.float64).T @ b.astype(np.float64)
    o = out.cpu().numpy()
    print(f"n={n} m={m} k={k} maxerr={np.abs(o-ref).max():.3e} ref_max={np.abs(ref).max():.2f} "
          f"o[0,:3]={o[0,:3]} ref[0,:3]={ref[0,:3]}")
