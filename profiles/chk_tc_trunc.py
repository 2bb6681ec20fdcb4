import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2306_01381_b200 import ops
rs = np.random.default_rng(0)
for din, dout in ((256, 256), (100, 256), (256, 47)):
    a = rs.standard_normal((4096, din)); w = rs.standard_normal((din, dout))
    ref = a @ w
    out = torch.zeros((4096, dout), dtype=torch.float32, device="cuda")
    ops.dense_forward(torch.as_tensor(a, dtype=torch.float32, device="cuda"), torch.as_tensor(w, dtype=torch.float32, device="cuda"), out, relu=False)
    a32 = a.astype(np.float32).astype(np.float64); w32 = w.astype(np.float32).astype(np.float64)
    ref32 = a32 @ w32
    err = np.abs(out.cpu().numpy() - ref32).max() / np.abs(ref32).max()
    print(os.environ.get("QGNN_EXP_NOHI", "0"), din, dout, "max rel err vs fp64 of fp32 inputs:", err)
