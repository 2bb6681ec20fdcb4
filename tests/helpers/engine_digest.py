"""Run the fp32 engine on a 1/64 sample of the bench workload (BASELINE config 4
shape) and print a digest of every epoch's metrics and the final weights, so
two engine settings (environment switches) can be compared bit for bit across
processes.  Used by tests/test_gpu_fused.py."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2306_01381_b200.engine import Engine  # noqa: E402
from synth import generate_planted  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "adaptive"
    bits = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    g = generate_planted(2449029 // 64, 61859140 // 64, 100, 47, 8, 0.0085, gamma=2.8, seed=1)
    eng = Engine(g, [100, 256, 256, 47], n_parts=8, bit_mode=mode, fixed_bits=bits, seed=7,
                 group_size=2000, period=2, theta=1.0 / (900e9 * 8), gamma=2e-5, dtype="f32",
                 owner=g["owner"], kstats=True)
    ep = []
    for _ in range(4):
        m = eng.run_epoch()
        ep.append([m["train_loss"], m["val_acc"], m["test_acc"], m["bytes_total"], m["msgs_b2"],
                   m["msgs_b4"], m["msgs_b8"], m["plan_version"]])
    w = np.concatenate([x.reshape(-1) for x in eng.weights()]).astype(np.float32)
    ks = eng.kernel_stats()
    print(json.dumps({"epochs": ep, "weights_sha": hashlib.sha1(w.tobytes()).hexdigest(),
                      "dequant_launches": ks["dequant"]["launches"]}))
    eng.close()


if __name__ == "__main__":
    main()
