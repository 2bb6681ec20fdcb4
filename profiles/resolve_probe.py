"""Adaptive re-solve cost on the bench workload: run 50 epochs (period 50) and
report the host solver time of the re-solve epoch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2306_01381_b200.engine import Engine, generate_planted  # noqa: E402

w = bench.WORKLOAD
g = generate_planted(w["nodes"], w["n_edges"], w["feat"], w["classes"], w["parts"],
                     w["cross_frac"], gamma=w["gamma"], seed=w["seed"])
eng = Engine(g, [w["feat"], w["hidden"], w["hidden"], w["classes"]], n_parts=w["parts"],
             bit_mode="adaptive", fixed_bits=8, seed=7, group_size=2000, period=50,
             theta=1.0 / (900e9 * 8), gamma=2e-5, dtype="f32", owner=g["owner"])
t0 = time.time()
for e in range(1, 51):
    m = eng.run_epoch()
    if m["resolve_seconds"] > 0:
        print(f"epoch {e}: resolve {m['resolve_seconds']:.3f} s, plan v{m['plan_version']}, "
              f"b2/b4/b8 = {m['msgs_b2']}/{m['msgs_b4']}/{m['msgs_b8']}, device ms {m['ms_total']:.1f}")
print(f"50 epochs wall {time.time() - t0:.2f} s")
m = eng.run_epoch()
print(f"epoch 51 after re-solve: device ms {m['ms_total']:.1f}, loss {m['train_loss']:.4f}")
eng.close()
