import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2306_01381_b200.engine import Engine
G = np.load("tests/golden/golden.npz")
GRAPH = {k: G[f"g_{k}"] for k in ("adj_ptr", "adj", "features", "labels", "train", "val", "test")}
tr = sys.argv[1]
t = time.time()
eng = Engine(GRAPH, [8, 12, 3], n_parts=4, bit_mode="fixed", fixed_bits=4, seed=11, dtype="f32", transport=tr, kstats=bool(int(sys.argv[2])))
print("created", time.time() - t, flush=True)
for i in range(4):
    m = eng.run_epoch()
    print(i, m["train_loss"], m["ms_exchange"], time.time() - t, flush=True)
eng.close()
print("ok", flush=True)
