# Row-granular LRU simulation of the 256-wide source-row gathers of partition 0 (bench graph):
# hit rate for four destination-row orders at a 100k-row (~100 MB of 1 KB rows) cache.
# gcc -O2 -o profiles/_l2_order_sim profiles/l2_order_sim.c && python profiles/l2_order_sim.py 100000
import numpy as np, sys, subprocess, collections
sys.path.insert(0, '/root/repo')
import synth
g = synth.generate_planted(2449029, 61859140, 4, 47, 8, 0.0085, gamma=2.8, seed=1)
ptr, adj, own = g['adj_ptr'], g['adj'], g['owner']
rows = np.where(own == 0)[0]
lo, hi = rows[0], rows[-1] + 1
sub = adj[ptr[lo]:ptr[hi]]
uniq, inv = np.unique(sub, return_inverse=True)
lptr = (ptr[lo:hi + 1] - ptr[lo]).astype(np.int64)
col = inv.astype(np.int32)
n = hi - lo
deg = np.diff(lptr)
def write(order, name):
    with open('/tmp/l2_order_g.bin', 'wb') as f:
        np.array([n, len(col)], np.int64).tofile(f); np.array([len(uniq)], np.int32).tofile(f)
        lptr.tofile(f); col.tofile(f); order.astype(np.int32).tofile(f)
    for cap in (int(sys.argv[1]),):
        print(name, subprocess.run(['./profiles/_l2_order_sim', '/tmp/l2_order_g.bin', str(cap)], capture_output=True, text=True).stdout.strip())
write(np.arange(n), 'ascending')
write(np.random.default_rng(0).permutation(n), 'random')
write(np.argsort(-deg, kind='stable'), 'deg-desc')
# BFS order within the partition from the max-degree row (RCM-like: neighbours by ascending degree)
local = {}
seen = np.zeros(n, bool); order = []
gid2row = np.full(len(uniq), -1); m = (uniq >= lo) & (uniq < hi); gid2row[m] = uniq[m] - lo
for start in np.argsort(-deg, kind='stable'):
    if seen[start]: continue
    seen[start] = True; q = collections.deque([start])
    while q:
        r = q.popleft(); order.append(r)
        nb = gid2row[col[lptr[r]:lptr[r+1]]]; nb = nb[nb >= 0]; nb = nb[~seen[nb]]
        nb = np.unique(nb); nb = nb[np.argsort(deg[nb], kind='stable')]
        seen[nb] = True; q.extend(nb.tolist())
write(np.array(order), 'bfs')
