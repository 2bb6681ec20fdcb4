"""CPU tests of the C-ABI library: it loads, exports every declared symbol, and
its host-side logic (RNG, wire layout, partitioning, coefficients, solver,
cost fit) matches the oracle / reference.  No kernels are launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import port, ref_available
from paper_2306_01381_b200 import _lib
from paper_2306_01381_b200._lib import check, lib

GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _declared_symbols():
    text = open(_lib.HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qgnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    syms = _declared_symbols()
    assert len(syms) > 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.HEADER_SYMBOLS)


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = lib.qgnn_ctx_create(0, C.byref(h))
    assert st == _lib.ECUDA
    assert b"no CUDA device" in lib.qgnn_last_error()


def test_rng_matches_oracle():
    rs = np.random.default_rng(1)
    for _ in range(50):
        seed = int(rs.integers(0, 2**63))
        coords = [int(x) for x in rs.integers(0, 2**63, 4)]
        k = lib.qgnn_rng_seed_key(seed)
        for c in coords:
            k = lib.qgnn_rng_fork(k, c)
        assert k == port.stream(seed, *coords)
        for ctr in (1, 2, 1000):
            assert lib.qgnn_rng_u64(k, ctr) == port.draw_u64(k, ctr)


def test_chunk_sizes_ref_and_gpu_layout():
    assert lib.qgnn_chunk_wire_bytes(10, 8, _lib.WIRE_REF, 1) == 35
    assert lib.qgnn_chunk_wire_bytes(64, 2, _lib.WIRE_REF, 1) == 41
    assert lib.qgnn_chunk_wire_bytes(5, 4, _lib.WIRE_REF, 1) == 28
    assert lib.qgnn_chunk_wire_bytes(256, 8, _lib.WIRE_GPU, 0) == 16 + 256
    assert lib.qgnn_chunk_wire_bytes(100, 2, _lib.WIRE_GPU, 0) == 16 + 32
    assert lib.qgnn_chunk_wire_bytes(100, 0, _lib.WIRE_GPU, 0) == 400
    assert lib.qgnn_chunk_wire_bytes(10, 0, _lib.WIRE_GPU, 0) == 48  # raw rows padded to 16 B
    assert lib.qgnn_chunk_wire_bytes(100, 0, _lib.WIRE_REF, 1) == 800


def test_wire_layout_matches_encode_order():  # codec.hpp:56-69, test_quantcodec.cpp:293-315
    from paper_2306_01381_b200.ops import wire_layout
    pos, off, total = wire_layout(np.array([8, 2, 4, 2]), 5, _lib.WIRE_REF, 1)
    assert pos.tolist() == [1, 3, 2, 0]
    G = GOLDEN
    pos, off, total = wire_layout(G["enc_bits"], 96, _lib.WIRE_REF, 1)
    assert (G["enc_ids"][pos] == G["enc_idx_id"]).all()
    assert (off[pos] == G["enc_idx_off"]).all()
    assert total == len(G["enc_wire"])
    with pytest.raises(_lib.InvalidArgument):
        wire_layout(np.array([8, 3]), 5)


def test_partition_graph_matches_reference():
    G = GOLDEN
    ptr, adj = G["g_adj_ptr"], G["g_adj"]
    owner = np.zeros(len(ptr) - 1, np.uint32)
    check(lib.qgnn_partition_graph(ptr.ctypes.data, adj.ctypes.data, len(owner), 4, 11,
                                   owner.ctypes.data))
    assert (owner == G["g_owner_p4_s11"]).all()


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_partition_graph_matches_reference_cite():
    from oracle import ref
    g = ref.generate_dataset("cite", nodes=3000, classes=8, feature_dim=4, attach_edges=6, seed=3)
    for parts, seed in ((2, 7), (3, 1), (8, 99)):
        owner = np.zeros(3000, np.uint32)
        check(lib.qgnn_partition_graph(g["adj_ptr"].ctypes.data, g["adj"].ctypes.data, 3000,
                                       parts, seed, owner.ctypes.data))
        assert (owner == ref.partition_owner(g["adj_ptr"], g["adj"], parts, seed)).all()


def test_compute_coeffs_matches_reference():
    G = GOLDEN
    ptr, adj = G["g_adj_ptr"], G["g_adj"]
    n = len(ptr) - 1
    for sage, key in ((0, "g_alpha_gcn"), (1, "g_alpha_sage")):
        a = np.zeros(len(adj))
        sa = np.zeros(n)
        check(lib.qgnn_compute_coeffs(ptr.ctypes.data, adj.ctypes.data, n, sage, a.ctypes.data,
                                      sa.ctypes.data))
        assert (a == G[key]).all() and (sa == G["g_self_alpha"]).all()


def _solve(pairs, n_dev, theta, gamma, lam, gs, brute=False):
    src = np.array([p[0] for p in pairs], np.uint32)
    dst = np.array([p[1] for p in pairs], np.uint32)
    cnt = np.array([len(p[2]) for p in pairs], np.uint64)
    msgs = [m for p in pairs for m in p[2]]
    mid = np.array([m[0] for m in msgs], np.uint32)
    mdim = np.array([m[1] for m in msgs], np.uint64)
    mlo = np.array([m[2] for m in msgs])
    mhi = np.array([m[3] for m in msgs])
    masq = np.array([m[4] for m in msgs])
    th = np.ascontiguousarray(theta, np.float64)
    ga = np.ascontiguousarray(gamma, np.float64)
    bits = np.zeros(len(msgs), np.int32)
    ev = np.zeros(3)
    check(lib.qgnn_solve_instance(len(pairs), src.ctypes.data, dst.ctypes.data, cnt.ctypes.data,
                                  mid.ctypes.data, mdim.ctypes.data, mlo.ctypes.data,
                                  mhi.ctypes.data, masq.ctypes.data, n_dev, th.ctypes.data,
                                  ga.ctypes.data, lam, gs, int(brute), bits.ctypes.data,
                                  ev.ctypes.data))
    return bits, ev


def _random_instance(rs, n_dev, n_msgs, dims=(4, 8, 16)):
    pairs = []
    for s in range(n_dev):
        for d in range(n_dev):
            if s == d or rs.random() < 0.3:
                continue
            ids = np.sort(rs.choice(1000, int(rs.integers(1, n_msgs + 1)), replace=False))
            msgs = []
            for i in ids:
                lo = float(rs.normal())
                msgs.append((int(i), int(rs.choice(dims)), lo, lo + float(rs.exponential()),
                             float(rs.uniform(0.1, 2.0))))
            pairs.append((s, d, msgs))
    return pairs


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_solver_matches_reference_and_brute_force():  # test_assigner.cpp:228-245
    from oracle import ref
    rs = np.random.default_rng(2024)
    n_checked = 0
    for trial in range(60):
        n_dev = int(rs.integers(2, 4))
        pairs = _random_instance(rs, n_dev, 6)
        if not pairs:
            continue
        theta = rs.uniform(1e-4, 1e-2, n_dev * n_dev)
        gamma = rs.uniform(0, 1e-2, n_dev * n_dev)
        lam = float(rs.choice([0.0, 0.3, 0.5, 0.9, 1.0]))
        gs = int(rs.integers(1, 4))
        bits, ev = _solve(pairs, n_dev, theta, gamma, lam, gs)
        rbits, rev = ref.solve_instance(pairs, n_dev, theta, gamma, lam, gs)
        assert (bits == rbits).all() and (ev == rev).all(), trial
        n_groups = sum(-(-len(p[2]) // gs) for p in pairs)
        if n_groups <= 10:
            bb, bev = _solve(pairs, n_dev, theta, gamma, lam, gs, brute=True)
            rb, rbev = ref.solve_instance(pairs, n_dev, theta, gamma, lam, gs, brute=True)
            assert (bb == rb).all() and (bev == rbev).all()
            assert bev[0] == ev[0]  # exact solver reaches the exhaustive optimum
            n_checked += 1
    assert n_checked > 10


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
@pytest.mark.parametrize("threads", ["1", "3"])
def test_solver_large_instance_matches_reference(monkeypatch, threads):
    """A larger instance (12 device pairs, ~12 groups each, mixed dims), scanned
    on one and on several threads: plan, objective, variance and makespan must
    equal the reference's exactly."""
    import time
    from oracle import ref
    monkeypatch.setenv("QGNN_SOLVE_THREADS", threads)
    rs = np.random.default_rng(7)
    n_dev = 4
    pairs = []
    for s in range(n_dev):
        for d in range(n_dev):
            if s == d:
                continue
            msgs = []
            for i in range(int(rs.integers(500, 700))):
                lo = float(rs.normal())
                msgs.append((i, int(rs.choice([100, 256, 47])), lo, lo + float(rs.exponential()),
                             float(rs.uniform(0.1, 2.0))))
            pairs.append((s, d, msgs))
    theta = rs.uniform(1e-10, 1e-9, n_dev * n_dev)
    gamma = rs.uniform(1e-5, 2e-5, n_dev * n_dev)
    for lam in ((0.3,) if threads == "1" else (0.7,)):
        t0 = time.time()
        bits, ev = _solve(pairs, n_dev, theta, gamma, lam, 50)
        t1 = time.time()
        rbits, rev = ref.solve_instance(pairs, n_dev, theta, gamma, lam, 50)
        t2 = time.time()
        assert (bits == rbits).all() and (ev == rev).all(), lam
        print(f"lambda {lam}: ours {t1 - t0:.3f} s, reference {t2 - t1:.3f} s")


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_solver_frontier_tables_tie_cases_match_reference():
    """The knapsack rows are kept as frontiers and each pair is rebuilt only when
    its largest achievable total under the budget moves (host_solve.cpp).  Cases
    that stress that: equal group variances (ties between widths and between
    groups), lambda 0 and 1, theta = 0 (every budget equal), negative theta
    (non-monotone budgets: the binary-searched caps), ragged last groups
    (small gcd units), and ids in and out of ascending order (the grouping's
    radix and stable_sort paths)."""
    from oracle import ref
    rs = np.random.default_rng(99)
    n_ok = n_raise = 0
    for trial in range(80):
        n_dev = int(rs.integers(2, 5))
        tie = trial % 2 == 0
        pairs = []
        for s in range(n_dev):
            for d in range(n_dev):
                if s == d or rs.random() < 0.2:
                    continue
                n = int(rs.integers(1, 40))
                msgs = []
                for i in range(n):
                    lo = 0.0 if tie else float(rs.normal())
                    hi = lo + (1.0 if tie else float(rs.exponential()))
                    dim = int(rs.choice([4, 8] if tie else [3, 47, 100, 256]))
                    msgs.append((i, dim, lo, hi, 1.0 if tie else float(rs.uniform(0.1, 2.0))))
                if trial % 3 == 0:  # ids out of order: the grouping's stable_sort path
                    msgs = [msgs[j] for j in rs.permutation(len(msgs))]
                pairs.append((s, d, msgs))
        if not pairs:
            continue
        kind = trial % 4
        theta = (np.zeros(n_dev * n_dev) if kind == 1 else
                 rs.uniform(-3e-4, 1e-3, n_dev * n_dev) if kind == 3 else
                 rs.uniform(1e-5, 1e-3, n_dev * n_dev))
        gamma = rs.uniform(0, 1e-2, n_dev * n_dev)
        lam = float(rs.choice([0.0, 0.25, 0.5, 1.0]))
        gs = int(rs.integers(1, 9))
        try:
            rbits, rev = ref.solve_instance(pairs, n_dev, theta, gamma, lam, gs)
        except Exception as e:  # e.g. negative theta: no budget admits any total
            with pytest.raises(_lib.InvalidArgument, match=str(e).split(": ", 1)[-1]):
                _solve(pairs, n_dev, theta, gamma, lam, gs)
            n_raise += 1
            continue
        bits, ev = _solve(pairs, n_dev, theta, gamma, lam, gs)
        assert (bits == rbits).all() and (ev == rev).all(), trial
        n_ok += 1
    assert n_ok > 40


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
def test_solver_bench_shaped_instance_matches_reference():
    """The bench's re-solve shape (8 partitions: 56 pairs of 2000-5000
    messages, one width per pair, groups of 500 with ragged last groups) with
    slow enough links that all three widths are chosen."""
    from oracle import ref
    rs = np.random.default_rng(5)
    n_dev = 8
    pairs = []
    for s in range(n_dev):
        for d in range(n_dev):
            if s == d:
                continue
            dim = int(rs.choice([100, 256, 47]))
            lo = rs.normal(size=int(rs.integers(2000, 5000)))
            hi = lo + rs.exponential(size=lo.size)
            asq = rs.uniform(0.1, 2.0, lo.size)
            pairs.append((s, d, [(i, dim, float(lo[i]), float(hi[i]), float(asq[i]))
                                 for i in range(lo.size)]))
    theta = np.full(n_dev * n_dev, 1e-5)
    gamma = np.full(n_dev * n_dev, 2e-5)
    bits, ev = _solve(pairs, n_dev, theta, gamma, 0.01, 500)
    rbits, rev = ref.solve_instance(pairs, n_dev, theta, gamma, 0.01, 500)
    assert (bits == rbits).all() and (ev == rev).all()
    assert set(np.unique(bits)) == {2, 4, 8}


def test_solver_rejects_bad_instances():  # test_assigner.cpp:265-297
    pairs = [(0, 1, [(1, 4, 0.0, 1.0, 1.0)])]
    with pytest.raises(_lib.InvalidArgument):
        _solve(pairs, 2, [0] * 4, [0] * 4, 1.5, 1)
    with pytest.raises(_lib.InvalidArgument):
        _solve(pairs, 2, [0] * 4, [0] * 4, 0.5, 0)
    big = [(0, 1, [(i, 4, 0.0, 1.0, 1.0) for i in range(20)])]
    with pytest.raises(_lib.ResourceLimitError):
        _solve(big, 2, [1e-3] * 4, [0] * 4, 0.5, 1, brute=True)


def test_pure_variance_weighting_is_all_eight():  # test_assigner.cpp:192-205
    rs = np.random.default_rng(3)
    pairs = _random_instance(rs, 3, 5)
    bits, _ = _solve(pairs, 3, [1e-3] * 9, [1e-3] * 9, 1.0, 2)
    assert (bits == 8).all()


def test_fit_affine():  # cost_model.hpp:78-109, test_commsim.cpp:65-99
    th, ga = C.c_double(), C.c_double()
    x = np.array([1e6, 2e6])
    y = np.array([1e-3 + 1e6 * 2e-9, 1e-3 + 2e6 * 2e-9])
    check(lib.qgnn_fit_affine(x.ctypes.data, y.ctypes.data, 2, C.byref(th), C.byref(ga)))
    assert abs(th.value - 2e-9) < 1e-18 and abs(ga.value - 1e-3) < 1e-12
    y2 = np.array([5.0, 1.0])  # negative slope clamps to zero
    check(lib.qgnn_fit_affine(x.ctypes.data, y2.ctypes.data, 2, C.byref(th), C.byref(ga)))
    assert th.value == 0.0
    with pytest.raises(_lib.InvalidArgument):
        x1 = np.array([1.0, 1.0])
        check(lib.qgnn_fit_affine(x1.ctypes.data, y.ctypes.data, 2, C.byref(th), C.byref(ga)))


def _validate(bits, off, dim, n_bytes, total, layout=_lib.WIRE_REF, dtype=_lib.F64):
    b = np.ascontiguousarray(bits, np.uint8)
    o = np.ascontiguousarray(off, np.uint64)
    d = np.ascontiguousarray(dim, np.uint64)
    st = lib.qgnn_decode_validate(b.ctypes.data, o.ctypes.data, d.ctypes.data, len(b), layout,
                                  dtype, total, n_bytes)
    return st, lib.qgnn_last_error().decode()


def test_decode_index_validation_matches_reference():
    """qgnn_decode_validate raises DecodeError with the reference's own message
    (codec.hpp:82-95, quant.hpp:122-133) on every corrupt-index case of
    test_quantcodec.cpp:389-420; the clean index passes."""
    G = GOLDEN
    wire, bits, dim, off = G["enc_wire"], G["enc_idx_bits"], G["enc_idx_dim"], G["enc_idx_off"]
    n = len(wire)
    assert _validate(bits, off, dim, n, n)[0] == _lib.OK
    gap = off.copy()
    gap[1] += 1
    short = wire[:-3]
    cases = {  # name: (bits, off, dim, bytes, total, reference message)
        "total": (bits, off, dim, wire, n + 1, "message set: byte count mismatch"),
        "gap": (bits, gap, dim, wire, n, "message set: index offsets not contiguous"),
        "trailing": (bits[:-1], off[:-1], dim[:-1], wire, n, "message set: trailing bytes"),
        "truncated": (bits, off, dim, short, len(short), "chunk: truncated payload"),
    }
    for name, (b, o, d, w, total, msg) in cases.items():
        st, got = _validate(b, o, d, len(w), total)
        assert st == _lib.EDECODE and got == msg, (name, got)
        if ref_available():
            from oracle import RefError, ref
            idx = dict(id=G["enc_idx_id"][:len(b)], bits=b, off=o, dim=d)
            with pytest.raises(RefError) as ei:
                ref.decode_message_set(w, idx, total)
            assert msg in str(ei.value), (name, str(ei.value))


@pytest.mark.skipif(not ref_available(), reason="compiled reference not present")
@pytest.mark.parametrize("n_parts", [2, 8, 70])
def test_partitions_and_views_match_reference(n_parts):
    """partitions_from_owner (partition.hpp:39-84) and DeviceAggView::build
    (aggregate.hpp:41-89) through the C-ABI equal the compiled reference's, for
    BFS and random owner maps, GCN and SAGE coefficients (P = 70 > 64 too)."""
    from oracle import ref
    from paper_2306_01381_b200 import ops
    g = ref.generate_dataset("cite", nodes=2500, classes=8, feature_dim=4, attach_edges=6, seed=5)
    ptr, adj = g["adj_ptr"], g["adj"]
    rs = np.random.default_rng(n_parts)
    owners = [ref.partition_owner(ptr, adj, n_parts, 7),
              rs.integers(0, n_parts, len(ptr) - 1).astype(np.uint32)]
    for owner in owners:
        parts = ops.partitions_from_owner(ptr, adj, owner, n_parts)
        for dev in sorted({0, n_parts // 2, n_parts - 1}):
            for sage in (False, True):
                rv = ref.view(ptr, adj, owner, n_parts, dev, sage=sage).v
                P = parts[dev]
                assert (P["owned"] == rv["owned"]).all()
                for q in range(n_parts):
                    assert (P["remote_in"][q] == rv["remote_in"][q]).all(), q
                    assert (P["remote_out"][q] == rv["remote_out"][q]).all(), q
                v = ops.agg_view(ptr, adj, owner, n_parts, dev, sage=sage)
                assert (P["owned"][v["central"]] == P["central"]).all()
                assert (P["owned"][v["marginal"]] == P["marginal"]).all()
                for k in ("self_alpha", "local_ptr", "local_row", "local_alpha_fwd",
                          "local_alpha_bwd", "remote_ptr", "remote_slot", "remote_alpha",
                          "slot_node", "slot_owner", "device_slot_offset", "central",
                          "marginal"):
                    assert np.array_equal(v[k], rv[k].astype(v[k].dtype)), (k, dev, sage)


def test_plan_bits_for_lookup():  # plan.hpp:60-72
    from paper_2306_01381_b200 import InvalidArgument, ops
    ids = np.array([3, 9, 10, 44], np.uint32)
    bits = np.array([2, 8, 4, 8], np.int32)
    assert list(ops.plan_bits_for(ids, bits, [44, 3, 10, 9])) == [8, 2, 4, 8]
    with pytest.raises(InvalidArgument, match="unknown message id"):
        ops.plan_bits_for(ids, bits, [5])
