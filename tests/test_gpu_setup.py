"""GPU-side setup against the host builders and the reference.

* qgnn_partitions_from_owner_gpu: every list of every partition equal to the
  host partitions_from_owner (partition.hpp:39-84) — planted graphs with the
  bench's owner map, the reference's BFS owner map, P = 1, P = 70 (a
  multi-word consumer bitmap), and an empty partition.
* qgnn_agg_view_build_gpu: every array of DeviceAggView::build
  (aggregate.hpp:41-89, fp64 coefficients of coeffs.hpp:30-45) bit-identical to
  the host C-ABI view, GCN and SAGE-mean, and to the reference itself through
  oracle/_ref.
* The engine: QGNN_GPU_SETUP=1 (default) and =0 give bit-identical epochs
  (losses, accuracies, wire bytes, weights) in f64 and f32, fixed and adaptive
  (the adaptive statistics consume the GPU-computed Σα² weights).
"""
import os

import numpy as np
import pytest

from oracle import ref
from paper_2306_01381_b200 import _lib, ops
from paper_2306_01381_b200.engine import Engine
from synth import generate_planted

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
SMALL = {k: G[f"g_{k}"] for k in ("adj_ptr", "adj", "features", "labels", "train", "val", "test")}


@pytest.fixture(scope="module")
def planted():
    # 1/64 of the bench graph (config 4 shape, planted owner map, P = 8)
    return generate_planted(2449029 // 64, 61859140 // 64, 16, 47, 8, 0.0085, gamma=2.8, seed=1)


def _same_parts(a, b):
    assert len(a) == len(b)
    for pa, pb in zip(a, b):
        for k in ("owned", "central", "marginal"):
            assert np.array_equal(pa[k], pb[k]), k
        for k in ("remote_in", "remote_out"):
            assert len(pa[k]) == len(pb[k])
            for x, y in zip(pa[k], pb[k]):
                assert np.array_equal(x, y), k


def _owner_cases(planted):
    n = len(planted["owner"])
    rs = np.random.default_rng(3)
    bfs = np.zeros(n, np.uint32)
    ops.lib.qgnn_partition_graph(planted["adj_ptr"].ctypes.data, planted["adj"].ctypes.data, n,
                                 4, 7, bfs.ctypes.data)
    empty = (planted["owner"] % 3).astype(np.uint32)  # partition 3 of 4 owns nothing
    return [("planted", planted["owner"], 8), ("bfs", bfs, 4), ("one", np.zeros(n, np.uint32), 1),
            ("p70", rs.integers(0, 70, n).astype(np.uint32), 70), ("empty", empty, 4)]


def test_partitions_gpu_equal_host(cuda, planted):
    for name, owner, P in _owner_cases(planted):
        host = ops.partitions_from_owner(planted["adj_ptr"], planted["adj"], owner, P)
        gpu = ops.partitions_from_owner(planted["adj_ptr"], planted["adj"], owner, P, gpu_device=0)
        _same_parts(host, gpu)


def test_partitions_gpu_rejects_bad_owner(cuda, planted):
    owner = planted["owner"].copy()
    owner[5] = 9
    with pytest.raises(_lib.InvalidArgument, match="owner id out of range"):
        ops.partitions_from_owner(planted["adj_ptr"], planted["adj"], owner, 8, gpu_device=0)


def _same_view(a, b):
    assert a.keys() == b.keys()
    for k in a:
        if isinstance(a[k], np.ndarray):
            assert a[k].dtype == b[k].dtype, k
            assert np.array_equal(a[k], b[k]), k  # fp64 coefficients bit-identical
        else:
            assert a[k] == b[k], k


@pytest.mark.parametrize("sage", [False, True])
def test_view_gpu_equal_host(cuda, planted, sage):
    for name, owner, P in _owner_cases(planted):
        for d in sorted({0, P - 1, P // 2}):
            host = ops.agg_view(planted["adj_ptr"], planted["adj"], owner, P, d, sage=sage)
            gpu = ops.agg_view(planted["adj_ptr"], planted["adj"], owner, P, d, sage=sage,
                               gpu_device=0)
            _same_view(host, gpu)


@pytest.mark.parametrize("sage", [False, True])
def test_view_gpu_equals_reference(cuda, sage):
    """The reference's own DeviceAggView on its test graph (SBM 120 nodes, P=4)."""
    g = SMALL
    owner = np.zeros(len(g["labels"]), np.uint32)
    ops.lib.qgnn_partition_graph(g["adj_ptr"].ctypes.data, g["adj"].ctypes.data,
                                 len(owner), 4, 11, owner.ctypes.data)
    for d in range(4):
        gpu = ops.agg_view(g["adj_ptr"], g["adj"], owner, 4, d, sage=sage, gpu_device=0)
        exp = ref.view(g["adj_ptr"], g["adj"], owner, 4, d, sage=sage).v
        for k in ("self_alpha", "local_ptr", "local_row", "local_alpha_fwd", "local_alpha_bwd",
                  "remote_ptr", "remote_slot", "remote_alpha", "slot_node", "slot_owner",
                  "device_slot_offset", "central", "marginal"):
            assert np.array_equal(np.asarray(gpu[k]), np.asarray(exp[k]).astype(gpu[k].dtype)), k


def _epochs(g, dims, P, epochs, gpu_setup, **kw):
    old = os.environ.get("QGNN_GPU_SETUP")
    os.environ["QGNN_GPU_SETUP"] = "1" if gpu_setup else "0"
    try:
        eng = Engine(g, dims, n_parts=P, **kw)
    finally:
        if old is None:
            del os.environ["QGNN_GPU_SETUP"]
        else:
            os.environ["QGNN_GPU_SETUP"] = old
    out = [eng.run_epoch() for _ in range(epochs)]
    w = np.concatenate([x.reshape(-1) for x in eng.weights()])
    eng.close()
    keys = ("train_loss", "val_acc", "test_acc", "bytes_total", "ref_bytes_total", "msgs_b2",
            "msgs_b4", "msgs_b8", "plan_version")
    return [tuple(m[k] for k in keys) for m in out], w


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("mode", ["fixed", "adaptive"])
def test_engine_gpu_setup_bit_identical(cuda, planted, dtype, mode):
    kw = dict(bit_mode=mode, fixed_bits=4, seed=5, dtype=dtype, period=2, owner=planted["owner"])
    a, wa = _epochs(planted, [16, 32, 47], 8, 3, True, **kw)
    b, wb = _epochs(planted, [16, 32, 47], 8, 3, False, **kw)
    assert a == b
    assert np.array_equal(wa, wb)


def test_engine_gpu_setup_sage_bfs(cuda):
    kw = dict(bit_mode="adaptive", seed=11, dtype="f64", period=2, sage=True)
    a, wa = _epochs(SMALL, [8, 12, 3], 4, 4, True, **kw)
    b, wb = _epochs(SMALL, [8, 12, 3], 4, 4, False, **kw)
    assert a == b
    assert np.array_equal(wa, wb)
