"""World > 1 engine: ranks as threads on one GPU through the loopback transport
(same routing as the NCCL path: arena offsets, remote pairs, rank slices of the
weight-gradient / loss / trace-window all-gathers).  Splitting the partitions
over ranks must not change a single bit: every partition computes the same
thing and the weight gradient is summed in ascending partition order
(engine.hpp:786-788)."""
import os
import threading

import numpy as np
import pytest

from paper_2306_01381_b200.engine import Engine, generate_planted, loopback_id

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
GRAPH = {k: G[f"g_{k}"] for k in ("adj_ptr", "adj", "features", "labels", "train", "val", "test")}
_GROUP = [1000]


def _run_world(graph, world, epochs, **kw):
    gid = _GROUP[0]
    _GROUP[0] += 1
    nid = loopback_id(gid) if world > 1 else None
    out = [None] * world
    err = []
    engines = [None] * world

    def worker(r):
        try:
            eng = Engine(graph, rank=r, world=world, nccl_id=nid, **kw)
            engines[r] = eng
            ms = [eng.run_epoch() for _ in range(epochs)]
            w = np.concatenate([x.reshape(-1) for x in eng.weights()])
            out[r] = (ms, w)
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not err, err
    for e in engines:
        if e is not None:
            e.close()
    return out


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode,dtype", [("fixed", "f32"), ("uniform", "f32"), ("fp", "f64")])
def test_world_split_is_bit_identical(cuda, world, mode, dtype):
    kw = dict(dims=[8, 12, 3], n_parts=4, bit_mode=mode, fixed_bits=4, seed=11, dtype=dtype)
    (base_ms, base_w), = _run_world(GRAPH, 1, 4, **kw)
    res = _run_world(GRAPH, world, 4, **kw)
    for ms, w in res:
        assert [m["train_loss"] for m in ms] == [m["train_loss"] for m in base_ms]
        assert [m["val_acc"] for m in ms] == [m["val_acc"] for m in base_ms]
        assert [m["bytes_total"] for m in ms] == [m["bytes_total"] for m in base_ms]
        assert (w == base_w).all()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode,dtype", [("fixed", "f32"), ("uniform", "f32"), ("fp", "f64"),
                                        ("adaptive", "f32")])
def test_peer_store_is_bit_identical(cuda, world, mode, dtype):
    """Peer-store transport (K1 writes straight into the receivers' arenas, ready /
    consumed flags instead of exchange copies; SURVEY §8f rank 1 at N > 1): the
    same bits as one rank, across plan changes (adaptive re-solves every 2 epochs)."""
    kw = dict(dims=[8, 12, 3], n_parts=4, bit_mode=mode, fixed_bits=4, seed=11, dtype=dtype,
              period=2)
    (base_ms, base_w), = _run_world(GRAPH, 1, 5, **kw)
    res = _run_world(GRAPH, world, 5, transport="p2p", **kw)
    for ms, w in res:
        assert [m["train_loss"] for m in ms] == [m["train_loss"] for m in base_ms]
        assert [m["val_acc"] for m in ms] == [m["val_acc"] for m in base_ms]
        assert [m["bytes_total"] for m in ms] == [m["bytes_total"] for m in base_ms]
        assert [m["plan_version"] for m in ms] == [m["plan_version"] for m in base_ms]
        assert (w == base_w).all()


def test_peer_store_planted_graph(cuda):
    """Peer stores on the production kernels (256-wide fused receive, 8 partitions
    over 4 ranks) and the planted owner map."""
    g = generate_planted(20000, 200000, 32, 8, 8, 0.02, gamma=2.8, seed=4)
    kw = dict(dims=[32, 256, 8], n_parts=8, bit_mode="adaptive", seed=3, period=2,
              owner=g["owner"])
    (base_ms, base_w), = _run_world(g, 1, 4, **kw)
    for world in (2, 4):
        res = _run_world(g, world, 4, transport="p2p", **kw)
        for ms, w in res:
            assert [m["train_loss"] for m in ms] == [m["train_loss"] for m in base_ms]
            assert (w == base_w).all()


def test_peer_store_missing_payload_is_protocol_error(cuda, monkeypatch):
    """A rank whose stores never get published (fault injection: rank 1 drops its
    first ready flag) makes its peer's flag wait time out and the epoch fail with
    ProtocolError "missing payload" (engine.hpp:530) instead of hanging the GPU
    (both threads return well within the join timeout)."""
    from paper_2306_01381_b200._lib import ProtocolError
    monkeypatch.setenv("QGNN_TEST_P2P_DROP", "1")
    monkeypatch.setenv("QGNN_P2P_TIMEOUT_MS", "300")
    gid = _GROUP[0]
    _GROUP[0] += 1
    nid = loopback_id(gid)
    errs = [None, None]
    engines = [None, None]

    def worker(r):
        try:
            engines[r] = Engine(GRAPH, dims=[8, 12, 3], n_parts=4, bit_mode="fixed", fixed_bits=8,
                                seed=11, dtype="f32", rank=r, world=2, nccl_id=nid,
                                transport="p2p")
            engines[r].run_epoch()
        except Exception as e:  # noqa: BLE001 - inspected below
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    for e in engines:
        if e is not None:
            e.close()
    assert isinstance(errs[0], ProtocolError) and "missing payload" in str(errs[0]), errs
    # the sender is stalled behind the receiver's late consumed flag: it may time out
    # too, but only ever with the same ProtocolError
    assert errs[1] is None or isinstance(errs[1], ProtocolError), errs


def test_world_split_adaptive_matches_reference(cuda):
    """Adaptive re-solves gather trace windows across ranks: same plans, same losses."""
    kw = dict(dims=[8, 12, 3], n_parts=4, bit_mode="adaptive", seed=11, period=5, dtype="f64")
    ref = G["eng_ad_epochs"]
    res = _run_world(GRAPH, 2, len(ref), **kw)
    for ms, _ in res:
        for e, m in enumerate(ms):
            assert abs(m["train_loss"] - ref[e, 0]) <= 1e-12 * abs(ref[e, 0])
            assert (m["msgs_b2"], m["msgs_b4"], m["msgs_b8"]) == tuple(ref[e, 4:7])
            assert m["plan_version"] == ref[e, 8]


def test_world_split_planted_graph(cuda):
    g = generate_planted(20000, 200000, 32, 8, 8, 0.02, gamma=2.8, seed=4)
    kw = dict(dims=[32, 64, 64, 8], n_parts=8, bit_mode="fixed", fixed_bits=8, seed=3,
              owner=g["owner"])
    (base_ms, base_w), = _run_world(g, 1, 3, **kw)
    for world in (2, 8):
        for ms, w in _run_world(g, world, 3, **kw):
            assert [m["train_loss"] for m in ms] == [m["train_loss"] for m in base_ms]
            assert (w == base_w).all()


def test_negotiated_size_mismatch_is_protocol_error(cuda, monkeypatch):
    """Every rank checks its incoming pairs against the senders' all-gathered
    sizes (negotiate_buffers, plan.hpp:140-154): a disagreeing rank makes every
    rank fail with ProtocolError (engine.hpp:546-547)."""
    from paper_2306_01381_b200._lib import ProtocolError
    monkeypatch.setenv("QGNN_TEST_NEGOTIATE", "1")
    kw = dict(dims=[8, 12, 3], n_parts=4, bit_mode="fixed", fixed_bits=4, seed=11)
    with pytest.raises(AssertionError) as ei:
        _run_world(GRAPH, 2, 1, **kw)
    assert "negotiated buffer size mismatch" in str(ei.value)
    assert str(ei.value).count("ProtocolError") >= 2  # both ranks fail together
