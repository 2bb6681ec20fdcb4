"""K2 exchange through the C-ABI (qgnn_comm_* / qgnn_exchange) and the engine's
NCCL transport on one device.

The reference simulates the exchange (commsim/exchange.hpp:45-78, an in-process
mailbox at trainer/engine.hpp:502 / :528-529).  Here it is a grouped NCCL
send/receive (or the in-process loopback transport for ranks-as-threads on one
GPU).  On a single B200 NCCL runs as a one-rank communicator: every pair of the
engine's partitions goes through ncclSend/ncclRecv to self, which executes the
same grouped point-to-point code as the multi-GPU run.
"""
import os
import threading

import numpy as np
import pytest
import torch

from paper_2306_01381_b200 import _lib, ops
from paper_2306_01381_b200.engine import Engine, loopback_id

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
GRAPH = {k: G[f"g_{k}"] for k in ("adj_ptr", "adj", "features", "labels", "train", "val", "test")}


def _layout(sizes):
    off = np.zeros(len(sizes), np.uint64)
    o = 0
    for i, s in enumerate(sizes):
        off[i] = o
        o = (o + int(s) + 255) // 256 * 256
    return off, max(o, 256)


def test_exchange_nccl_world1_self(cuda):
    comm = ops.Comm(world=1, rank=0)
    rs = np.random.default_rng(0)
    n = 1_000_003
    src = torch.as_tensor(rs.integers(0, 256, n + 64, dtype=np.uint8), device="cuda")
    dst = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    comm.exchange(src, [17], [n], dst, [5], [n])
    torch.cuda.synchronize()
    assert torch.equal(dst[5:5 + n], src[17:17 + n])
    assert int(dst[:5].sum()) == 0 and int(dst[5 + n:].sum()) == 0
    comm.close()


def _loop_run(world, sizes, group, corrupt=None):
    """sizes[a][b] = bytes rank a sends to rank b; returns per-rank (recv, expected) or errors."""
    lid = loopback_id(group)
    out, errs = [None] * world, [None] * world

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            comm = ops.Comm(world=world, rank=r, id128=lid)
            s_off, s_tot = _layout(sizes[r])
            rcv = [sizes[a][r] for a in range(world)]
            if corrupt is not None and r == corrupt:
                rcv[(r + 1) % world] += 1
            r_off, r_tot = _layout(rcv)
            g = torch.Generator(device="cpu").manual_seed(100 + r)
            send = torch.randint(0, 256, (s_tot,), dtype=torch.uint8, generator=g).cuda()
            recv = torch.zeros(r_tot, dtype=torch.uint8, device="cuda")
            for _ in range(3):  # reuse the buffers: each call waits for the previous readers
                comm.exchange(send, s_off, sizes[r], recv, r_off, rcv)
            torch.cuda.synchronize()
            out[r] = (send.cpu(), s_off, recv.cpu(), r_off)
            comm.close()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out, errs


def test_exchange_loopback_all_to_all_v(cuda):
    world = 4
    rs = np.random.default_rng(3)
    sizes = rs.integers(0, 50_000, (world, world))
    sizes[1][2] = 0  # empty pairs are skipped on both sides
    out, errs = _loop_run(world, sizes, group=9001)
    assert errs == [None] * world, errs
    for b in range(world):
        _, _, recv, r_off = out[b]
        for a in range(world):
            send, s_off, _, _ = out[a]
            n = int(sizes[a][b])
            got = recv[int(r_off[a]):int(r_off[a]) + n]
            exp = send[int(s_off[b]):int(s_off[b]) + n]
            assert torch.equal(got, exp), (a, b)


def test_exchange_loopback_size_mismatch_is_protocol_error(cuda):
    world = 3
    sizes = np.full((world, world), 1000)
    _, errs = _loop_run(world, sizes, group=9002, corrupt=1)
    assert all(isinstance(e, _lib.ProtocolError) for e in errs), errs


def _engine_run(transport, epochs=4, kstats=False, graph=GRAPH, dims=(8, 12, 3), parts=4,
                **kw):
    eng = Engine(graph, list(dims), n_parts=parts, bit_mode="fixed", fixed_bits=4, seed=11,
                 dtype="f32", transport=transport, kstats=kstats, **kw)
    ms = [eng.run_epoch() for _ in range(epochs)]
    w = np.concatenate([x.reshape(-1) for x in eng.weights()])
    ks = eng.kernel_stats() if kstats else None
    eng.close()
    return ms, w, ks


@pytest.mark.parametrize("kstats", [False, True])
def test_engine_nccl_transport_bit_identical(cuda, kstats):
    """Every partition pair through NCCL self send/receive (replayed in the CUDA
    graph when kstats is off) gives the zero-copy run's bits."""
    a, wa, _ = _engine_run("zero_copy", kstats=kstats)
    b, wb, ks = _engine_run("nccl", kstats=kstats)
    assert [m["train_loss"] for m in a] == [m["train_loss"] for m in b]
    assert [m["bytes_total"] for m in a] == [m["bytes_total"] for m in b]
    assert (wa == wb).all()
    if kstats:
        assert ks["exchange"]["bytes"] > 0 and ks["exchange"]["ms"] > 0
        assert b[-1]["ms_exchange"] > 0


def test_engine_nccl_transport_serialized_overlap_identical(cuda):
    a, wa, _ = _engine_run("nccl", overlap=1)
    b, wb, _ = _engine_run("nccl", overlap=0)
    assert [m["train_loss"] for m in a] == [m["train_loss"] for m in b]
    assert (wa == wb).all()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (NCCL over NVLink)")
def test_exchange_nccl_multi_gpu():
    """Real NCCL p2p between GPUs (one process per GPU, spawned)."""
    import torch.multiprocessing as mp
    from paper_2306_01381_b200.engine import nccl_unique_id
    world = min(4, torch.cuda.device_count())
    nid = nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_mp_rank, args=(r, world, nid, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for ok in res), res


def _mp_rank(rank, world, nid, q):
    try:
        torch.cuda.set_device(rank)
        comm = ops.Comm(world=world, rank=rank, id128=nid, device=rank)
        n = 1 << 20
        send = torch.full((world * n,), rank, dtype=torch.uint8, device="cuda")
        for b in range(world):
            send[b * n:(b + 1) * n] += 16 * b
        recv = torch.zeros(world * n, dtype=torch.uint8, device="cuda")
        off = [b * n for b in range(world)]
        comm.exchange(send, off, [n] * world, recv, off, [n] * world)
        torch.cuda.synchronize()
        ok = all(int(recv[a * n]) == a + 16 * rank for a in range(world))
        comm.close()
        q.put(ok)
    except Exception as e:  # noqa: BLE001
        q.put(repr(e))


@pytest.mark.parametrize("skew,transport", [("source", "zero_copy"), ("version", "zero_copy"),
                                            ("source", "nccl")])
def test_envelope_mismatch_is_protocol_error(cuda, monkeypatch, skew, transport):
    """Senders stamp a wrong source / plan version into the chunk envelope; the
    receivers' K3 rejects it: ProtocolError ("misrouted payload" / "plan version
    skew", engine.hpp:530-541) at the phase boundary."""
    monkeypatch.setenv("QGNN_TEST_ENVELOPE", skew)
    monkeypatch.setenv("QGNN_GRAPH", "0")
    eng = Engine(GRAPH, [8, 12, 3], n_parts=4, bit_mode="fixed", fixed_bits=8, seed=11,
                 dtype="f32", transport=transport)
    with pytest.raises(_lib.ProtocolError):
        eng.run_epoch()
    eng.close()


def test_envelope_through_the_c_abi(cuda):
    """qgnn_quantize_pack stamps (source, set, version); qgnn_dequant_scatter with
    the matching expectation decodes, a wrong one latches ProtocolError."""
    x = torch.randn((6, 32), device=cuda)
    wire, idx = ops.encode_message_set(x, list(range(6)), list(range(6)), [8] * 6, 5)
    # re-encode with an envelope: source 3, version 7 (set index 0)
    keys = torch.as_tensor(np.array([5], np.uint64).view(np.int64), device=cuda)
    rows = torch.arange(6, dtype=torch.int32, device=cuda)
    bits_t = torch.full((6,), 8, dtype=torch.uint8, device=cuda)
    off_t = torch.as_tensor(idx["off"].astype(np.int64), device=cuda)
    out = torch.zeros_like(wire)
    ops.quantize_pack(x, rows, rows, bits_t, off_t, keys, out, envelope=3 | 7 << 8)
    good = torch.full((6,), 3 | 0 << 8 | 7 << 16, dtype=torch.int32, device=cuda)
    dec = torch.zeros((6, 32), device=cuda)
    ops.dequant_scatter(out, bits_t, off_t, 32, dec, expect_envelope=good)
    ref = ops.decode_message_set(wire, idx["bits"], idx["off"], 32)
    assert torch.equal(dec, ref)  # the envelope does not change the payload
    bad = good.clone()
    bad[4] += 1 << 16  # plan version 8 expected
    with pytest.raises(_lib.ProtocolError):
        ops.dequant_scatter(out, bits_t, off_t, 32, dec, expect_envelope=bad)
