"""World-size-2 host tests of the multi-GPU path over torch.distributed/gloo on
CPU (127.0.0.1).  The GPU engine shards the partitions over ranks and moves
packed payloads with grouped NCCL send/recv whose sizes each side derives from
its own partitions (no size handshake).  Here every rank
computes its exchange schedule with qgnn_exchange_plan and the ranks check,
through real collectives, that what one rank plans to send is exactly what its
peer plans to receive — for every key direction and bit width — plus the
bench's rendezvous helpers (unique-id broadcast, max-over-ranks timing)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_parts, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2306_01381_b200.engine import exchange_plan, generate_planted
        import bench

        g = generate_planted(3000, 24000, 8, 4, n_parts, 0.05, seed=11)
        owner = g["owner"]
        checks = 0
        for bwd in (False, True):
            for bits in (0, 2, 4, 8):
                for dim in (100, 256, 47):
                    send, recv = exchange_plan(g, owner, n_parts, world, rank, dim, bits, bwd)
                    assert send[rank] == 0 and recv[rank] == 0  # same GPU: zero copy
                    got = torch.zeros(world, dtype=torch.int64)
                    dist.all_to_all_single(got, torch.from_numpy(send.astype(np.int64)))
                    assert (got.numpy() == recv.astype(np.int64)).all(), (bwd, bits, dim, got, recv)
                    tot = torch.tensor([int(send.sum()), int(recv.sum())], dtype=torch.int64)
                    dist.all_reduce(tot)
                    assert tot[0] == tot[1] and tot[0] > 0
                    checks += 1
        # forward and backward of one key move the same number of messages
        f_send, f_recv = exchange_plan(g, owner, n_parts, world, rank, 16, 8, False)
        b_send, b_recv = exchange_plan(g, owner, n_parts, world, rank, 16, 8, True)
        assert (f_send == b_recv).all() and (f_recv == b_send).all()
        # rendezvous helpers used by bench.py under torchrun
        blob = bench.bcast_bytes(bytes(range(128)) if rank == 0 else None, world, rank)
        assert blob == bytes(range(128))
        assert bench.allmax(float(rank + 1), world) == float(world)
        bench.barrier(world)
        q.put((rank, checks, None))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, 0, repr(exc)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("n_parts", [2, 4, 8])
def test_exchange_plan_agrees_across_ranks(n_parts):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_parts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, checks, err in res:
        assert err is None, f"rank {rank}: {err}"
        assert checks == 24


def test_exchange_plan_world_one_is_all_local():
    sys.path.insert(0, ROOT)
    from paper_2306_01381_b200.engine import exchange_plan, generate_planted
    g = generate_planted(2000, 12000, 8, 4, 4, 0.05, seed=3)
    send, recv = exchange_plan(g, g["owner"], 4, 1, 0, 64, 8)
    assert send.tolist() == [0] and recv.tolist() == [0]
    with pytest.raises(ValueError):
        exchange_plan(g, g["owner"], 4, 3, 0, 64, 8)  # 4 partitions do not split over 3 ranks
