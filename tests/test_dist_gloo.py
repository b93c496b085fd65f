"""world_size-2 gloo tests on CPU for the multi-process host logic (rendezvous on 127.0.0.1)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2411_02797_b200 import dist as dd
    r, w, lr = dd.init("gloo")
    try:
        out = {}
        out["max"] = dd.max_over_ranks(1.5 + r, device="cpu")
        uid = bytes(range(128)) if r == 0 else None
        out["uid"] = dd.broadcast_bytes(uid, 0, device="cpu")
        out["shards"] = dd.shards_for_rank(8, r, w)
        out["rw"] = (r, w, lr)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_host_logic():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=100) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["max"] == 2.5                      # max over ranks
        assert res[r]["uid"] == bytes(range(128))        # the NCCL unique id reaches every rank
        assert res[r]["rw"] == (r, world, r)
    assert res[0]["shards"] == [0, 2, 4, 6] and res[1]["shards"] == [1, 3, 5, 7]
    assert sorted(res[0]["shards"] + res[1]["shards"]) == list(range(8))


def test_single_process_defaults():
    from paper_2411_02797_b200 import dist as dd
    assert dd.max_over_ranks(3.0) == 3.0 and dd.broadcast_bytes(b"x" * 128) == b"x" * 128
    assert dd.shards_for_rank(5, 0, 1) == [0, 1, 2, 3, 4]
    assert torch.distributed.is_available()
