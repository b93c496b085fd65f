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


# ---------------------------------------------------------------- merge exchange plan (host logic)
W_NODE, W_BIN = 3, 4


def _records(rank, P):
    """Rank `rank`'s synthetic node / bin records (u64 words; word 1 = the hash's high word, as in
    merge.cu), deterministic per rank so every peer can regenerate what it should receive."""
    import numpy as np
    rng = np.random.default_rng(100 + rank)
    nodes = rng.integers(0, 2**63, size=(1000 + 37 * rank, W_NODE), dtype=np.int64).view(np.uint64)
    bins = rng.integers(0, 2**63, size=(5000 + 11 * rank, W_BIN), dtype=np.int64).view(np.uint64)
    own_n = np.array([(int(h) * P) >> 64 for h in nodes[:, 1]], np.int64)  # owner = floor(h_hi * P / 2^64)
    own_b = np.array([(int(h) * P) >> 64 for h in bins[:, 0]], np.int64)
    # slabs: records grouped by destination (stable), as k_part_nodes / k_part_bins lay them out
    return nodes[np.argsort(own_n, kind="stable")], np.sort(own_n), bins[np.argsort(own_b, kind="stable")], np.sort(own_b)


def _plan(P, send, recv):
    import ctypes
    import numpy as np
    from paper_2411_02797_b200 import _lib
    L = ctypes.CDLL(_lib.SO_PATH)  # dc_merge_plan is host-only: no device needed
    so, ro, tot = np.zeros(2 * P, np.uint64), np.zeros(2 * P, np.uint64), np.zeros(2, np.uint64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.dc_merge_plan(ctypes.c_uint32(P), p(send), p(recv), p(so), p(ro), p(tot))
    return st, so, ro, tot


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import numpy as np
    dist.init_process_group("gloo")
    try:
        P = world
        nodes, own_n, bins, own_b = _records(rank, P)
        send = np.zeros(2 * P, np.uint64)
        send[0::2] = np.bincount(own_n, minlength=P)
        send[1::2] = np.bincount(own_b, minlength=P)
        # step 4a: all-to-all of the counts (dc_cct_merge_ranks: ncclAlltoAll of 2 x u64 per peer)
        rc = torch.empty(2 * P, dtype=torch.int64)
        dist.all_to_all_single(rc, torch.from_numpy(send.view(np.int64).copy()))
        recv = rc.numpy().view(np.uint64).copy()
        st, so, ro, tot = _plan(P, send, recv)
        assert st == 0
        # step 4b: the slabs, with the plan's offsets (grouped send / recv in dc_cct_merge_ranks)
        out = {}
        for k, (recs, W) in enumerate([(nodes, W_NODE), (bins, W_BIN)]):
            sc, rcn = send[k::2].astype(np.int64), recv[k::2].astype(np.int64)
            assert (so[k::2].astype(np.int64) == np.concatenate([[0], np.cumsum(sc)[:-1]])).all()
            buf = torch.empty(int(tot[k]) * W, dtype=torch.int64)
            dist.all_to_all_single(buf, torch.from_numpy(recs.view(np.int64).reshape(-1).copy()),
                                   output_split_sizes=(rcn * W).tolist(), input_split_sizes=(sc * W).tolist())
            got = buf.numpy().view(np.uint64).reshape(-1, W)
            ok = True
            for src in range(P):  # what src must have sent me, regenerated locally
                s_nodes, s_own_n, s_bins, s_own_b = _records(src, P)
                srecs, sown = (s_nodes, s_own_n) if k == 0 else (s_bins, s_own_b)
                exp = srecs[sown == rank]
                o = int(ro[2 * src + k])
                ok &= bool(np.array_equal(got[o:o + len(exp)], exp))
            out[k] = (ok, int(tot[k]), int(sum(rcn)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_merge_exchange_plan():
    """dc_cct_merge_ranks' host logic (counts all-to-all + libdc's dc_merge_plan offsets + slab
    exchange) on a real world-size-2 process group (gloo on CPU): every rank receives exactly
    the records its peers route to it (owner = floor(h_hi * P / 2^64)), each source's block at the
    plan's receive offset, totals consistent."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=100) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    for r in range(world):
        for k in (0, 1):
            ok, tot, s = res[r][k]
            assert ok and tot == s


def test_merge_plan_single_rank_and_args():
    import numpy as np
    st, so, ro, tot = _plan(1, np.array([5, 7], np.uint64), np.array([5, 7], np.uint64))
    assert st == 0 and so.tolist() == [0, 0] and ro.tolist() == [0, 0] and tot.tolist() == [5, 7]
    st, so, ro, tot = _plan(3, np.array([1, 2, 3, 4, 5, 6], np.uint64), np.array([6, 5, 4, 3, 2, 1], np.uint64))
    assert so.tolist() == [0, 0, 1, 2, 4, 6] and ro.tolist() == [0, 0, 6, 5, 10, 8] and tot.tolist() == [12, 9]
