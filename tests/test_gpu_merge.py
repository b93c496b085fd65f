"""Cross-rank merge (a9) on one GPU through the emulated-rank loopback (dc_cct_merge_local):
the merged canonical CCT of P shards must equal the oracle's CCT of the concatenated trace
(reading R19) — the oracle has no merge code at all."""
import numpy as np
import pytest
import torch

import gen
import oracle
from pipeline import assert_same

pytestmark = pytest.mark.gpu


def _shard_run(dc, ctx, keys, off, X, samples=None, launch_off=None, n_stall=24):
    dev = "cuda:0"
    kk = torch.from_numpy(np.ascontiguousarray(keys).view(np.int32).reshape(-1, 4)).to(dev)
    o = torch.from_numpy(np.ascontiguousarray(off).view(np.int64)).to(dev)
    ids, d = dc.dc_intern_frames(ctx, kk)
    cct, leaf = dc.dc_cct_build(ctx, o, ids, d.size, d)
    dc.dc_cct_attribute_metrics(ctx, cct, leaf, torch.from_numpy(np.ascontiguousarray(X).view(np.int64)).to(dev))
    if samples is not None:
        s = torch.from_numpy(np.ascontiguousarray(samples).view(np.int32).reshape(-1, 4)).to(dev)
        lo = torch.from_numpy(np.ascontiguousarray(launch_off).view(np.int64)).to(dev) if launch_off is not None else None
        dc.dc_pc_sample_attribute(ctx, cct, s, leaf, lo, n_stall=n_stall)
    dc.dc_cct_rollup(ctx, cct)
    return cct, d


def _split(tr, P, with_pc=False):
    off = tr.offsets.numpy().view(np.uint64)
    keys = tr.keys.numpy()
    X = tr.metrics.numpy().view(np.uint64)
    R = len(off) - 1
    cuts = np.linspace(0, R, P + 1).astype(np.int64)
    shards = []
    for p in range(P):
        a, b = int(cuts[p]), int(cuts[p + 1])
        so = (off[a:b + 1] - off[a]).astype(np.uint64)
        sk = keys[int(off[a]):int(off[b])]
        sx = np.ascontiguousarray(X[:, a:b])
        sh = dict(off=so, keys=sk, X=sx)
        if with_pc:
            lo = tr.launch_off.numpy().view(np.uint64)
            S = tr.samples.numpy()
            ss = S[int(lo[a]):int(lo[b])].copy()
            ss[:, 0] -= a  # launch index local to the shard
            sh.update(samples=ss, launch_off=(lo[a:b + 1] - lo[a]).astype(np.uint64))
        shards.append(sh)
    return shards


def _oracle_concat(tr, M, with_pc=False):
    ids, d = oracle.intern(tr.keys.numpy())
    o = oracle.OracleCCT(M, 24).insert(tr.offsets.numpy(), ids, tr.metrics.numpy())
    if with_pc:
        o.pc(tr.samples.numpy(), tr.n_records)
    return o.finalize(), d


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_merge_local_config1(P):
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    p = gen.programs.program(1)
    tr = gen.make_trace(p)
    parts = [_shard_run(dc, ctx, **sh) for sh in _split(tr, P)]
    merged, gd = dc.dc_cct_merge_local(ctx, [c for c, _ in parts], [d for _, d in parts])
    o, od = _oracle_concat(tr, p.n_metrics)
    ref = o.arrays()
    got = merged.to_numpy()
    assert np.array_equal(gd.keys(), od)
    keys = ["parent", "frame", "depth", "xcnt", "icnt", "xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]
    assert_same(got, ref, keys=keys, ctx=f"merge P={P}")
    # views on the merged tree equal the oracle's
    fk = np.asarray(od["kind"], np.uint8)
    hot = dc.dc_hotspots_topk(ctx, merged, dc.DC_VIEW_INCLUSIVE, 0, 1 << 4, 0.001, 10)
    exp = o.topk(oracle.VIEW_INCLUSIVE, 0, 1 << 4, fk, 0.001, 10)
    assert hot == [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in exp]


def test_merge_local_with_pc_samples():
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    p = gen.programs.config3(n_samples=3_000_000)
    tr = gen.make_trace(p, pc=True, bad_per_million=300)
    P = 4
    parts = [_shard_run(dc, ctx, **sh) for sh in _split(tr, P, with_pc=True)]
    merged, gd = dc.dc_cct_merge_local(ctx, [c for c, _ in parts], [d for _, d in parts])
    o, od = _oracle_concat(tr, p.n_metrics, with_pc=True)
    assert_same(merged.to_numpy(), o.arrays(), ctx="merge pc")


def test_merge_collision_is_detected(monkeypatch):
    """DC_TEST_WEAK_MERGE_HASH=4 keeps 4 bits of each 64-bit half: different paths collide and
    the (parent hash, frame, depth) check must refuse the merge (DC_ERR_COLLISION)."""
    monkeypatch.setenv("DC_TEST_WEAK_MERGE_HASH", "4")
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    p = gen.programs.program(1)
    tr = gen.make_trace(p, n_records=3000)
    parts = [_shard_run(dc, ctx, **sh) for sh in _split(tr, 2)]
    with pytest.raises(dc.DcError) as e:
        dc.dc_cct_merge_local(ctx, [c for c, _ in parts], [d for _, d in parts])
    assert e.value.status == 7


def test_chunked_online_aggregation_config3():
    """NEXT-1: a config-3-shaped trace ingested in 4 chunks (records + their PC samples), each
    built into its own CCT, folded with aggregate_chunks == the oracle's CCT of the whole trace."""
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    p = gen.programs.config3(n_samples=2_000_000)
    tr = gen.make_trace(p, pc=True, bad_per_million=300)
    chunks = (_shard_run(dc, ctx, **sh) for sh in _split(tr, 4, with_pc=True))
    acc, d = dc.aggregate_chunks(ctx, chunks)
    o, od = _oracle_concat(tr, p.n_metrics, with_pc=True)
    assert np.array_equal(d.keys(), od)
    assert_same(acc.to_numpy(), o.arrays(), ctx="chunked")


def test_merge_ranks_nccl_single_rank():
    """The NCCL path of dc_cct_merge_ranks / dc_cct_gather on a one-rank communicator (every
    collective and send/recv runs, to self): the gathered canonical CCT equals the oracle's."""
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    p = gen.programs.config3(n_samples=1_000_000)
    tr = gen.make_trace(p, pc=True, bad_per_million=200)
    sh = _split(tr, 1, with_pc=True)[0]
    cct, d = _shard_run(dc, ctx, **sh)
    comm = dc.dc_comm_create(ctx, dc.dc_nccl_unique_id(), 1, 0)
    part, gd = dc.dc_cct_merge_ranks(ctx, comm, cct, d)
    canon = dc.dc_cct_gather(ctx, comm, part, 0)
    o, od = _oracle_concat(tr, p.n_metrics, with_pc=True)
    assert np.array_equal(gd.keys(), od)
    assert_same(canon.to_numpy(), o.arrays(), ctx="nccl merge, 1 rank")
