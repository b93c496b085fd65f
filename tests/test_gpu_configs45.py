"""GPU parity on BASELINE.json configs 4 (JAX-compiled-graph-shaped, depth up to 256) and 5
(DDP-style shards with per-shard dictionaries, merged across ranks).

- Config 4 prefix (2M records, all 41.5k launch sites, static + dynamic recursion up to
  depth 256): CUDA path vs the oracle element by element.
- Config 4 at full size (200M records, 9.2G frame entries) in the bench's launch
  configuration: properties that hold at any size (SURVEY §8(c) "Any size" invariants), all
  exact on integers and computed here with numpy / torch reductions that share nothing with
  the library.
- Config 5: per-shard CCTs built from each shard's own raw keys and dictionary, merged with
  the emulated-rank exchange (dc_cct_merge_local); the result must equal the oracle's CCT of
  the concatenated shards (reading R19), dictionary included.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from pipeline import CMP_KEYS, as_u64, assert_same, gpu_run, oracle_run

pytestmark = pytest.mark.gpu
NOPC = [k for k in CMP_KEYS if "samples" not in k and "stall" not in k and "pc" not in k and "bin" not in k]


@pytest.mark.parametrize("rollup", ["levels", "push"])
def test_config4_prefix_vs_oracle(rollup, monkeypatch):
    if rollup == "push":
        monkeypatch.setenv("DC_TEST_ROLLUP_PUSH", "1")
    p = gen.programs.config4()
    tr = gen.make_trace(p, n_records=2_000_000, raw_keys=False)
    off = tr.offsets.numpy().view(np.uint64)
    assert int(np.diff(off).max()) == 256
    a = gpu_run(off, tr.ids.numpy().view(np.uint32), tr.metrics.numpy(), n_frames=tr.n_frames)
    ref = oracle_run(off, tr.ids.numpy().view(np.uint32), tr.metrics.numpy(), p.n_metrics).arrays()
    assert_same(a, ref, keys=NOPC, ctx="cfg4 prefix")
    assert a["max_depth"] == 256


def _invariants(a, R, Xsum):
    N = a["n_nodes"]
    par = a["parent"].astype(np.int64)
    dep = a["depth"].astype(np.int64)
    fr = a["frame"].astype(np.int64)
    ids = np.arange(N)
    assert par[0] == 0xFFFFFFFF and dep[0] == 0
    assert (par[1:] < ids[1:]).all()
    assert (dep[1:] == dep[par[1:]] + 1).all()
    assert (np.diff(dep) >= 0).all()  # levels contiguous
    # siblings: frames strictly ascending within one parent (children contiguous, parents ascending)
    same = par[2:] == par[1:-1]
    assert (np.diff(par[1:]) >= 0).all()
    assert (fr[2:][same] > fr[1:-1][same]).all()
    # incl = excl (+) sum of children incl, exactly
    icnt, xcnt = a["icnt"].astype(object), a["xcnt"].astype(object)
    kid_cnt = np.zeros(N, dtype=object)
    np.add.at(kid_cnt, par[1:], icnt[1:])
    assert (icnt == xcnt + kid_cnt).all()
    for m in range(a["n_metrics"]):
        isum, xsum = a["isum"][m].astype(object), a["xsum"][m].astype(object)
        ks = np.zeros(N, dtype=object)
        np.add.at(ks, par[1:], isum[1:])
        assert (isum == xsum + ks).all()
        imin, xmin = a["imin"][m], a["xmin"][m]
        km = np.full(N, np.iinfo(np.uint64).max, np.uint64)
        np.minimum.at(km, par[1:], imin[1:])
        assert (imin == np.minimum(xmin, km)).all()
        isq = (a["isq_hi"][m].astype(object) << 64) + a["isq_lo"][m].astype(object)
        xsq = (a["xsq_hi"][m].astype(object) << 64) + a["xsq_lo"][m].astype(object)
        kq = np.zeros(N, dtype=object)
        np.add.at(kq, par[1:], isq[1:])
        assert (isq == xsq + kq).all()
        assert int(isum[0]) == Xsum[m]
        assert int(xsum.sum()) == Xsum[m]
    assert int(icnt[0]) == R and int(xcnt.sum()) == R


def test_config4_full_size_invariants():
    """200M records exactly as bench.py --config 4 builds them (pre-interned ids, dictionary
    from the sorted pool keys)."""
    import paper_2411_02797_b200 as dc
    p = gen.programs.config4()
    tr = gen.make_trace(p, device="cuda", raw_keys=False)
    R = tr.n_records
    assert R == 200_000_000
    ctx = dc.Context(0)
    keys = torch.from_numpy(np.ascontiguousarray(p.pool_keys).view(np.int32).reshape(-1, 4).copy()).cuda()
    d = dc.dc_dict_from_sorted(ctx, keys)
    cct, leaf = dc.dc_cct_build(ctx, tr.offsets, tr.ids, tr.n_frames, d)
    dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics)
    dc.dc_cct_rollup(ctx, cct)
    a = cct.to_numpy()
    # per-metric totals by a plain reduction of the input columns (int64 is exact here: < 2^63)
    Xsum = [int(tr.metrics[m].sum().item()) for m in range(p.n_metrics)]
    _invariants(a, R, Xsum)
    assert a["max_depth"] == 256
    # every record's leaf sits at the depth of its path length
    lens = (tr.offsets[1:] - tr.offsets[:-1]).to(torch.int64)
    dep = torch.from_numpy(a["depth"].astype(np.int64)).cuda()
    lf = leaf[:R].to(torch.int64) & 0xFFFFFFFF
    assert bool((dep[lf] == lens).all())
    # exact parity for sampled records: the path of the leaf, walked up the node table, is
    # the record's frame sequence
    rng = np.random.default_rng(0)
    off = tr.offsets
    lf_h = lf.cpu().numpy()
    for r in rng.choice(R, size=64, replace=False).tolist():
        path = tr.ids[int(off[r]):int(off[r + 1])].cpu().numpy().view(np.uint32).tolist()
        n, walk = int(lf_h[r]), []
        while n != 0:
            walk.append(int(a["frame"][n]))
            n = int(a["parent"][n])
        assert walk[::-1] == path
    cct.free()


def test_config5_shards_merge_vs_oracle():
    """Three config-5 shards (each its own program seed and rank-local frames, own raw-key
    dictionary) -> local CCTs -> merge == oracle over the concatenated trace."""
    import paper_2411_02797_b200 as dc
    from test_gpu_merge import _shard_run
    ctx = dc.Context(0)
    trs = [gen.make_trace(gen.programs.config5(s), n_records=60_000 + 7_000 * s) for s in range(3)]
    parts = []
    for tr in trs:
        parts.append(_shard_run(dc, ctx, tr.keys.numpy(), tr.offsets.numpy().view(np.uint64),
                                tr.metrics.numpy().view(np.uint64)))
    merged, gd = dc.dc_cct_merge_local(ctx, [c for c, _ in parts], [d for _, d in parts])
    # oracle over the concatenation
    offs, base = [np.zeros(1, np.uint64)], 0
    for tr in trs:
        o = tr.offsets.numpy().view(np.uint64)
        offs.append(o[1:] + np.uint64(base))
        base += int(o[-1])
    off = np.concatenate(offs)
    keys = np.concatenate([tr.keys.numpy() for tr in trs])
    X = np.concatenate([as_u64(tr.metrics.numpy()) for tr in trs], axis=1)
    ids, od = oracle.intern(keys)
    ref = oracle_run(off, ids, X, 2).arrays()
    assert np.array_equal(gd.keys(), od)
    assert_same(merged.to_numpy(), ref, keys=NOPC, ctx="cfg5 merge")
