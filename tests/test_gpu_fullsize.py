"""Full-size parity on BASELINE.json configs 3, 4 and 5, in the launch configuration bench.py
times (north_star: "bit-exact CCT and metric views versus the CPU oracle on all five configs").

- Config 3 (100M PC samples, 20k launch records): bench.py's own workload and step
  (bench.make_workload / bench.run_step: intern -> build -> attribute -> PC histogram with the
  per-launch offsets -> rollup -> views), compared ELEMENT BY ELEMENT with the oracle run on
  the same trace generated on the host: every CCT array, the leaves, the interned ids, the
  dictionary, the views and the derived floats.
- Config 4 (200M records, depth <= 256, 9.2G frame entries) and config 5 (8 shards x 125M
  records with per-shard raw-key dictionaries, merged over 8 emulated ranks): the canonical
  SHA-256 digest of the whole CCT against the oracle's digest cached in
  tests/golden/digest_cfg{4,5}.json by tools/golden_digest.py (oracle/ + gen/ only; the
  oracle takes minutes on these), plus the leaves (config 4) and sampled derived floats.
"""
import json
import os
import sys

import numpy as np
import pytest
import torch

import gen
import oracle
from pipeline import CMP_KEYS, assert_same

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _golden(cfg):
    path = os.path.join(GOLD, f"digest_cfg{cfg}.json")
    g = json.load(open(path))
    assert g["generator_version"] == gen.generator_version(), \
        f"{path} is stale (generator changed): rerun tools/golden_digest.py {cfg}"
    return g


def _check_derived(dc, ctx, cct, g):
    nodes = torch.tensor(g["derived"]["nodes"], dtype=torch.int64, device="cuda")
    for m in range(g["n_metrics"]):
        for incl in (True, False):
            mean, std = dc.dc_cct_derived(ctx, cct, m, incl)
            ref = np.asarray(g["derived"][f"m{m}_{'incl' if incl else 'excl'}"], np.float64)
            got = np.stack([mean[nodes].cpu().numpy(), std[nodes].cpu().numpy()], 1)
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)


def test_full_size_config3_every_array_vs_oracle():
    import bench
    import paper_2411_02797_b200 as dc
    p, tr = bench.make_workload(3, 0, "cuda:0")
    F = int(tr.offsets[-1].item())
    tr.ids_buf = torch.empty(F, dtype=torch.int32, device="cuda")
    tr.leaf_buf = torch.empty(tr.n_records, dtype=torch.int32, device="cuda")
    ctx = dc.Context(0)
    cct, views = bench.run_step(dc, ctx, tr, 3)
    got = cct.to_numpy()
    got["leaf"] = tr.leaf_buf.cpu().numpy().view(np.uint32)
    gpu_ids = tr.ids_buf.cpu().numpy().view(np.uint32)
    diag = ctx.diag()
    # the same trace on the host (byte-identical generator), through the oracle
    h = gen.make_trace(p, pc=True)
    assert torch.equal(h.samples.cuda(), tr.samples) and torch.equal(h.keys.cuda(), tr.keys)
    oids, od = oracle.intern(h.keys.numpy())
    assert np.array_equal(gpu_ids, oids)
    o = oracle.OracleCCT(p.n_metrics, 24).insert(h.offsets.numpy(), oids, h.metrics.numpy())
    o.pc(h.samples.numpy(), h.n_launch)
    ref = o.finalize().arrays()
    assert got["n_pc_nodes"] == ref["n_pc_nodes"] and got["n_bins"] == ref["n_bins"]
    assert_same(got, ref, keys=CMP_KEYS, ctx="config 3 full size")
    assert ref["n_bins"] > 2_900_000 and int(ref["isamples"][0]) == 100_000_000
    od_ = o.diag()
    assert (diag["samples_bad_launch"], diag["samples_bad_stall"], diag["samples_zero_count"]) == \
        (od_["samples_bad_launch"], od_["samples_bad_stall"], od_["samples_zero_count"])
    # dictionary and views
    _, d = dc.dc_intern_frames(ctx, tr.keys)
    assert np.array_equal(d.keys(), od)
    kinds = np.asarray(od["kind"], np.uint8)
    oh = o.topk(oracle.VIEW_INCLUSIVE, 0, 1 << dc.DC_KIND_KERNEL, kinds, 0.01, 10)
    assert views["hotspots"] == [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in oh]
    os_ = o.topk(oracle.VIEW_STALL, k=5, stall_node=int(oh[0]["id"]))
    assert views["stall"] == [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in os_]
    for m in range(p.n_metrics):
        mean, std = dc.dc_cct_derived(ctx, cct, m, True)
        rm, rs = o.derived(m, True)
        np.testing.assert_allclose(mean.cpu().numpy(), rm, rtol=1e-12, atol=0)
        np.testing.assert_allclose(std.cpu().numpy(), rs, rtol=1e-12, atol=0)
    cct.free()


def test_full_size_config4_digest():
    import paper_2411_02797_b200 as dc
    g = _golden(4)
    p = gen.programs.config4()
    tr = gen.make_trace(p, device="cuda", raw_keys=False)
    assert tr.n_records == g["records"] == 200_000_000
    ctx = dc.Context(0)
    keys = torch.from_numpy(np.ascontiguousarray(p.pool_keys).view(np.int32).reshape(-1, 4).copy()).cuda()
    d = dc.dc_dict_from_sorted(ctx, keys)
    cct, leaf = dc.dc_cct_build(ctx, tr.offsets, tr.ids, tr.n_frames, d)
    dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics)
    dc.dc_cct_rollup(ctx, cct)
    del tr
    v = cct.view()
    assert (v.n_nodes, v.max_depth) == (g["n_nodes"], g["max_depth"])
    assert cct.digest(d) == g["sha256"]
    assert _leaf_sha256(leaf) == g["leaf_sha256"]
    _check_derived(dc, ctx, cct, g)
    cct.free()


def _leaf_sha256(leaf: torch.Tensor) -> str:
    import hashlib
    return hashlib.sha256(leaf.cpu().numpy().view(np.uint32).tobytes()).hexdigest()


def test_full_size_config5_eight_shard_merge_digest():
    """8 shards x 125M records, each interned from its own raw keys and built into a local CCT,
    then merged over 8 emulated ranks (dc_cct_merge_local: partition, exchange, reduce with
    exact verification, canonical gather); equals the oracle over the 1B-record concatenation."""
    import paper_2411_02797_b200 as dc
    g = _golden(5)
    ctx = dc.Context(0)
    parts, dicts = [], []
    for s in range(g["shards"]):
        p = gen.programs.config5(s)
        tr = gen.make_trace(p, device="cuda")
        ids, d = dc.dc_intern_frames(ctx, tr.keys)
        cct, leaf = dc.dc_cct_build(ctx, tr.offsets, ids, d.size, d)
        dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics)
        dc.dc_cct_rollup(ctx, cct)
        ctx.sync()
        parts.append(cct)
        dicts.append(d)
        del tr, ids, leaf
        torch.cuda.empty_cache()
    merged, gd = dc.dc_cct_merge_local(ctx, parts, dicts)
    v = merged.view()
    assert (v.n_nodes, gd.size) == (g["n_nodes"], g["n_frames"])
    assert merged.digest(gd) == g["sha256"]
    _check_derived(dc, ctx, merged, g)
