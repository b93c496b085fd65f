"""Test helpers: run the same seeded trace through the CUDA path (C ABI) and the oracle."""
from __future__ import annotations

import numpy as np
import torch

import oracle

CMP_KEYS = ["parent", "frame", "depth", "xcnt", "icnt", "xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo",
            "isq_hi", "xsamples", "isamples", "xstall", "istall", "pc_ctx", "pc_off", "bin_pcnode", "bin_stall", "bin_count"]


def as_u64(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.int64 else a.astype(np.uint64)


def gpu_run(offsets, frames=None, metrics=None, keys=None, n_frames=None, samples=None, n_launch=None, launch_off=None,
            n_stall=24, kinds=None, views=None, ctx=None):
    """Runs intern (if keys) -> build -> attribute -> [pc] -> rollup on cuda:0.
    Returns (arrays, leaf, extras). frames/keys are numpy or torch (CPU)."""
    import paper_2411_02797_b200 as dc
    ctx = ctx or dc.Context(0)
    dev = "cuda:0"
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
    off = t(offsets, np.int64)
    d = None
    ids_np = None
    if keys is not None:
        kk = torch.from_numpy(np.ascontiguousarray(np.asarray(keys)).view(np.int32).reshape(-1, 4)).to(dev)
        ids, d = dc.dc_intern_frames(ctx, kk)
        n_frames = d.size
        fr = ids
        ids_np = ids.cpu().numpy().view(np.uint32)
    else:
        fr = t(np.asarray(frames, np.uint32), np.int32) if len(frames) else torch.zeros(1, dtype=torch.int32, device=dev)
        if kinds is not None:
            pass
    cct, leaf = dc.dc_cct_build(ctx, off, fr, n_frames, d)
    if metrics is not None:
        X = t(as_u64(metrics), np.int64)
        dc.dc_cct_attribute_metrics(ctx, cct, leaf, X)
    if samples is not None:
        S = torch.from_numpy(np.ascontiguousarray(np.asarray(samples)).view(np.int32).reshape(-1, 4)).to(dev)
        lo = t(np.asarray(launch_off, np.uint64), np.int64) if launch_off is not None else None
        nl = n_launch if n_launch is not None else len(offsets) - 1
        dc.dc_pc_sample_attribute(ctx, cct, S, leaf[:nl] if nl else leaf, lo, n_stall=n_stall, n_launch=nl)
    dc.dc_cct_rollup(ctx, cct)
    a = cct.to_numpy()
    a["leaf"] = leaf.cpu().numpy().view(np.uint32)
    a["ids"] = ids_np
    a["_cct"], a["_ctx"], a["_dict"] = cct, ctx, d
    return a


def oracle_run(offsets, frames, metrics, n_metrics, samples=None, n_launch=0, n_stall=24):
    if samples is None:
        n_stall = 0  # no PC columns, as on the GPU side
    o = oracle.OracleCCT(n_metrics, n_stall).insert(np.asarray(offsets).view(np.uint64) if np.asarray(offsets).dtype == np.int64
                                                    else offsets, frames, as_u64(metrics))
    if samples is not None:
        o.pc(samples, n_launch)
    return o.finalize()


def assert_same(got: dict, ref: dict, keys=CMP_KEYS, ctx=""):
    assert got["n_nodes"] == ref["n_nodes"], f"{ctx}: n_nodes {got['n_nodes']} != {ref['n_nodes']}"
    for k in keys:
        g, r = np.asarray(got[k]), np.asarray(ref[k])
        if g.size == 0 and r.size == 0:
            continue
        assert g.shape == r.shape, f"{ctx}: {k} shape {g.shape} != {r.shape}"
        if not np.array_equal(g, r):
            bad = np.argwhere(g != r)[:5]
            raise AssertionError(f"{ctx}: {k} differs at {bad.tolist()}: got {g[tuple(bad[0])]} ref {r[tuple(bad[0])]}")
    if "level_off" in got:  # level_off[d] = first node of depth >= d (depth is non-decreasing)
        dep, lo = np.asarray(got["depth"]), np.asarray(got["level_off"])
        assert np.array_equal(lo, np.searchsorted(dep, np.arange(len(lo)), side="left")), f"{ctx}: level_off"
    if "leaf" in ref and ref["leaf"] is not None and "leaf" in got:
        assert np.array_equal(got["leaf"], ref["leaf"]), f"{ctx}: leaf differs"
