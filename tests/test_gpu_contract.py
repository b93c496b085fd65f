"""GPU tests of the §8(b) handle contract (include/dc.h):
- dc_pc_sample_attribute accumulates over repeated calls (one per sample chunk / activity
  buffer): any split equals one call and the oracle;
- dc_cct_view_get reports DC_ERR_STATE (inclusive columns NULL) before dc_cct_rollup;
- argument errors (NULL frames with non-empty paths, n_stall changing between calls) are
  DC_ERR_ARG, and a failed call leaves the handle as it was."""
import numpy as np
import pytest
import torch

import gen
import oracle
from pipeline import CMP_KEYS, assert_same

pytestmark = pytest.mark.gpu


def _base(p, tr, dc, ctx):
    ids, d = dc.dc_intern_frames(ctx, tr.keys.cuda())
    cct, leaf = dc.dc_cct_build(ctx, tr.offsets.cuda(), ids, d.size, d)
    dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics.cuda())
    return cct, leaf


def _oracle(p, tr):
    oids, _ = oracle.intern(tr.keys.numpy())
    o = oracle.OracleCCT(p.n_metrics, 24).insert(tr.offsets.numpy(), oids, tr.metrics.numpy())
    o.pc(tr.samples.numpy(), tr.n_launch)
    return o.finalize().arrays(), o.diag()


@pytest.mark.parametrize("schedule", ["owner", "generic"])
def test_pc_attribute_accumulates_over_chunks(schedule):
    import paper_2411_02797_b200 as dc
    p = gen.programs.config3(n_launch=2000, n_samples=4_000_000)
    tr = gen.make_trace(p, n_records=2000, pc=True, n_launch=2000, bad_per_million=2000)
    ref, odiag = _oracle(p, tr)
    ctx = dc.Context(0)
    S = tr.samples.cuda()
    lo = tr.launch_off.cpu().numpy().view(np.uint64).astype(np.int64)
    # one call
    one, leaf = _base(p, tr, dc, ctx)
    dc.dc_pc_sample_attribute(ctx, one, S, leaf, tr.launch_off.cuda() if schedule == "owner" else None, n_stall=24)
    dc.dc_cct_rollup(ctx, one)
    a1 = one.to_numpy()
    # four calls: launch ranges (owner: each with its own rebased per-launch offsets), or
    # arbitrary sample ranges (generic)
    many, leaf2 = _base(p, tr, dc, ctx)
    if schedule == "owner":
        cuts = [0, 1, 700, 1500, 2000]
        for l0, l1 in zip(cuts[:-1], cuts[1:]):
            s0, s1 = int(lo[l0]), int(lo[l1])
            sub = S[s0:s1].clone()
            sub[:, 0] -= l0  # launch field relative to the chunk's launch_leaf slice
            off = torch.from_numpy(lo[l0:l1 + 1] - s0).cuda()
            dc.dc_pc_sample_attribute(ctx, many, sub, leaf2[l0:l1].contiguous(), off, n_stall=24)
    else:
        n = S.shape[0]
        cuts = [0, 12345, n // 2, n - 7, n]
        for s0, s1 in zip(cuts[:-1], cuts[1:]):
            dc.dc_pc_sample_attribute(ctx, many, S[s0:s1].contiguous(), leaf2, None, n_stall=24)
    dc.dc_cct_rollup(ctx, many)
    a4 = many.to_numpy()
    assert_same(a1, ref, keys=CMP_KEYS, ctx="one call")
    # (rebased bad launch fields n_launch + k - l0 stay >= each chunk's launch count)
    assert_same(a4, a1, keys=CMP_KEYS, ctx=f"four calls ({schedule})")
    d = ctx.diag()  # both trees were built on this context: every drop counted twice
    for k in ["samples_bad_launch", "samples_bad_stall", "samples_zero_count"]:
        assert d[k] == 2 * odiag[k] and odiag[k] > 0, k


def test_pc_attribute_repeated_same_samples_doubles_counts():
    import paper_2411_02797_b200 as dc
    p = gen.programs.config3(n_launch=300, n_samples=500_000)
    tr = gen.make_trace(p, n_records=300, pc=True, n_launch=300)
    ctx = dc.Context(0)
    cct, leaf = _base(p, tr, dc, ctx)
    S, lo = tr.samples.cuda(), tr.launch_off.cuda()
    dc.dc_pc_sample_attribute(ctx, cct, S, leaf, lo, n_stall=24)
    dc.dc_cct_rollup(ctx, cct)
    a = cct.to_numpy()
    dc.dc_pc_sample_attribute(ctx, cct, S, leaf, lo, n_stall=24)  # after ROLLED: accumulates, DIRTY again
    assert cct.view(before_rollup=True).state == 1
    dc.dc_cct_rollup(ctx, cct)
    b = cct.to_numpy()
    for k in ["pc_ctx", "pc_off", "bin_pcnode", "bin_stall"]:
        assert np.array_equal(a[k], b[k]), k
    for k in ["bin_count", "xsamples", "isamples", "xstall", "istall"]:
        assert np.array_equal(2 * a[k], b[k]), k


def test_pc_attribute_stall_count_fixed_and_failed_call_keeps_results():
    import paper_2411_02797_b200 as dc
    p = gen.programs.config3(n_launch=100, n_samples=100_000)
    tr = gen.make_trace(p, n_records=100, pc=True, n_launch=100)
    ctx = dc.Context(0)
    cct, leaf = _base(p, tr, dc, ctx)
    dc.dc_pc_sample_attribute(ctx, cct, tr.samples.cuda(), leaf, tr.launch_off.cuda(), n_stall=24)
    dc.dc_cct_rollup(ctx, cct)
    a = cct.to_numpy()
    with pytest.raises(dc.DcError) as e:
        dc.dc_pc_sample_attribute(ctx, cct, tr.samples.cuda(), leaf, tr.launch_off.cuda(), n_stall=20)
    assert e.value.status == 1  # DC_ERR_ARG
    b = cct.to_numpy()
    for k in CMP_KEYS:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_view_inclusive_fields_need_rollup():
    import ctypes
    import paper_2411_02797_b200 as dc
    from paper_2411_02797_b200 import _lib
    p = gen.programs.config1()
    tr = gen.make_trace(p, n_records=500)
    ctx = dc.Context(0)
    cct, leaf = _base(p, tr, dc, ctx)
    v = dc.dc_cct_view()
    assert _lib.lib().dc_cct_view_get(cct.h, ctypes.byref(v)) == _lib.DC_ERR_STATE
    assert v.n_nodes > 1 and v.parent and v.xcnt and v.xsum  # structure + exclusive columns filled
    assert not v.icnt and not v.isum and not v.imin and not v.isq_lo and not v.isq_hi
    with pytest.raises(dc.DcError):
        cct.view()
    a = cct.to_numpy()
    assert a["icnt"] is None and a["isum"] is None and a["xcnt"] is not None
    dc.dc_cct_rollup(ctx, cct)
    assert _lib.lib().dc_cct_view_get(cct.h, ctypes.byref(v)) == 0 and v.icnt and v.isum


def test_build_null_frames_rejected_unless_all_paths_empty():
    import paper_2411_02797_b200 as dc
    from paper_2411_02797_b200 import _lib
    import ctypes
    ctx = dc.Context(0)
    off = torch.tensor([0, 0, 3], dtype=torch.int64, device="cuda")
    paths = _lib.dc_paths(n_records=2, offsets=ctypes.c_void_p(off.data_ptr()), frames=None)
    h = ctypes.c_void_p()
    st = _lib.lib().dc_cct_build(ctx.h, ctypes.byref(paths), None, 10, None, ctypes.byref(h))
    assert st == _lib.DC_ERR_ARG and not h.value
    off0 = torch.zeros(3, dtype=torch.int64, device="cuda")
    paths = _lib.dc_paths(n_records=2, offsets=ctypes.c_void_p(off0.data_ptr()), frames=None)
    st = _lib.lib().dc_cct_build(ctx.h, ctypes.byref(paths), None, 10, None, ctypes.byref(h))
    assert st == 0 and h.value
    t = dc.CCT(h, ctx)
    assert t.n_nodes == 1
