"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element, on the
same seeded inputs. Integer outputs bit-exact; derived floats within 1e-12 relative
(BASELINE.json north_star)."""
import json
import os

import numpy as np
import pytest
import torch

import gen
import oracle
from pipeline import CMP_KEYS, as_u64, assert_same, gpu_run, oracle_run

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _csr(paths):
    off = np.zeros(len(paths) + 1, np.uint64)
    off[1:] = np.cumsum([len(p) for p in paths])
    fr = np.asarray([f for p in paths for f in p], np.uint32)
    return off, fr


def _samples(lst):
    s = np.zeros(len(lst), oracle.SAMPLE_DTYPE)
    for i, (l, pc, st, c) in enumerate(lst):
        s[i] = (l, pc, st, 0, c)
    return s


def test_f1_fixture_gpu():
    g = json.load(open(os.path.join(GOLD, "f1.json")))
    keys = np.zeros(0, oracle.KEY_DTYPE)
    # records as raw keys (interned on the GPU)
    kk = np.asarray([tuple(g["raw_keys"][f]) for p in g["paths"] for f in p], oracle.KEY_DTYPE)
    off, _ = _csr(g["paths"])
    a = gpu_run(off, keys=kk, metrics=np.asarray(g["metrics"], np.uint64), samples=_samples(g["samples"]), n_stall=24)
    for k in ["leaf", "parent", "depth", "frame", "xcnt", "icnt", "xsamples", "isamples"]:
        assert np.asarray(a[k]).tolist() == g[k], k
    assert a["isum"][0].tolist() == g["isum_ns"] and a["imin"][0].tolist() == g["imin_ns"]
    import paper_2411_02797_b200 as dc
    ctx, cct = a["_ctx"], a["_cct"]
    mean, std = dc.dc_cct_derived(ctx, cct, 0, True)
    assert mean.cpu().numpy().tolist() == g["imean_ns"]
    np.testing.assert_allclose(std.cpu().numpy(), g["istd_ns"], rtol=1e-12, atol=0)
    hot = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_INCLUSIVE, 0, 1 << dc.DC_KIND_KERNEL, 0.1, 3)
    assert [list(e) for e in hot] == g["hotspot_kernels_incl_ns_theta0.1_k3"]
    bu = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_BOTTOM_UP, 0, 0xFFFFFFFF, 0.0, 10)
    assert [[i, v] for i, v, _ in bu] == g["bottom_up_excl_ns"]
    for node, key in [(8, "stall_top2_node8"), (10, "stall_top2_node10")]:
        st = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_STALL, k=2, stall_node=node)
        assert [list(e) for e in st] == g[key]
    assert list(map(list, zip(a["bin_pcnode"].tolist(), a["bin_stall"].tolist(), a["bin_count"].tolist()))) == g["bins"]
    d = ctx.diag()
    assert (d["samples_bad_launch"], d["samples_bad_stall"], d["samples_zero_count"], d["empty_paths"]) == (1, 1, 1, 1)


def _rand_trace(rng, R_max=300, A_max=40):
    R = int(rng.integers(1, R_max))
    A = int(rng.integers(2, A_max))
    paths = []
    for _ in range(R):
        L = int(rng.integers(0, 20))
        if paths and rng.random() < 0.4:
            base = list(paths[int(rng.integers(0, len(paths)))])
            p = base[: min(L, len(base))] + [int(rng.integers(0, A)) for _ in range(max(0, L - len(base)))]
        else:
            p = [int(rng.integers(0, A)) for _ in range(L)]
        if p and rng.random() < 0.1:
            i = int(rng.integers(0, len(p)))
            p = p[: i + 1] + [p[i]] * 2 + p[i + 1:]
        paths.append(tuple(p))
    M = int(rng.integers(1, 4))
    X = rng.integers(0, 2**40 if rng.random() < 0.3 else 10**6, size=(M, R), dtype=np.uint64)
    if rng.random() < 0.2:
        X[:, : max(1, R // 7)] = np.uint64(2**63 // max(R, 1))  # large values: u128 sums of squares
    S = int(rng.integers(1, 33))
    ns = int(rng.integers(0, 400))
    smp = _samples([(int(rng.integers(0, R + 2)), int(rng.integers(0, 50)) * 16, int(rng.integers(0, S + 2)),
                     int(rng.integers(0, 5))) for _ in range(ns)])
    return paths, X, smp, S, A


@pytest.mark.parametrize("seed", range(8))
def test_random_traces_vs_oracle(seed, monkeypatch):
    # rollup schedules: per-column shared-memory level walk (default for small trees; seeds 2,
    # 7), level-synchronous cooperative kernel (odd seeds but 7), ancestor push with 32-bit limbs
    # (6), with returned u128 atomics (0, 4)
    if seed % 2 and seed != 7:
        monkeypatch.setenv("DC_TEST_ROLLUP_LEVELS", "1")
    if seed >= 4 and seed != 6:  # the one-CTA level loop instead of the lexicographic-rank build
        monkeypatch.setenv("DC_TEST_BUILD_LEVELS", "1")
    if seed in (0, 4):
        monkeypatch.setenv("DC_TEST_ROLLUP_PUSH_RETURNED", "1")
    if seed == 6:
        monkeypatch.setenv("DC_TEST_ROLLUP_PUSH", "1")
    if seed in (3, 5):  # views: the multi-kernel sort path instead of the one-CTA radix select
        monkeypatch.setenv("DC_TEST_TOPK_GENERAL", "1")
    rng = np.random.default_rng(500 + seed)
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    for it in range(25):
        paths, X, smp, S, A = _rand_trace(rng)
        off, fr = _csr(paths)
        a = gpu_run(off, fr, X, n_frames=A, samples=smp, n_stall=S, ctx=ctx)
        ref = oracle_run(off, fr, X, X.shape[0], smp, len(paths), S).arrays()
        assert_same(a, ref, ctx=f"seed {seed} it {it}")
        # views vs oracle
        fk = rng.integers(0, 6, size=A).astype(np.uint8)
        o = oracle_run(off, fr, X, X.shape[0], smp, len(paths), S)
        for view in [0, 1, 2, 3]:
            th = float(rng.choice([-1.0, 0.0, 0.01, 0.2]))
            k = int(rng.integers(1, 12))
            m = int(rng.integers(0, X.shape[0]))
            node = int(rng.integers(0, a["n_nodes"]))
            got = dc.dc_hotspots_topk(ctx, a["_cct"], view, m, 0xFFFFFFFF, th, k, node)
            exp = o.topk(view, m, 0xFFFFFFFF, None, th, k, node)
            assert got == [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in exp], (view, th, k)
        # derived
        for m in range(X.shape[0]):
            for incl in (True, False):
                mg, sg = dc.dc_cct_derived(ctx, a["_cct"], m, incl)
                mo, so = o.derived(m, incl)
                np.testing.assert_allclose(mg.cpu().numpy(), mo, rtol=1e-12, atol=0)
                np.testing.assert_allclose(sg.cpu().numpy(), so, rtol=1e-12, atol=0)


def test_kind_mask_and_bottom_up_with_dict():
    p = gen.programs.program(1)
    tr = gen.make_trace(p)
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy())
    import paper_2411_02797_b200 as dc
    oids, odict = oracle.intern(tr.keys.numpy())
    o = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), 2)
    fk = np.asarray(odict["kind"], np.uint8)
    assert np.array_equal(a["ids"], oids)
    assert np.array_equal(a["_dict"].kinds(), fk)
    for view in [0, 1, 2]:
        for mask in [1 << 4, (1 << 0) | (1 << 2), 0xFFFFFFFF]:
            for th in [0.0, 0.001, 0.05]:
                got = dc.dc_hotspots_topk(a["_ctx"], a["_cct"], view, 0, mask, th, 20)
                exp = o.topk(view, 0, mask, fk, th, 20)
                assert got == [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in exp]


@pytest.mark.parametrize("cfg,R", [(1, None), (2, 200_000), (2, 1_000_000), (3, None)])
def test_configs_vs_oracle(cfg, R):
    p = gen.programs.program(cfg) if cfg != 3 else gen.programs.config3(n_samples=4_000_000)
    tr = gen.make_trace(p, n_records=R, pc=(cfg == 3), bad_per_million=500 if cfg == 3 else 0)
    kw = {}
    if cfg == 3:
        kw = dict(samples=tr.samples.numpy(), launch_off=tr.launch_off.numpy(), n_launch=tr.n_launch)
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy(), **kw)
    oids, _ = oracle.intern(tr.keys.numpy())
    assert np.array_equal(a["ids"], oids)
    ref = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), p.n_metrics,
                     tr.samples.numpy() if cfg == 3 else None, tr.n_launch if cfg == 3 else 0).arrays()
    ref["leaf"] = ref["leaf"]
    assert_same(a, ref, ctx=f"cfg{cfg}")


def test_generic_schedule_equals_owner_schedule(monkeypatch):
    """launch_sample_off given vs NULL: identical results (and oracle); the owner schedule's
    launch ordering by the one-CTA counting sort and by the multi-pass radix sort."""
    p = gen.programs.config3(n_samples=2_000_000)
    tr = gen.make_trace(p, pc=True, bad_per_million=1000)
    kw = dict(keys=tr.keys.numpy(), metrics=tr.metrics.numpy(), samples=tr.samples.numpy(), n_launch=tr.n_launch)
    a = gpu_run(tr.offsets.numpy(), launch_off=tr.launch_off.numpy(), **kw)
    b = gpu_run(tr.offsets.numpy(), launch_off=None, **kw)
    assert_same(a, b, ctx="owner vs generic")
    monkeypatch.setenv("DC_TEST_OWN_RADIX", "1")
    c = gpu_run(tr.offsets.numpy(), launch_off=tr.launch_off.numpy(), **kw)
    assert_same(a, c, ctx="owner (radix-sorted launches)")


@pytest.mark.parametrize("reduce", ["ctx", "br", "cap1"])
@pytest.mark.parametrize("n,npc,big", [(3_000_000, 2000, False), (400_000, 20_000, False), (200_000, 300, True)])
def test_owner_high_cardinality_flush_spill_and_wrap(n, npc, big, reduce, monkeypatch):
    """One context with up to 480k (pc, stall) keys: mid-context flushes and spills in the
    context-owner schedule; big=True uses counts up to 2^31 (32-bit shared-counter carries),
    so every sample is spilled (many spill-chunk switches). The schedule must not fall back.
    Reduce: the one-pass context reduce (shared counts for <= 12,288 bins, global atomics past
    that; 20,000 PCs exceed its shared bitmap and take the global-bitmap reduce), the global
    bitmap reduce forced, or the context reduce with a 1-bin capacity guess (reallocate + rerun)."""
    monkeypatch.setenv("DC_TEST_OWNER_STRICT", "1")
    if reduce == "br":
        monkeypatch.setenv("DC_TEST_PC_BR", "1")
    if reduce == "cap1":
        monkeypatch.setenv("DC_TEST_PC_CAP", "1")
    rng = np.random.default_rng(n)
    s = np.zeros(n, oracle.SAMPLE_DTYPE)
    s["launch"] = 0
    s["pc_off"] = 16 * rng.integers(0, npc, n)
    s["stall"] = rng.integers(0, 24, n)
    s["count"] = rng.integers(1, 2**31, n) if big else 1
    off, fr = _csr([(0, 1)])
    X = np.ones((1, 1), np.uint64)
    lo = np.array([0, n], np.uint64)
    a = gpu_run(off, fr, X, n_frames=2, samples=s, launch_off=lo, n_stall=24)
    ref = oracle_run(off, fr, X, 1, s, 1, 24).arrays()
    assert_same(a, ref, ctx=f"owner n={n} npc={npc}")


@pytest.mark.parametrize("n_launch,heavy,pcs", [(3, 1, 30_000), (300, 40, 30_000), (2000, 5, 30_000), (300, 40, 6000),
                                                (2000, 5, 6000)])
def test_owner_work_stealing_skewed_contexts(n_launch, heavy, pcs, monkeypatch):
    """Stage ranges of very unequal cost: a few launches carry most samples with many distinct
    keys (flushes, spill chunks), the rest are light; with 3 launches most CTAs start with an
    empty range and only steal. Every stage must be aggregated exactly once: oracle and generic
    schedule agree, and the owner schedule must not fall back."""
    monkeypatch.setenv("DC_TEST_OWNER_STRICT", "1")
    rng = np.random.default_rng(n_launch)
    paths = [(0, 1), (0, 2), (1, 3), (1, 2, 4), (3,), (0, 1, 2, 3)]
    off, fr = _csr([paths[i % len(paths)] for i in range(n_launch)])  # launch i = record i
    X = np.ones((1, n_launch), np.uint64)
    cnt = rng.integers(1, 300, n_launch)
    cnt[:heavy] = rng.integers(100_000, 400_000, heavy)
    lo = np.zeros(n_launch + 1, np.uint64)
    lo[1:] = np.cumsum(cnt)
    n = int(lo[-1])
    s = np.zeros(n, oracle.SAMPLE_DTYPE)
    s["launch"] = np.repeat(np.arange(n_launch, dtype=np.uint32), cnt)
    heavy_s = s["launch"] < heavy
    s["pc_off"] = np.where(heavy_s, 16 * rng.integers(0, pcs, n), 16 * rng.integers(0, 50, n))
    s["stall"] = rng.integers(0, 24, n)
    s["count"] = 1
    kw = dict(n_frames=5, samples=s, n_stall=24)
    a = gpu_run(off, fr, X, launch_off=lo, **kw)
    b = gpu_run(off, fr, X, launch_off=None, **kw)
    assert_same(a, b, ctx="owner vs generic (skewed)")
    ref = oracle_run(off, fr, X, 1, s, n_launch, 24).arrays()
    assert_same(a, ref, ctx=f"owner skewed n_launch={n_launch}")


@pytest.mark.parametrize("builder", ["rank_spec", "rank", "levels"])
def test_small_build_deep_and_prefix_paths(builder, monkeypatch):
    """Small-P build at the depth limit: chains up to 1000 frames, paths that are prefixes of
    other paths, shared deep prefixes that branch late, an empty path; both small-P builders,
    the rank builder launched speculatively (behind the record pass's readback) and not."""
    if builder == "levels":
        monkeypatch.setenv("DC_TEST_BUILD_LEVELS", "1")
    if builder == "rank":
        monkeypatch.setenv("DC_TEST_BUILD_NOSPEC", "1")
    rng = np.random.default_rng(77)
    base = [int(x) for x in rng.integers(0, 40, 1000)]
    paths = [tuple(base), tuple(base[:500]), tuple(base[:499] + [41]), tuple(base[:999] + [0]), (), tuple(base[:1]),
             tuple(base[:3] + [7, 7, 7]), (5,), (5, 5), tuple(base[:700] + [3] * 50)]
    paths += [tuple(base[: int(rng.integers(1, 1000))]) + tuple(int(x) for x in rng.integers(0, 42, 3)) for _ in range(60)]
    off, fr = _csr(paths)
    X = rng.integers(0, 1000, size=(1, len(paths)), dtype=np.uint64)
    a = gpu_run(off, fr, X, n_frames=42)
    ref = oracle_run(off, fr, X, 1).arrays()
    assert_same(a, ref, ctx=f"deep small build {builder}")


def test_dedup_independent_of_tile_staging():
    """One path hashed in a tile whose frames are staged in shared memory and in a tile read from
    global memory (frames > the staging window) must give one item: with DC_STRICT=1 (conftest)
    a repeated table item is an error, and the tree must equal the oracle's."""
    rng = np.random.default_rng(3)
    X = tuple(int(x) for x in rng.integers(0, 50, 40))
    deep = [tuple(int(x) for x in rng.integers(0, 50, 100)) for _ in range(127)]
    paths = deep + [X] + [X] * 128 + [X[:20], X] * 100  # tile 0: 12,740 frames (global), tile 1: staged
    off, fr = _csr(paths)
    M = np.ones((1, len(paths)), np.uint64)
    a = gpu_run(off, fr, M, n_frames=50)
    ref = oracle_run(off, fr, M, 1).arrays()
    assert_same(a, ref, ctx="dedup across staged / global tiles")


def test_edge_cases():
    # empty trace
    a = gpu_run(np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros((1, 0), np.uint64), n_frames=5)
    assert a["n_nodes"] == 1 and a["icnt"].tolist() == [0]
    # all empty paths
    off = np.zeros(5, np.uint64)
    a = gpu_run(off, np.zeros(0, np.uint32), np.arange(4, dtype=np.uint64)[None], n_frames=1)
    assert a["n_nodes"] == 1 and a["xcnt"].tolist() == [4] and a["isum"][0].tolist() == [6]
    # single record, single frame
    a = gpu_run(np.array([0, 1], np.uint64), np.array([0], np.uint32), np.array([[7]], np.uint64), n_frames=1)
    assert a["parent"].tolist() == [0xFFFFFFFF, 0] and a["isum"][0].tolist() == [7, 7]
    # depth == DC_MAX_DEPTH (1024) recursion chain; prefix-of-another; all identical
    K = 1024
    paths = [tuple([3] * k) for k in range(1, K + 1)] + [tuple([3] * 10)] * 50
    off, fr = _csr(paths)
    X = np.ones((1, len(paths)), np.uint64)
    a = gpu_run(off, fr, X, n_frames=4)
    ref = oracle_run(off, fr, X, 1).arrays()
    assert_same(a, ref, ctx="chain")
    assert a["max_depth"] == K


def test_too_deep_and_bad_frame_are_trace_errors():
    import paper_2411_02797_b200 as dc
    off, fr = _csr([tuple([1] * 1025)])
    with pytest.raises(dc.DcError) as e:
        gpu_run(off, fr, np.ones((1, 1), np.uint64), n_frames=2)
    assert e.value.status == 6
    off, fr = _csr([(0, 9)])
    with pytest.raises(dc.DcError) as e:
        gpu_run(off, fr, np.ones((1, 1), np.uint64), n_frames=5)
    assert e.value.status == 6


def test_large_P_multikernel_build():
    """> 4096 distinct paths takes the per-level multi-kernel build."""
    rng = np.random.default_rng(3)
    paths = [tuple(int(x) for x in rng.integers(0, 30, size=int(rng.integers(1, 12)))) for _ in range(20_000)]
    paths += paths[:5000]
    off, fr = _csr(paths)
    X = rng.integers(0, 10**9, size=(2, len(paths)), dtype=np.uint64)
    a = gpu_run(off, fr, X, n_frames=30)
    ref = oracle_run(off, fr, X, 2).arrays()
    assert_same(a, ref, ctx="largeP")


@pytest.mark.parametrize("verify", ["sweep", "rows"])
def test_hash_collisions_resolved_exactly(verify, monkeypatch):
    """DC_TEST_WEAK_HASH=6 keeps 6 bits of the path hash: thousands of collisions, same tree;
    with k_path_group's window-sweep verify and with its per-record verify (DC_PG_ROWS)."""
    monkeypatch.setenv("DC_TEST_WEAK_HASH", "6")
    if verify == "rows":
        monkeypatch.setenv("DC_PG_ROWS", "1")
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    rng = np.random.default_rng(4)
    paths = [tuple(int(x) for x in rng.integers(0, 8, size=int(rng.integers(0, 9)))) for _ in range(3000)]
    off, fr = _csr(paths)
    X = rng.integers(0, 1000, size=(1, len(paths)), dtype=np.uint64)
    a = gpu_run(off, fr, X, n_frames=8, ctx=ctx)
    ref = oracle_run(off, fr, X, 1).arrays()
    assert_same(a, ref, ctx="weak hash")
    assert ctx.diag()["collisions_detected"] > 0


def test_permutation_invariance_and_determinism():
    p = gen.programs.program(1)
    tr = gen.make_trace(p)
    off = tr.offsets.numpy().view(np.uint64)
    ids = tr.ids.numpy().view(np.uint32)
    X = as_u64(tr.metrics.numpy())
    R = len(off) - 1
    perm = np.random.default_rng(9).permutation(R)
    paths = [ids[off[r]:off[r + 1]] for r in perm]
    off2 = np.zeros(R + 1, np.uint64)
    off2[1:] = np.cumsum([len(q) for q in paths])
    fr2 = np.concatenate(paths).astype(np.uint32)
    a = gpu_run(off, ids, X, n_frames=tr.n_frames)
    b = gpu_run(off2, fr2, X[:, perm], n_frames=tr.n_frames)
    c = gpu_run(off, ids, X, n_frames=tr.n_frames)
    la, lb = a.pop("leaf"), b.pop("leaf")
    assert_same(a, b, keys=[k for k in CMP_KEYS if "samples" not in k and "stall" not in k and "pc" not in k and "bin" not in k])
    a["leaf"] = la
    assert_same(a, c)
    a["leaf"], b["leaf"] = la, lb
    assert np.array_equal(a["leaf"][perm], b["leaf"])


@pytest.mark.parametrize("env", [{}, {"DC_TEST_LEVELWISE": "1"}, {"DC_TEST_WEAK_NODE_HASH": "7"}, {"DC_TEST_NO_TMA": "1"}])
def test_large_P_build_variants(monkeypatch, env):
    """> 4096 distinct paths, deep recursion and shared prefixes: the Euler-tour build, the
    level-wise build (forced), the Euler build with prefix-node hashes cut to 7 bits (its
    collision check must detect it and fall back to the exact level-wise build), and the record
    pass without TMA staging — all equal to the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    rng = np.random.default_rng(11)
    paths = []
    for _ in range(12_000):
        pre = [0, 1, 2][: int(rng.integers(0, 4))]
        rec = [5, 6] * int(rng.integers(0, 120)) if rng.random() < 0.1 else []
        tail = [int(x) for x in rng.integers(0, 40, size=int(rng.integers(0, 14)))]
        paths.append(tuple(pre + rec + tail))
    paths += paths[:3000] + [()] * 5
    order = rng.permutation(len(paths))
    paths = [paths[i] for i in order]
    off, fr = _csr(paths)
    X = rng.integers(0, 10**9, size=(2, len(paths)), dtype=np.uint64)
    a = gpu_run(off, fr, X, n_frames=40, ctx=ctx)
    ref = oracle_run(off, fr, X, 2).arrays()
    assert_same(a, ref, ctx=f"largeP {env}")
    dep = a["depth"].astype(np.int64)
    lo = [int(np.searchsorted(dep, d, side="left")) for d in range(int(a["max_depth"]) + 2)]
    assert a["level_off"].tolist() == lo
    if "DC_TEST_WEAK_NODE_HASH" in env:
        assert ctx.diag()["collisions_detected"] > 0


@pytest.mark.parametrize("direct", [False, True])
def test_attribute_contended_columns(monkeypatch, direct):
    """Many records on few nodes (the replicated-column attribution path, K copies folded) and the
    direct path: identical to the oracle, with values up to 2^40 (128-bit squares)."""
    if direct:
        monkeypatch.setenv("DC_TEST_ATTR_DIRECT", "1")
    rng = np.random.default_rng(77)
    base = [tuple(int(x) for x in rng.integers(0, 20, size=int(rng.integers(1, 7)))) for _ in range(60)]
    paths = [base[i] for i in rng.integers(0, len(base), size=300_000)]
    off, fr = _csr(paths)
    X = np.stack([rng.integers(0, 2**40, size=len(paths), dtype=np.uint64),
                  rng.integers(0, 1000, size=len(paths), dtype=np.uint64)])
    a = gpu_run(off, fr, X, n_frames=20)
    ref = oracle_run(off, fr, X, 2).arrays()
    assert_same(a, ref, ctx=f"contended direct={direct}")


@pytest.mark.parametrize("D,radix", [(3000, False), (3000, True), (20000, False), (40000, False), (1, False)])
def test_intern_rank_paths(D, radix, monkeypatch):
    """Frame interning: the direct-count rank (D <= 8192) and the two-pass radix sort (forced, or
    D > 8192) give the oracle's ids and sorted dictionary; keys share kinds / strings / addresses
    so every field of the (kind, str_id, addr) order decides some pairs."""
    if radix:
        monkeypatch.setenv("DC_TEST_INTERN_RADIX", "1")
    import paper_2411_02797_b200 as dc
    rng = np.random.default_rng(D)
    base = np.zeros(D, oracle.KEY_DTYPE)
    base["kind"] = rng.integers(0, 6, D)
    base["str_id"] = rng.integers(0, max(2, D // 50), D)
    base["addr"] = rng.integers(0, 2**40, D, dtype=np.uint64)
    base["addr"][: D // 3] = rng.integers(0, 8, D // 3)  # small addresses: ties on the high words
    keys = base[rng.integers(0, D, 400_000)]
    ctx = dc.Context(0)
    kk = torch.from_numpy(np.ascontiguousarray(keys).view(np.int32).reshape(-1, 4)).to("cuda:0")
    ids, d = dc.dc_intern_frames(ctx, kk)
    oids, od = oracle.intern(keys)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), oids)
    assert np.array_equal(d.keys(), od)
    assert np.array_equal(d.kinds(), np.minimum(od["kind"], 255).astype(np.uint8))


def test_ctx_reserve():
    """dc_ctx_reserve grows the pool (results unchanged); an impossible size is DC_ERR_OOM."""
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    ctx.reserve(1 << 30)
    off, fr = _csr([(0, 1), (0, 2), (1,)])
    X = np.array([[3, 4, 5]], np.uint64)
    a = gpu_run(off, fr, X, n_frames=3, ctx=ctx)
    assert_same(a, oracle_run(off, fr, X, 1).arrays(), ctx="after reserve")
    with pytest.raises(dc.DcError) as e:
        ctx.reserve(1 << 50)
    assert e.value.status == 2  # DC_ERR_OOM


def test_path_table_overflow_retry(monkeypatch):
    """5,000 distinct paths into a 1,024-slot path table (DC_TEST_PATH_CAP): the record pass
    detects the overflow, discards the attempt (diagnostics counted once) and retries larger."""
    monkeypatch.setenv("DC_TEST_PATH_CAP", "1")
    rng = np.random.default_rng(11)
    paths = [tuple(int(x) for x in rng.integers(0, 60, int(rng.integers(1, 12)))) for _ in range(5000)] + [()] * 7
    off, fr = _csr(paths)
    X = rng.integers(0, 100, size=(1, len(paths)), dtype=np.uint64)
    a = gpu_run(off, fr, X, n_frames=60)
    assert_same(a, oracle_run(off, fr, X, 1).arrays(), ctx="path table retry")
    assert a["_ctx"].diag()["empty_paths"] == 7


@pytest.mark.parametrize("general", [False, True])
def test_topk_ties_and_large_k(general, monkeypatch):
    """Top-k on a star of 5,000 leaves whose values take only 3 distinct values (massive ties:
    the order is value desc, then id asc), k from 1 to 1,000 and thresholds around the tie
    values; the one-CTA radix select (and the general sort path) equal the oracle's sort."""
    if general:
        monkeypatch.setenv("DC_TEST_TOPK_GENERAL", "1")
    import paper_2411_02797_b200 as dc
    W = 5000
    rng = np.random.default_rng(77)
    paths = [[0, 1 + j] for j in range(W)] + [[0]]
    off, fr = _csr(paths)
    X = np.zeros((1, len(paths)), np.uint64)
    X[0, :W] = rng.choice(np.array([5, 7, 9], np.uint64), size=W)
    X[0, W] = 3
    a = gpu_run(off, fr, X, n_frames=W + 1)
    o = oracle_run(off, fr, X, 1)
    total = float(X.sum())
    for view in [0, 1, 2]:
        for k in [1, 7, 100, 1000]:
            for th in [-1.0, 0.0, 5.5 / total, 7.0 / total, 8.0 / total]:
                got = dc.dc_hotspots_topk(a["_ctx"], a["_cct"], view, 0, 0xFFFFFFFF, th, k)
                exp = o.topk(view, 0, 0xFFFFFFFF, None, th, k)
                assert got == [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in exp], (view, k, th)


@pytest.mark.parametrize("schedule", ["partition", "table"])
def test_config3s_stress_generic_schedule_vs_oracle(schedule, monkeypatch):
    """Config 3s (gen/stress.py): every launch its own context and the samples of 8 concurrent
    launches interleaved (no per-launch offsets): the any-order schedules — the launch partition
    + context-owner schedule, and the L2 table (DC_TEST_PC_GENERIC) — element by element against
    the oracle on the same re-arranged trace, with the same invalid-sample counts."""
    from gen import stress
    if schedule == "table":
        monkeypatch.setenv("DC_TEST_PC_GENERIC", "1")
    p = gen.programs.config3(n_launch=3000, n_samples=3_000_000)
    tr = stress.make_3s(gen.make_trace(p, n_records=3000, pc=True, n_launch=3000, bad_per_million=500))
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy(), samples=tr.samples.numpy(),
                n_launch=tr.n_launch)
    dg = a["_ctx"].diag()
    smp = tr.samples.numpy().view(np.uint32).reshape(-1, 4)
    bad_l = smp[:, 0] >= tr.n_launch
    assert dg["samples_bad_launch"] == int(bad_l.sum())
    assert dg["samples_bad_stall"] == int((~bad_l & ((smp[:, 2] & 0xFFFF) >= 24)).sum())
    oids, _ = oracle.intern(tr.keys.numpy())
    assert np.array_equal(a["ids"], oids)
    ref = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), p.n_metrics, tr.samples.numpy(), tr.n_launch).arrays()
    assert_same(a, ref, ctx="config 3s")
    assert len(np.unique(a["leaf"])) == 3000  # distinct contexts


def test_config3_aggregated_counts_on_the_table_path(monkeypatch):
    """Per-PC aggregated records (counts > 1, gen/stress.make_aggregated) go through the
    context-owner table (counts < 2^16) and equal both the oracle and the raw-sample result."""
    monkeypatch.setenv("DC_TEST_OWNER_STRICT", "1")
    from gen import stress
    p = gen.programs.config3(n_launch=2000, n_samples=4_000_000)
    raw = gen.make_trace(p, n_records=2000, pc=True, n_launch=2000)
    ag = stress.make_aggregated(raw)
    assert int(ag.samples[:, 3].max()) > 1
    kw = dict(keys=raw.keys.numpy(), metrics=raw.metrics.numpy(), n_launch=2000)
    a = gpu_run(raw.offsets.numpy(), samples=ag.samples.numpy(), launch_off=ag.launch_off.numpy(), **kw)
    b = gpu_run(raw.offsets.numpy(), samples=raw.samples.numpy(), launch_off=raw.launch_off.numpy(), **kw)
    oids, _ = oracle.intern(raw.keys.numpy())
    ref = oracle_run(raw.offsets.numpy(), oids, raw.metrics.numpy(), p.n_metrics, ag.samples.numpy(), 2000).arrays()
    assert_same(a, ref, ctx="aggregated")
    assert_same(a, b, ctx="aggregated vs raw")


def test_owner_large_counts_extra_flush_budget(monkeypatch):
    """2M records of one context with counts up to 65,535 (the table path) and above (spilled):
    far more than 2^32 in total, so the counts-above-1 budget must force flushes before any
    32-bit table counter could wrap."""
    monkeypatch.setenv("DC_TEST_OWNER_STRICT", "1")
    n = 2_000_000
    rng = np.random.default_rng(5)
    s = np.zeros(n, oracle.SAMPLE_DTYPE)
    s["launch"] = 0
    s["pc_off"] = 16 * rng.integers(0, 40, n)
    s["stall"] = rng.integers(0, 24, n)
    s["count"] = np.where(rng.random(n) < 0.01, rng.integers(65_536, 2**31, n), rng.integers(60_000, 65_536, n))
    off, fr = _csr([(0, 1)])
    X = np.ones((1, 1), np.uint64)
    a = gpu_run(off, fr, X, n_frames=2, samples=s, launch_off=np.array([0, n], np.uint64), n_stall=24)
    ref = oracle_run(off, fr, X, 1, s, 1, 24).arrays()
    assert_same(a, ref, ctx="large counts")
    assert int(ref["bin_count"].sum()) > 2**40
