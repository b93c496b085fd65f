"""GPU parity of the analyzer rules (include/dc.h dc_analyze_flags /
dc_analyze_stalls) against the oracle, element by element: random tiny traces (every frame
counts as a kernel: no dictionary), config 2 (ResNet-50-shaped, kinds from the interned
dictionary) and config 3 (PC samples: analysis ④)."""
import numpy as np
import pytest

import gen
import oracle
from pipeline import gpu_run, oracle_run
from test_oracle_pins import _rand_trace

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("seed", range(3))
def test_rules_random_vs_oracle(seed):
    import paper_2411_02797_b200 as dc
    rng = np.random.default_rng(9100 + seed)
    ctx = dc.Context(0)
    for _ in range(20):
        paths, X, samples, S = _rand_trace(rng)
        off, fr = _csr(paths)
        A = 1 + max([f for p in paths for f in p] + [0])
        Xa = np.asarray(X, np.uint64).reshape(len(X), -1)
        smp = _samples(samples)
        a = gpu_run(off, fr, Xa, n_frames=A, samples=smp, n_stall=S, ctx=ctx)
        o = oracle_run(off, fr, Xa, len(X), smp, len(paths), S)
        M = len(X)
        vals = [v for row in X for v in row] or [1]
        for rule in (dc.DC_RULE_SMALL_KERNELS, dc.DC_RULE_CPU_LATENCY):
            ma, mb = int(rng.integers(0, M)), int(rng.integers(0, M))
            thr = float(rng.choice([0.5, 2.0, float(np.median(vals)) + 0.5]))
            floor = int(rng.choice([0, int(np.median(vals))]))
            got = dc.dc_analyze_flags(ctx, a["_cct"], rule, ma, mb, 1 << 4, thr, floor)
            exp = o.rule_flags(rule, ma, mb, kind_mask=1 << 4, threshold=thr, floor=floor)
            assert got == exp, (rule, thr, floor)
        for hot_thr, st_thr, k in [(0.0, 0.0, 3), (0.1, 0.2, 2), (0.3, 0.05, 5)]:
            got = dc.dc_analyze_stalls(ctx, a["_cct"], 0, 0xFFFFFFFF, hot_thr, st_thr, k)
            exp = o.stall_issues(0, hot_threshold=hot_thr, stall_threshold=st_thr, k=k)
            assert got == exp, (hot_thr, st_thr, k)


def test_rules_config2_vs_oracle():
    """ResNet-50-shaped trace (raw keys, kinds from the dictionary): ② on gpu_time (metric 0)
    over kernel launches; ⑤ with metric 2 (blocks) as the 'cpu' column against gpu_time."""
    import paper_2411_02797_b200 as dc
    p = gen.programs.program(2)
    tr = gen.make_trace(p, n_records=120_000)
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy())
    ctx = a["_ctx"]
    oids, od = oracle.intern(tr.keys.numpy())
    o = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), p.n_metrics)
    fk = np.asarray(od["kind"], np.uint8)
    for thr in (5_000.0, 20_000.0, 60_000.0):
        got = dc.dc_analyze_flags(ctx, a["_cct"], dc.DC_RULE_SMALL_KERNELS, 0, 0, 1 << dc.DC_KIND_KERNEL, thr)
        exp = o.rule_flags(oracle.RULE_SMALL_KERNELS, 0, kind_mask=1 << dc.DC_KIND_KERNEL, frame_kind=fk, threshold=thr)
        assert got == exp and (thr < 10_000 or got), thr
    for thr in (0.01, 0.5):
        got = dc.dc_analyze_flags(ctx, a["_cct"], dc.DC_RULE_CPU_LATENCY, 2, 0, 0, thr, 1000)
        exp = o.rule_flags(oracle.RULE_CPU_LATENCY, 2, 0, threshold=thr, floor=1000)
        assert got == exp, thr


def test_stalls_config3_vs_oracle():
    """Analysis ④ on an LLM-decode-shaped PC-sampling trace (kinds from the dictionary)."""
    import paper_2411_02797_b200 as dc
    p = gen.programs.config3(n_samples=3_000_000)
    tr = gen.make_trace(p, pc=True, bad_per_million=200)
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy(), samples=tr.samples.numpy(),
                launch_off=tr.launch_off.numpy(), n_launch=tr.n_launch)
    ctx = a["_ctx"]
    oids, od = oracle.intern(tr.keys.numpy())
    o = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), p.n_metrics, tr.samples.numpy(), tr.n_launch)
    fk = np.asarray(od["kind"], np.uint8)
    for hot_thr, st_thr, k in [(0.01, 0.02, 3), (0.0, 0.0, 5), (0.05, 0.1, 1)]:
        got = dc.dc_analyze_stalls(ctx, a["_cct"], 0, 1 << dc.DC_KIND_KERNEL, hot_thr, st_thr, k)
        exp = o.stall_issues(0, kind_mask=1 << dc.DC_KIND_KERNEL, frame_kind=fk, hot_threshold=hot_thr,
                             stall_threshold=st_thr, k=k)
        assert got == exp, (hot_thr, st_thr, k)
        assert got or hot_thr > 0.0


def test_folded_export_vs_oracle():
    """NEXT-3: folded flame-graph text of the CUDA path == the oracle's, byte for byte, on random
    traces and on a config-2 trace (labels = frame ids)."""
    import paper_2411_02797_b200 as dc
    rng = np.random.default_rng(9300)
    ctx = dc.Context(0)
    for _ in range(15):
        paths, X, samples, S = _rand_trace(rng)
        off, fr = _csr(paths)
        A = 1 + max([f for p in paths for f in p] + [0])
        Xa = np.asarray(X, np.uint64).reshape(len(X), -1)
        a = gpu_run(off, fr, Xa, n_frames=A, ctx=ctx)
        o = oracle_run(off, fr, Xa, len(X)).arrays()
        labels = [f"f{i};x" if i % 5 == 0 else f"f{i}" for i in range(A)]
        for m in range(len(X)):
            assert dc.folded_text(ctx, a["_cct"], labels, m) == oracle.folded(o, m, labels)
    p = gen.programs.program(2)
    tr = gen.make_trace(p, n_records=50_000)
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy())
    oids, od = oracle.intern(tr.keys.numpy())
    o = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), p.n_metrics).arrays()
    labels = [str(i) for i in range(len(od))]
    text = dc.folded_text(a["_ctx"], a["_cct"], labels, 0)
    assert text == oracle.folded(o, 0, labels) and text.count("\n") > 100


def test_cpu_intervals_vs_oracle_and_attribution():
    """NEXT-4: intervals of the CUDA path == the oracle's replay; the valid intervals attributed to
    their samples' call paths give the oracle's CCT of the same (filtered) records."""
    import torch
    import paper_2411_02797_b200 as dc
    rng = np.random.default_rng(9400)
    ctx = dc.Context(0)
    for n in (1, 17, 3000, 250_000):
        th = rng.integers(0, 33, n).astype(np.int32)
        kd = rng.integers(0, 2, n).astype(np.uint8)
        ts = np.cumsum(rng.integers(0, 10**6, n)).astype(np.int64)
        iv, ok = dc.dc_cpu_intervals(ctx, torch.from_numpy(th).cuda(), torch.from_numpy(kd).cuda(), torch.from_numpy(ts).cuda())
        eiv, eok = oracle.cpu_intervals(th, kd, ts)
        assert iv.cpu().numpy().tolist() == eiv and ok.cpu().numpy().astype(bool).tolist() == eok
    # attribution: each sample has a call path; valid samples' intervals are the metric
    n = 20_000
    paths = [tuple(int(x) for x in rng.integers(0, 12, size=int(rng.integers(1, 8)))) for _ in range(n)]
    th = rng.integers(0, 4, n).astype(np.int32)
    kd = np.zeros(n, np.uint8)
    ts = np.cumsum(rng.integers(1, 5000, n)).astype(np.int64)
    iv, ok = dc.dc_cpu_intervals(ctx, torch.from_numpy(th).cuda(), torch.from_numpy(kd).cuda(), torch.from_numpy(ts).cuda())
    keep = ok.cpu().numpy().astype(bool)
    kp = [p for p, k in zip(paths, keep) if k]
    off, fr = _csr(kp)
    X = iv.cpu().numpy()[keep].astype(np.uint64)[None]
    a = gpu_run(off, fr, X, n_frames=12, ctx=ctx)
    eiv, eok = oracle.cpu_intervals(th, kd, ts)
    ref = oracle_run(off, fr, np.asarray([[v for v, o in zip(eiv, eok) if o]], np.uint64), 1).arrays()
    for key in ("parent", "frame", "xcnt", "xsum", "isum", "imin"):
        assert np.array_equal(np.asarray(a[key]), np.asarray(ref[key])), key


def test_seq_associate_and_bwd_fwd_rule_vs_oracle():
    """NEXT-4: forward/backward association (registry with repeated and negative ids, unknown ids)
    == the oracle's replay; then ③ on the CCT of the integrated paths == the oracle's."""
    import torch
    import paper_2411_02797_b200 as dc
    rng = np.random.default_rng(9500)
    ctx = dc.Context(0)
    nf, nb = 3000, 20_000
    fwd_seq = rng.integers(-1, 2500, nf).astype(np.int64)
    fwd_paths = [[int(x) for x in rng.integers(0, 40, size=int(rng.integers(0, 6)))] for _ in range(nf)]
    bwd_seq = rng.integers(-1, 2700, nb).astype(np.int64)
    bwd_paths = [[int(x) for x in rng.integers(40, 60, size=int(rng.integers(0, 5)))] for _ in range(nb)]
    foff, ffr = _csr(fwd_paths)
    boff, bfr = _csr(bwd_paths)
    cu = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()  # noqa: E731
    off, fr, unm = dc.dc_seq_associate(ctx, cu(fwd_seq, np.int64), cu(foff, np.int64), cu(ffr, np.int32),
                                       cu(bwd_seq, np.int64), cu(boff, np.int64), cu(bfr, np.int32))
    exp, eunm = oracle.seq_associate(fwd_seq, fwd_paths, bwd_seq, bwd_paths)
    o_np, f_np = off.cpu().numpy().view(np.uint64), fr.cpu().numpy().view(np.uint32)
    got = [f_np[o_np[r]:o_np[r + 1]].tolist() for r in range(nb)]
    assert got == exp and unm == eunm and unm > 0
    # ③ over the integrated paths: metric 0 = backward time, 1 = forward time
    X = np.zeros((2, nb), np.uint64)
    t = rng.integers(1, 10**6, nb).astype(np.uint64)
    back = rng.random(nb) < 0.5
    X[0, back] = t[back]
    X[1, ~back] = t[~back]
    a = gpu_run(o_np, f_np, X, n_frames=60, ctx=ctx)
    ref = oracle_run(o_np, f_np, X, 2)
    for thr, floor in [(2.0, 1), (1.0, 10**5), (0.5, 0)]:
        got = dc.dc_analyze_flags(ctx, a["_cct"], dc.DC_RULE_BWD_FWD, 0, 1, 0xFFFFFFFF, thr, floor)
        assert got == ref.rule_flags(oracle.RULE_BWD_FWD, 0, 1, threshold=thr, floor=floor), (thr, floor)


INV_KEYS = ["parent", "frame", "depth", "xcnt", "icnt", "xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]


def _same_inverted(got, ref, what):
    assert got["n_nodes"] == ref["n_nodes"], what
    for k in INV_KEYS:
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), (what, k)


@pytest.mark.parametrize("seed", range(3))
def test_inverted_random_vs_oracle(seed):
    """NEXT-3 bottom-up caller inversion (dc_cct_invert, reading R27): every array of the
    inverted tree equals oracle.inverted, for a metric and for the PC-sample column."""
    import paper_2411_02797_b200 as dc
    rng = np.random.default_rng(9300 + seed)
    ctx = dc.Context(0)
    for it in range(20):
        paths, X, samples, S = _rand_trace(rng)
        off, fr = _csr(paths)
        A = 1 + max([f for p in paths for f in p] + [0])
        Xa = np.asarray(X, np.uint64).reshape(len(X), -1)
        smp = _samples(samples)
        a = gpu_run(off, fr, Xa, n_frames=A, samples=smp, n_stall=S, ctx=ctx)
        ref = oracle_run(off, fr, Xa, Xa.shape[0], smp, len(paths), S).arrays()
        for m in list(range(Xa.shape[0])) + [dc.DC_METRIC_SAMPLES]:
            inv = dc.dc_cct_invert(ctx, a["_cct"], m)
            _same_inverted(inv.to_numpy(), oracle.inverted(ref, oracle.METRIC_SAMPLES if m == dc.DC_METRIC_SAMPLES else m),
                           f"seed {seed} it {it} metric {m}")
            inv.free()


def test_inverted_config2_vs_oracle_and_views():
    """Config 2 (ResNet-50-shaped, 1M launches, M = 5, kinds from the dictionary): the inverted
    tree of the kernel time equals the oracle's; its roots' hotspot view (kernel kind) equals
    the bottom-up view of the original tree."""
    import paper_2411_02797_b200 as dc
    p = gen.programs.program(2)
    tr = gen.make_trace(p, n_records=300_000)
    a = gpu_run(tr.offsets.numpy(), keys=tr.keys.numpy(), metrics=tr.metrics.numpy())
    oids, odict = oracle.intern(tr.keys.numpy())
    ref = oracle_run(tr.offsets.numpy(), oids, tr.metrics.numpy(), p.n_metrics).arrays()
    ctx, cct = a["_ctx"], a["_cct"]
    inv = dc.dc_cct_invert(ctx, cct, 0)
    _same_inverted(inv.to_numpy(), oracle.inverted(ref, 0), "config 2")
    km = 1 << dc.DC_KIND_KERNEL
    bu = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_BOTTOM_UP, 0, km, 0.0, 50)
    iv = dc.dc_hotspots_topk(ctx, inv, dc.DC_VIEW_INCLUSIVE, 0, km, 0.0, 1 << 10)
    ia = inv.to_numpy()
    roots = [(int(ia["frame"][i]), val) for i, val, _ in iv if ia["depth"][i] == 1][:50]
    assert roots == [(i, v) for i, v, _ in bu]
