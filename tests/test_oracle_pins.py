"""Pins of the CPU oracle against things other than itself (runs without a GPU).

* brute force by definition on >= 1000 random tiny traces (tests/bruteforce.py);
* SPEC.md / paper worked examples and the F1 fixture (tests/golden/f1.json);
* closed forms (complete b-ary tree, recursion chain, star);
* invariants on generated configs;
* Python's correctly rounded int -> float for the 256-bit RNE conversion.
"""
import json
import math
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import bruteforce as bf
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def csr(paths):
    off = np.zeros(len(paths) + 1, np.uint64)
    off[1:] = np.cumsum([len(p) for p in paths])
    fr = np.asarray([f for p in paths for f in p], np.uint32)
    return off, fr


def run(paths, X, samples=None, n_stall=0):
    off, fr = csr(paths)
    o = oracle.OracleCCT(len(X), n_stall).insert(off, fr, np.asarray(X, np.uint64).reshape(len(X), -1))
    if samples is not None:
        s = np.zeros(len(samples), oracle.SAMPLE_DTYPE)
        for i, (l, pc, st, c) in enumerate(samples):
            s[i] = (l, pc, st, 0, c)
        o.pc(s, len(paths))
    return o.finalize()


# ------------------------------------------------------------------ F1 fixture
def test_f1_fixture():
    g = json.load(open(os.path.join(GOLD, "f1.json")))
    ids, d = oracle.intern(np.asarray([(k[0], k[1], k[2]) for k in g["raw_keys"]], oracle.KEY_DTYPE))
    assert ids.tolist() == list(range(11))  # raw keys are listed in rank order
    o = run(g["paths"], g["metrics"], [tuple(s) for s in g["samples"]], g["n_stall"])
    a = o.arrays()
    for k in ["leaf", "parent", "depth", "frame", "xcnt", "icnt", "xsamples", "isamples"]:
        assert a[k].tolist() == g[k], k
    assert a["xsum"][0].tolist() == g["xsum_ns"]
    assert a["isum"][0].tolist() == g["isum_ns"]
    assert a["imin"][0].tolist() == g["imin_ns"]
    assert (a["isq_lo"][0] + (a["isq_hi"][0].astype(object) << 64)).tolist() == g["isq_ns"]
    mean, std = o.derived(0, True)
    assert mean.tolist() == g["imean_ns"]
    np.testing.assert_allclose(std, g["istd_ns"], rtol=1e-12, atol=0)
    fk = np.asarray(g["frame_kind"], np.uint8)
    hot = o.topk(oracle.VIEW_INCLUSIVE, 0, 1 << 4, fk, 0.1, 3)
    assert [[int(e["id"]), int(e["value"]), float(e["fraction"])] for e in hot] == g["hotspot_kernels_incl_ns_theta0.1_k3"]
    bu = o.topk(oracle.VIEW_BOTTOM_UP, 0, 0xFFFFFFFF, fk, 0.0, 10)
    assert [[int(e["id"]), int(e["value"])] for e in bu] == g["bottom_up_excl_ns"]
    assert list(map(list, zip(a["pc_ctx"].tolist(), a["pc_off"].tolist()))) == g["pc_nodes"]
    assert list(map(list, zip(a["bin_pcnode"].tolist(), a["bin_stall"].tolist(), a["bin_count"].tolist()))) == g["bins"]
    assert a["istall"][3].tolist() == g["istall3"] and a["istall"][7].tolist() == g["istall7"]
    assert o.diag() == g["diag"]
    for node, key in [(8, "stall_top2_node8"), (10, "stall_top2_node10")]:
        st = o.topk(oracle.VIEW_STALL, k=2, stall_node=node)
        assert [[int(e["id"]), int(e["value"]), float(e["fraction"])] for e in st] == g[key]
    # the same numbers by the plain definition
    ref = bf.cct([tuple(p) for p in g["paths"]], g["metrics"])
    assert ref["leaf"] == g["leaf"] and ref["isum"][0] == g["isum_ns"] and ref["isq"][0] == g["isq_ns"]


# ------------------------------------------------------------------ SPEC.md worked examples
def test_spec_aggregate_246():
    """SPEC.md:341 values 2,4,6 on one node -> sum 12, min 2, mean 4, std sqrt(8/3)."""
    o = run([(5,), (5,), (5,)], [[2, 4, 6]])
    a = o.arrays()
    assert a["xsum"][0][1] == 12 and a["xmin"][0][1] == 2 and a["xcnt"][1] == 3
    mean, std = o.derived(0, False)
    assert mean[1] == 4.0
    assert abs(std[1] - math.sqrt(8 / 3)) <= 1e-15 * math.sqrt(8 / 3)
    o1 = run([(5,)], [[5]])  # single value -> std 0
    assert o1.derived(0, False)[1][1] == 0.0


def test_spec_insert_semantics():
    """SPEC.md:331-333."""
    assert run([(1, 2, 3)], [[1]]).counts()["n_nodes"] == 4          # 3 nodes + root
    assert run([(1, 2, 3), (1, 2, 3)], [[1, 1]]).counts()["n_nodes"] == 4
    a = run([(1, 2), (1, 3)], [[1, 1]]).arrays()
    assert (a["parent"] == 1).sum() == 2                               # A has 2 children


def test_spec_propagation_and_exclusive():
    """SPEC.md:351-353 (propagate) and 401-402 (exclusive)."""
    a = run([(1, 2, 3)], [[10]]).arrays()
    assert a["isum"][0].tolist() == [10, 10, 10, 10] and a["icnt"].tolist() == [1, 1, 1, 1]
    a = run([(1, 2), (1, 3)], [[3, 7]]).arrays()
    assert a["isum"][0][1] == 10 and a["icnt"][1] == 2 and a["imin"][0][1] == 3
    assert a["xsum"][0][1] == 0                                         # no direct attribution
    assert a["xsum"][0][2] == a["isum"][0][2] == 3                      # leaf excl == incl


def test_spec_bottom_up():
    """kernel K attributed 20.5 s + 10.0 s under two paths -> one entry 30.5 s."""
    o = run([(1, 9), (2, 9)], [[20_500, 10_000]])
    bu = o.topk(oracle.VIEW_BOTTOM_UP, 0, 0xFFFFFFFF, None, 0.0, 10)
    assert int(bu[0]["id"]) == 9 and int(bu[0]["value"]) == 30_500


def test_spec_pc_extension():
    """SPEC.md:381-383."""
    o = run([(1, 2)], [[1]], [(0, 0xA, 3, 5), (0, 0xB, 7, 3)], n_stall=24)
    a = o.arrays()
    assert a["n_pc_nodes"] == 2 and a["xsamples"][2] == 8
    o = run([(1, 2)], [[1]], [(0, 0xA, 3, 5), (0, 0xA, 3, 4)], n_stall=24)
    a = o.arrays()
    assert a["n_pc_nodes"] == 1 and a["bin_count"].tolist() == [9]


def test_spec_hotspot_threshold_strict():
    """SPEC.md:460-461 / PAPER.md:616: 30.5 s of 77.0 s -> 0.396 > 0.10; exactly at threshold -> not flagged."""
    o = run([(1, 4), (2, 5)], [[30_500, 46_500]])
    fk = np.asarray([0, 0, 0, 0, 4, 4], np.uint8)
    hot = o.topk(oracle.VIEW_INCLUSIVE, 0, 1 << 4, fk, 0.10, 5)
    ids = [int(e["id"]) for e in hot]
    node_30 = [int(e["id"]) for e in hot if int(e["value"]) == 30_500]
    assert node_30 and abs(float(hot[ids.index(node_30[0])]["fraction"]) - 0.396) < 5e-4
    o = run([(1, 4), (2, 5)], [[10, 90]])
    hot = o.topk(oracle.VIEW_INCLUSIVE, 0, 1 << 4, fk, 0.10, 5)
    assert [int(e["value"]) for e in hot] == [90]                       # 10/100 == 0.10 is not > 0.10


def test_spec_stall_topk():
    """stalls {math_dep: 60, const_mem_miss: 30, other: 10}, k = 2 -> [math_dep, const_mem_miss]."""
    o = run([(1, 2)], [[1]], [(0, 0x10, 3, 60), (0, 0x20, 7, 30), (0, 0x30, 23, 10)], n_stall=24)
    st = o.topk(oracle.VIEW_STALL, k=2, stall_node=2)
    assert [int(e["id"]) for e in st] == [3, 7]


def test_spec_frame_identity():
    """SPEC.md:118-120 via raw keys: same module+pc -> equal; line 10 vs 11 -> unequal; op by name -> equal."""
    K = np.asarray([(2, 7, 0x4F10), (2, 7, 0x4F10), (0, 1, 10), (0, 1, 11), (1, 3, 0), (1, 3, 0)], oracle.KEY_DTYPE)
    ids, d = oracle.intern(K)
    assert ids[0] == ids[1] and ids[2] != ids[3] and ids[4] == ids[5] and len(d) == 4


def test_paper_dlrm_ratio_fixture():
    """aten::index backward 39.9 % vs forward 0.8 % of 77.0 s; ratio 49.875."""
    # fwd 0.616 s (0.8 %), bwd 30.723 s (39.9 %), rest 45.661 s
    o = run([(1, 2, 10), (1, 3, 10), (1, 4)], [[616, 30_723, 45_661]])
    a = o.arrays()
    tot = int(a["isum"][0][0])
    assert tot == 77_000
    f, b = a["isum"][0][2] / tot, a["isum"][0][3] / tot
    assert round(f * 100, 1) == 0.8 and round(b * 100, 1) == 39.9 and round(b / f, 3) == 49.875


# ------------------------------------------------------------------ brute force on random tiny traces
def _rand_trace(rng):
    R = int(rng.integers(1, 73))
    A = int(rng.integers(2, 17))
    paths = []
    for _ in range(R):
        L = int(rng.integers(0, 12))
        if paths and rng.random() < 0.3:  # prefix / extension of an earlier record
            base = list(paths[int(rng.integers(0, len(paths)))])
            L = min(L, len(base)) if rng.random() < 0.5 else L
            p = base[:L] + [int(rng.integers(0, A)) for _ in range(max(0, L - len(base)))]
        else:
            p = [int(rng.integers(0, A)) for _ in range(L)]
        if p and rng.random() < 0.1:  # recursion A->A->A
            i = int(rng.integers(0, len(p)))
            p = p[:i + 1] + [p[i]] * 2 + p[i + 1:]
        paths.append(tuple(p))
    M = int(rng.integers(1, 4))
    big = rng.random() < 0.2
    X = [[int(rng.integers(0, 2**40 if big else 1000)) for _ in range(R)] for _ in range(M)]
    S = int(rng.integers(1, 9))
    samples = [(int(rng.integers(0, R + 2)), int(rng.integers(0, 6)) * 16, int(rng.integers(0, S + 1)),
                int(rng.integers(0, 4))) for _ in range(int(rng.integers(0, 40)))]
    return paths, X, samples, S


@pytest.mark.parametrize("seed", range(10))
def test_bruteforce_random(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(110):
        paths, X, samples, S = _rand_trace(rng)
        o = run(paths, X, samples, S)
        a = o.arrays()
        ref = bf.cct(paths, X)
        N = ref["n_nodes"]
        assert a["n_nodes"] == N
        for k in ["parent", "frame", "depth", "leaf", "xcnt", "icnt"]:
            assert a[k].tolist() == ref[k], k
        for m in range(len(X)):
            for k in ["xsum", "xmin", "isum", "imin"]:
                assert a[k][m].tolist() == ref[k][m], k
            for k in ["xsq", "isq"]:
                got = [int(lo) + (int(hi) << 64) for lo, hi in zip(a[k + "_lo"][m], a[k + "_hi"][m])]
                assert got == ref[k][m], k
        pb = bf.pc_bins(ref, paths, samples, len(paths), S)
        assert list(zip(a["pc_ctx"].tolist(), a["pc_off"].tolist())) == pb["pcs"]
        assert list(zip(a["bin_pcnode"].tolist(), a["bin_stall"].tolist(), a["bin_count"].tolist())) == pb["bins"]
        assert a["xsamples"].tolist() == pb["xsamples"] and a["isamples"].tolist() == pb["isamples"]
        assert a["xstall"].tolist() == pb["xstall"] and a["istall"].tolist() == pb["istall"]
        d = o.diag()
        assert (d["samples_bad_launch"], d["samples_bad_stall"], d["samples_zero_count"]) == \
            (pb["diag"]["bad_launch"], pb["diag"]["bad_stall"], pb["diag"]["zero"])
        assert d["empty_paths"] == sum(1 for p in paths if not p)
        # views against a plain sort of the definition's values
        fk = rng.integers(0, 6, size=16).astype(np.uint8)
        mask = int(rng.integers(1, 64))
        th = float(rng.choice([-1.0, 0.0, 0.05, 0.2]))
        k = int(rng.integers(1, 8))
        m = int(rng.integers(0, len(X)))
        cand = [i for i in range(1, N) if (mask >> int(fk[ref["frame"][i]])) & 1]
        for view, col in [(oracle.VIEW_INCLUSIVE, "isum"), (oracle.VIEW_EXCLUSIVE, "xsum")]:
            got = [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in o.topk(view, m, mask, fk, th, k)]
            assert got == bf.topk_nodes(ref[col][m], ref["isum"][m][0], cand, th, k)
        byf = {}
        for i in cand:
            byf[ref["frame"][i]] = byf.get(ref["frame"][i], 0) + ref["xsum"][m][i]
        fr = sorted(byf)
        vals = {f: byf[f] for f in fr}
        exp = bf.topk_nodes(vals, ref["isum"][m][0], fr, th, k) if fr else []
        got = [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in o.topk(oracle.VIEW_BOTTOM_UP, m, mask, fk, th, k)]
        assert got == exp
        node = int(rng.integers(0, N))
        st = [pb["istall"][s][node] for s in range(S)]
        got = [(int(e["id"]), int(e["value"]), float(e["fraction"])) for e in o.topk(oracle.VIEW_STALL, 0, 0, None, th, k, node)]
        assert got == bf.topk_nodes(st, pb["isamples"][node], list(range(S)), th, k)


# ------------------------------------------------------------------ derived floats
def test_derived_against_exact():
    getcontext().prec = 60
    rng = np.random.default_rng(7)
    for _ in range(40):
        R = int(rng.integers(1, 50))
        big = [0, 2**20, 2**40, 2**47][int(rng.integers(0, 4))]
        X = [[int(rng.integers(0, big + 1000)) for _ in range(R)]]
        paths = [(int(rng.integers(0, 3)),) for _ in range(R)]
        o = run(paths, X)
        ref = bf.cct(paths, X)
        mean, std = o.derived(0, True)
        for i in range(ref["n_nodes"]):
            n, s1, s2 = ref["icnt"][i], ref["isum"][0][i], ref["isq"][0][i]
            em = Fraction(s1, n)
            assert abs(Fraction(mean[i]) - em) <= em * Fraction(1, 2**51)
            D = n * s2 - s1 * s1
            es = Decimal(D).sqrt() / Decimal(n)
            assert abs(Decimal(std[i]) - es) <= es * Decimal(2) ** -50


def test_u256_rne_against_python():
    rng = np.random.default_rng(11)
    vals = [0, 1, 2**53 - 1, 2**53, 2**53 + 1, 2**54 + 2, 2**54 + 6, 2**191 + 2**138, 2**191 + 2**138 + 1, 2**192 - 1]
    vals += [int.from_bytes(rng.bytes(24), "little") >> int(rng.integers(0, 190)) for _ in range(2000)]
    for v in vals:
        limbs = [(v >> (64 * q)) & (2**64 - 1) for q in range(4)]
        assert oracle.u256_to_double(limbs) == float(v), v   # Python int->float is correctly rounded


# ------------------------------------------------------------------ closed forms
def test_closed_form_bary():
    b, Dt, c, v = 4, 6, 3, 7
    paths = []
    for leaf in range(b ** Dt):
        digits = [(leaf // b ** (Dt - 1 - d)) % b for d in range(Dt)]
        paths += [tuple(d * b + j for d, j in enumerate(digits))] * c
    a = run(paths, [[v] * len(paths)]).arrays()
    assert a["n_nodes"] == (b ** (Dt + 1) - 1) // (b - 1)
    for d in range(Dt + 1):
        sel = a["depth"] == d
        assert (a["icnt"][sel] == c * b ** (Dt - d)).all()
        assert (a["isum"][0][sel] == c * v * b ** (Dt - d)).all()
        assert (a["xcnt"][sel] == (c if d == Dt else 0)).all()


def test_closed_form_recursion_chain():
    K = 256
    paths = [tuple([7] * k) for k in range(1, K + 1)]
    a = run(paths, [[1] * K]).arrays()
    assert a["n_nodes"] == K + 1 and a["depth"].max() == K
    assert a["icnt"].tolist() == [K] + [K - d + 1 for d in range(1, K + 1)]
    assert a["xcnt"].tolist() == [0] + [1] * K


def test_closed_form_star():
    W = 20_000
    paths = [(0, 1 + f) for f in range(W)]
    a = run(paths, [[3] * W]).arrays()
    assert a["n_nodes"] == W + 2 and (a["parent"] == 1).sum() == W
    assert a["frame"][2:].tolist() == list(range(1, W + 1))


# ------------------------------------------------------------------ invariants on generated configs
def check_invariants(a, R, X, total_valid_samples=None):
    N = a["n_nodes"]
    par, dep, fr = a["parent"].astype(np.int64), a["depth"].astype(np.int64), a["frame"]
    assert par[0] == 0xFFFFFFFF and dep[0] == 0
    assert (par[1:] < np.arange(1, N)).all()
    assert (dep[1:] == dep[par[1:]] + 1).all()
    # siblings strictly ascending by frame, levels contiguous, children grouped by parent
    assert (np.diff(dep) >= 0).all()
    key = par[1:] * 2**32 + fr[1:].astype(np.int64)
    assert (np.diff(key) > 0).all()
    assert a["icnt"][0] == R and a["xcnt"].sum() == R
    for m in range(len(X)):
        assert int(a["isum"][m][0]) == int(np.asarray(X[m], np.uint64).astype(object).sum())
        # incl = excl (+) sum of children incl
        s = a["xsum"][m].astype(object).copy()
        cnt = a["xcnt"].astype(object).copy()
        mn = a["xmin"][m].copy()
        for n in range(N - 1, 0, -1):
            s[par[n]] += a["isum"][m][n]
            mn[par[n]] = min(mn[par[n]], a["imin"][m][n])
        assert (s == a["isum"][m].astype(object)).all() and (mn == a["imin"][m]).all()
    for n in range(N - 1, 0, -1):
        cnt[par[n]] += a["icnt"][n]
    assert (cnt == a["icnt"].astype(object)).all()
    if total_valid_samples is not None:
        assert int(a["bin_count"].sum()) == total_valid_samples == int(a["isamples"][0])


@pytest.mark.parametrize("cfg,R", [(1, None), (2, 50_000), (3, 2_000)])
def test_invariants_generated(cfg, R):
    import gen
    p = gen.programs.program(cfg) if cfg != 3 else gen.programs.config3(n_samples=2_000_000)
    tr = gen.make_trace(p, n_records=R, pc=(cfg == 3), n_launch=R if cfg == 3 else None, bad_per_million=2000)
    X = tr.metrics.numpy().view(np.uint64)
    o = oracle.OracleCCT(p.n_metrics, 24).insert(tr.offsets.numpy(), tr.ids.numpy(), X)
    valid = None
    if cfg == 3:
        s = tr.samples.numpy().view(np.uint32).reshape(-1, 4)
        stall = s[:, 2] & 0xFFFF
        ok = (s[:, 0] < tr.n_launch) & (stall < 24) & (s[:, 3] > 0)
        valid = int(s[ok, 3].astype(np.int64).sum())
        o.pc(tr.samples.numpy(), tr.n_launch)
    a = o.finalize().arrays()
    check_invariants(a, tr.n_records, X, valid)
    # raw-key interning agrees with the generator's pool ranks on this trace's distinct keys
    ids, d = oracle.intern(tr.keys.numpy())
    used = np.unique(tr.ids.numpy())
    assert len(d) == len(used) and (used[ids] == tr.ids.numpy().astype(np.int64)).all()
