"""Pins of the oracle's analyzer rules against the paper / SPEC worked
examples and a brute-force definition on random trees (independent of oracle/: the CCT is
rebuilt from distinct prefixes by tests/bruteforce.py).

② small kernels, PAPER.md:398-404 `n.gpu_time / n.count < gpu_threshold` over bfs(nodes);
⑤ CPU latency, PAPER.md:428-434 `n.cpu_time / n.gpu_time > cpu_threshold`;
④ fine-grained stalls; readings R22-R23 from SPEC.md
analyze_kernel_fusion / analyze_cpu_latency / analyze_stalls.
"""
import numpy as np
import pytest

import bruteforce as bf
import oracle
from test_oracle_pins import _rand_trace, run

KERNEL = 4
PY = 0


def test_spec_kernel_fusion_transformer_fixture():
    """SPEC.md analyze_kernel_fusion: loss_fn launches softmax, copy and
    nll_loss with equal counts and short kernels -> flagged at loss_fn, its kernels not
    re-flagged; a frame with 1 ms kernels is not flagged (threshold 20 us)."""
    # frames: 0 train.py:10, 1 loss_fn, 2 model_fwd (PY); 3 softmax, 4 copy, 5 nll_loss, 6 gemm (KERNEL)
    fk = np.array([PY, PY, PY, KERNEL, KERNEL, KERNEL, KERNEL], np.uint8)
    paths, ns = [], []
    for k in (3, 4, 5):
        paths += [(0, 1, k)] * 100
        ns += [5_000] * 100
    paths += [(0, 2, 6)] * 100
    ns += [1_000_000] * 100
    o = run(paths, [ns])
    ids = {tuple(q): i for i, q in enumerate(bf.cct(paths, [ns])["order"])}
    got = o.rule_flags(oracle.RULE_SMALL_KERNELS, 0, kind_mask=1 << KERNEL, frame_kind=fk, threshold=20_000.0)
    assert got == [ids[(0, 1)]]
    # one kernel of 1 ms, threshold 20 us -> nothing (SPEC.md: TRIVIAL)
    o2 = run([(0, 6)], [[1_000_000]])
    assert o2.rule_flags(oracle.RULE_SMALL_KERNELS, 0, kind_mask=1 << KERNEL, frame_kind=fk, threshold=20_000.0) == []


def test_spec_cpu_latency_fixtures():
    """SPEC.md analyze_cpu_latency: U-Net data_selection (69 % of CPU time, 1.3 s GPU) flagged;
    zero GPU time with 50 ms CPU and threshold 5 flagged through max(gpu, 1); a balanced frame
    not flagged; the 1 ms floor."""
    # metric 0 = cpu ns, metric 1 = gpu ns; frames 0 main, 1 data_selection, 2 train_step, 3 idle, 4 balanced
    paths = [(0, 1), (0, 2), (0, 3), (0, 4), (0, 4)]
    cpu = [69_000_000_000, 31_000_000_000, 50_000_000, 2_000_000, 2_000_000]
    gpu = [1_300_000_000, 40_000_000_000, 0, 2_000_000, 2_000_000]
    o = run(paths, [cpu, gpu])
    ids = {tuple(q): i for i, q in enumerate(bf.cct(paths, [cpu, gpu])["order"])}
    got = o.rule_flags(oracle.RULE_CPU_LATENCY, 0, 1, threshold=5.0, floor=1_000_000)
    assert got == [ids[(0, 1)], ids[(0, 3)]]
    # the floor: 50 ms of CPU below a 100 ms floor is not flagged
    assert o.rule_flags(oracle.RULE_CPU_LATENCY, 0, 1, threshold=5.0, floor=100_000_000) == [ids[(0, 1)]]


def test_spec_stall_issue_fixture():
    """SPEC.md analyze_stalls: hotspot kernel with {math_dep: 60, const_mem_miss: 30, other: 10}
    of 100 samples on three instructions, threshold 0.2, k = 2 -> [math_dep, const_mem_miss]
    (PAPER.md:699-702 names both reasons for the Llama3 RMSNorm kernel)."""
    MATH, CONST, OTHER = 3, 7, 19
    paths = [(0, 1)]
    samples = [(0, 0xA0, MATH, 60), (0, 0xB0, CONST, 30), (0, 0xC0, OTHER, 10)]
    o = run(paths, [[100]], samples, n_stall=24)
    got = o.stall_issues(0, hot_threshold=0.5, stall_threshold=0.2, k=2)
    assert got == [(2, MATH, 60), (2, CONST, 30)]
    # an instruction mixing reasons counts all of its reasons once it passes the threshold
    samples = [(0, 0xA0, MATH, 50), (0, 0xA0, OTHER, 5), (0, 0xB0, CONST, 10), (0, 0xC0, OTHER, 35)]
    o = run(paths, [[100]], samples, n_stall=24)
    assert o.stall_issues(0, hot_threshold=0.5, stall_threshold=0.2, k=3) == [(2, MATH, 50), (2, OTHER, 40)]
    # a kernel with no instruction samples -> no issue (SPEC.md: TRIVIAL)
    o = run(paths, [[100]], [], n_stall=24)
    assert o.stall_issues(0, hot_threshold=0.5, stall_threshold=0.2, k=3) == []


def _bf_flags(b, paths, X, rule, ma, mb, fk, mask, thr, floor):
    """Flagged ids by the plain definition: BFS (= (depth, lex) order), ancestor suppression."""
    N = b["n_nodes"]
    order = b["order"]
    launches = [0] * N
    for r, p in enumerate(paths):
        if p and (fk is None or (int(fk[p[-1]]) < 32 and (mask >> int(fk[p[-1]])) & 1)):
            for d in range(1, len(p) + 1):
                launches[b["ids"][tuple(p[:d])]] += 1

    def q(i):
        if rule == 2:
            return launches[i] > 0 and b["isum"][ma][i] / launches[i] < thr
        if rule == 3:
            f = order[i][-1]
            kind_ok = fk is None or (int(fk[f]) < 32 and (mask >> int(fk[f])) & 1)
            bwd, fwd = b["isum"][ma][i], b["isum"][mb][i]
            return bool(kind_ok) and fwd > 0 and fwd >= floor and bwd / fwd > thr
        cpu, gpu = b["isum"][ma][i], b["isum"][mb][i]
        return cpu > floor and cpu / max(gpu, 1) > thr

    flagged = []
    for i in range(1, N):
        anc = [b["ids"][order[i][:d]] for d in range(1, len(order[i]))]
        if q(i) and (rule == 3 or not any(q(a) for a in anc)):
            flagged.append(i)
    return flagged


@pytest.mark.parametrize("seed", range(6))
def test_rules_bruteforce_random(seed):
    rng = np.random.default_rng(7000 + seed)
    for _ in range(60):
        paths, X, samples, S = _rand_trace(rng)
        A = 1 + max([f for p in paths for f in p] + [0])
        fk = rng.integers(0, 6, size=A).astype(np.uint8)
        b = bf.cct(paths, X)
        o = run(paths, X)
        M = len(X)
        for rule in (2, 3, 5):
            ma, mb = int(rng.integers(0, M)), int(rng.integers(0, M))
            vals = [v for row in X for v in row] or [1]
            thr = float(rng.choice([0.5, 1.0, 2.0, float(np.median(vals)) + 0.5]))
            floor = int(rng.choice([0, int(np.median(vals))]))
            mask = int(rng.choice([1 << KERNEL, 0b110000, 0xFFFFFFFF]))
            exp = _bf_flags(b, paths, X, rule, ma, mb, fk, mask, thr, floor)
            got = o.rule_flags(rule, ma, mb, kind_mask=mask, frame_kind=fk, threshold=thr, floor=floor)
            assert got == exp, (rule, thr, floor, mask)


@pytest.mark.parametrize("seed", range(4))
def test_stall_issues_bruteforce_random(seed):
    rng = np.random.default_rng(8100 + seed)
    for _ in range(60):
        paths, X, samples, S = _rand_trace(rng)
        b = bf.cct(paths, X)
        pcb = bf.pc_bins(b, paths, samples, len(paths), S)
        o = run(paths, X, samples, n_stall=S)
        hot_thr = float(rng.choice([0.0, 0.05, 0.2]))
        st_thr = float(rng.choice([0.0, 0.1, 0.3]))
        k = int(rng.integers(1, 5))
        # hotspots by definition: all non-root nodes, inclusive metric 0, (value desc, id asc)
        hot = bf.topk_nodes(b["isum"][0], b["isum"][0][0], list(range(1, b["n_nodes"])), hot_thr, b["n_nodes"])
        exp = []
        for (n, _, _) in hot:
            kids = {pid: 0 for pid, (ctx, pc) in enumerate(pcb["pcs"], start=b["n_nodes"]) if ctx == n}
            for (pid, s, c) in pcb["bins"]:
                if pid in kids:
                    kids[pid] += c
            tot = pcb["isamples"][n]
            reasons = {}
            for (pid, s, c) in pcb["bins"]:
                if pid in kids and tot > 0 and kids[pid] / tot > st_thr:
                    reasons[s] = reasons.get(s, 0) + c
            r = sorted(((c, s) for s, c in reasons.items() if c), key=lambda e: (-e[0], e[1]))[:k]
            exp += [(n, s, c) for c, s in r]
        got = o.stall_issues(0, hot_threshold=hot_thr, stall_threshold=st_thr, k=k)
        assert got == exp


# ------------------------------------------------------------------ NEXT-3: folded stacks
def test_spec_folded_example():
    """SPEC.md export_folded: main -> train -> kernel with exclusive 3050 at the kernel ->
    "main;train.py:10;conv_kern 3050"; an empty tree gives an empty text; ';' in labels -> ','."""
    labels = ["main", "train.py:10", "conv_kern"]
    o = run([(0, 1, 2)], [[3050]])
    assert oracle.folded(o.arrays(), 0, labels) == "main;train.py:10;conv_kern 3050\n"
    assert oracle.folded(run([], [[]]).arrays(), 0, labels) == ""
    assert oracle.folded(run([(0,)], [[5]]).arrays(), 0, ["a;b"]) == "a,b 5\n"


@pytest.mark.parametrize("seed", range(4))
def test_folded_bruteforce_and_conservation(seed):
    rng = np.random.default_rng(8500 + seed)
    for _ in range(60):
        paths, X, samples, S = _rand_trace(rng)
        A = 1 + max([f for p in paths for f in p] + [0])
        labels = [f"f{i}" for i in range(A)]
        b = bf.cct(paths, X)
        o = run(paths, X)
        text = oracle.folded(o.arrays(), 0, labels)
        exp = "".join(";".join(labels[f] for f in q) + f" {b['xsum'][0][i]}\n"
                      for i, q in enumerate(b["order"]) if i > 0 and b["xsum"][0][i])
        assert text == exp
        # conservation: lines + the root's own (empty-path) value == the root inclusive value
        total = sum(int(line.rsplit(" ", 1)[1]) for line in text.splitlines())
        assert total + b["xsum"][0][0] == b["isum"][0][0]


# ------------------------------------------------------------------ NEXT-4: CPU-sample intervals
def test_spec_cpu_sample_intervals():
    """SPEC.md attribute_cpu_sample: samples at t=100, 350 on one stream -> one interval 250; a
    single sample -> none; alternating paths A, B at t=0, 10, 30 on one thread -> A baseline,
    B 10, A 20 (the interval goes to the sample's own path); streams are per (thread, kind)."""
    assert oracle.cpu_intervals([1, 1], [0, 0], [100, 350]) == ([0, 250], [False, True])
    assert oracle.cpu_intervals([1], [0], [100]) == ([0], [False])
    iv, ok = oracle.cpu_intervals([7, 7, 7], [0, 0, 0], [0, 10, 30])
    paths = ["A", "B", "A"]
    attributed = [(p, v) for p, v, o in zip(paths, iv, ok) if o]
    assert attributed == [("B", 10), ("A", 20)]
    # two threads and two kinds interleaved: four independent streams
    iv, ok = oracle.cpu_intervals([1, 2, 1, 1, 2, 1], [0, 0, 1, 0, 0, 1], [5, 6, 7, 15, 26, 27])
    assert iv == [0, 0, 0, 10, 20, 20] and ok == [False, False, False, True, True, True]


def test_cpu_intervals_sum_law():
    """Per stream the intervals telescope: their sum == last ts - first ts."""
    rng = np.random.default_rng(8800)
    n = 5000
    th = rng.integers(0, 7, n)
    kd = rng.integers(0, 2, n)
    ts = np.cumsum(rng.integers(0, 1000, n))
    iv, ok = oracle.cpu_intervals(th, kd, ts)
    for t in range(7):
        for k in range(2):
            sel = [i for i in range(n) if th[i] == t and kd[i] == k]
            if sel:
                assert sum(iv[i] for i in sel) == int(ts[sel[-1]] - ts[sel[0]])
                assert [ok[i] for i in sel] == [False] + [True] * (len(sel) - 1)


# ------------------------------------------------------------------ NEXT-4: forward/backward
def test_spec_associate_backward():
    """SPEC.md associate_backward: registry has seq 7 -> the output's root section is the forward
    prefix of seq 7; an absent id -> the backward path unchanged + 1 diagnostic; two backward ops
    with seq 7 get identical prefixes; a later registry entry replaces an earlier one."""
    fwd_seq = [7, 3, 7]
    fwd = [[0, 1, 5], [0, 2], [0, 1, 6]]          # the second seq-7 entry replaces the first
    bwd_seq = [7, 9, 7, -1]
    bwd = [[20, 21], [22], [23], [24]]
    paths, unmatched = oracle.seq_associate(fwd_seq, fwd, bwd_seq, bwd)
    assert paths == [[0, 1, 6, 20, 21], [22], [0, 1, 6, 23], [24]] and unmatched == 1


def test_spec_fwd_bwd_rule_dlrm_fixture():
    """③ (SPEC.md analyze_fwd_bwd): DLRM aten::index forward 0.8 % vs backward
    39.9 % of the time -> ratio 49.9 > 2 -> flagged; forward == backward -> not
    flagged; forward below the epsilon -> skipped."""
    OP, KERNEL = 1, 4
    # frames: 0 train.py (PY), 1 aten::index (OP), 2 aten::mm (OP), 3 fwd kernel, 4 bwd kernel (KERNEL)
    fk = np.array([0, OP, OP, KERNEL, KERNEL], np.uint8)
    # metric 0 = backward time, metric 1 = forward time (a record's time in its direction's column)
    paths = [(0, 1, 3), (0, 1, 4), (0, 2, 3), (0, 2, 4)]
    bwd = [0, 39_900, 0, 500]
    fwd = [800, 0, 500, 0]
    o = run(paths, [bwd, fwd])
    ids = {tuple(q): i for i, q in enumerate(bf.cct(paths, [bwd, fwd])["order"])}
    got = o.rule_flags(oracle.RULE_BWD_FWD, 0, 1, kind_mask=1 << OP, frame_kind=fk, threshold=2.0, floor=1)
    assert got == [ids[(0, 1)]]
    assert abs(39_900 / 800 - 49.875) < 1e-12
    # epsilon: a forward time below the floor is skipped
    assert o.rule_flags(oracle.RULE_BWD_FWD, 0, 1, kind_mask=1 << OP, frame_kind=fk, threshold=2.0, floor=1000) == []


# ------------------------------------------------------------------ NEXT-3: bottom-up (inverted) tree
def test_inverted_hand_example():
    """Reading R27 by hand (PAPER.md:444-446 bottom-up view; SPEC.md bottom-up: a kernel under
    two call paths aggregates into one entry): frames A=0, B=1, C=2, K=3; records
    [A,B,K]=20, [C,B,K]=10, [A,K]=5, [A,B]=7 -> reversed [K,B,A]=20, [K,B,C]=10, [K,A]=5, [B,A]=7;
    roots B (7) and K (35 = 20 + 10 + 5); K's callers A (5) and B (30); B-under-K's callers A (20)
    and C (10)."""
    o = run([(0, 1, 3), (2, 1, 3), (0, 3), (0, 1)], [[20, 10, 5, 7]])
    v = oracle.inverted(o.arrays(), 0)
    assert v["n_nodes"] == 8
    assert v["frame"].tolist()[1:] == [1, 3, 0, 0, 1, 0, 2]
    assert v["parent"].tolist()[1:] == [0, 0, 1, 2, 2, 5, 5]
    assert v["depth"].tolist() == [0, 1, 1, 2, 2, 2, 3, 3]
    assert v["isum"][0].tolist() == [42, 7, 35, 7, 5, 30, 20, 10]
    assert v["icnt"].tolist() == [4, 1, 3, 1, 1, 2, 1, 1]
    assert v["imin"][0].tolist() == [5, 7, 5, 7, 5, 10, 20, 10]
    assert v["xsum"][0].tolist() == [0, 0, 0, 7, 5, 0, 20, 10]


def test_inverted_recursion_chain_closed_form():
    """Paths A^k, k = 1..K, one record each of value 1: node A^j has exclusive 1, its reversed
    path is A^j again, so the inverted tree is the same chain with inclusive count K - d + 1 at
    depth d (a closed form, no oracle needed)."""
    K = 40
    o = run([(0,) * k for k in range(1, K + 1)], [[1] * K])
    v = oracle.inverted(o.arrays(), 0)
    assert v["n_nodes"] == K + 1
    assert v["icnt"].tolist() == [K] + [K - d + 1 for d in range(1, K + 1)]
    assert v["parent"].tolist()[1:] == list(range(K))


@pytest.mark.parametrize("seed", range(4))
def test_inverted_bruteforce_records_and_bottom_up_view(seed):
    """Against the definition computed from the RECORDS (no CCT): group records by their whole
    path, drop the empty path and zero sums, reverse, aggregate every prefix; the roots' values
    also equal the oracle's own bottom-up view (C++, per-frame exclusive sums)."""
    rng = np.random.default_rng(9100 + seed)
    for _ in range(60):
        paths, X, samples, S = _rand_trace(rng)
        o = run(paths, X)
        v = oracle.inverted(o.arrays(), 0)
        ex = {}
        for p, val in zip(paths, X[0]):
            if len(p):
                ex[tuple(p)] = ex.get(tuple(p), 0) + int(val)
        pre = {(): [0, 0]}
        for p, s_ in ex.items():
            if s_ == 0:
                continue
            rev = tuple(reversed(p))
            for k in range(len(rev) + 1):
                a = pre.setdefault(rev[:k], [0, 0])
                a[0] += 1
                a[1] += s_
        order = sorted(pre, key=lambda q: (len(q), q))
        assert v["n_nodes"] == len(order)
        assert v["frame"].tolist()[1:] == [q[-1] for q in order[1:]]
        assert v["icnt"].tolist() == [pre[q][0] for q in order]
        assert v["isum"][0].tolist() == [pre[q][1] for q in order]
        bu = o.topk(oracle.VIEW_BOTTOM_UP, 0, 0xFFFFFFFF, None, -1.0, 1000)
        roots = {int(v["frame"][i]): int(v["isum"][0][i]) for i in range(1, v["n_nodes"]) if v["depth"][i] == 1}
        assert roots == {int(e["id"]): int(e["value"]) for e in bu if int(e["value"])}
