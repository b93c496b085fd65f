"""Brute-force reference for tiny traces: the CCT by its plain definition, no trie.

Independent of oracle/ (shares no code): the CCT's nodes are the root plus every distinct
prefix q of any record path p_r ("inserting call paths ... collapsing
frames that refer to the same locations"); excl(q) aggregates the records with p_r == q and
incl(q) the records with q a prefix of p_r (propagation to the root).
Canonical ids sort the prefixes by (length, lexicographic frame-id sequence) — DESIGN.md
reading R2, equivalent to BFS with children in ascending frame id. Python ints are exact.
"""
from __future__ import annotations

U64_MAX = (1 << 64) - 1


def cct(paths: list[tuple[int, ...]], X: list[list[int]]):
    """paths: list of frame-id tuples; X[m][r]. Returns dict of python lists."""
    M = len(X)
    prefixes = {()}
    for p in paths:
        for d in range(1, len(p) + 1):
            prefixes.add(tuple(p[:d]))
    order = sorted(prefixes, key=lambda q: (len(q), q))
    ids = {q: i for i, q in enumerate(order)}
    N = len(order)
    out = dict(parent=[0xFFFFFFFF if not q else ids[q[:-1]] for q in order],
               frame=[0xFFFFFFFF if not q else q[-1] for q in order], depth=[len(q) for q in order],
               leaf=[ids[tuple(p)] for p in paths])
    xcnt, icnt = [0] * N, [0] * N
    agg = {k: [[0 if "min" not in k else U64_MAX] * N for _ in range(M)] for k in ["xsum", "xmin", "xsq", "isum", "imin", "isq"]}
    for r, p in enumerate(paths):
        p = tuple(p)
        for d in range(0, len(p) + 1):
            q = ids[p[:d]]
            icnt[q] += 1
            for m in range(M):
                v = X[m][r]
                agg["isum"][m][q] += v
                agg["imin"][m][q] = min(agg["imin"][m][q], v)
                agg["isq"][m][q] += v * v
        q = ids[p]
        xcnt[q] += 1
        for m in range(M):
            v = X[m][r]
            agg["xsum"][m][q] += v
            agg["xmin"][m][q] = min(agg["xmin"][m][q], v)
            agg["xsq"][m][q] += v * v
    out.update(xcnt=xcnt, icnt=icnt, **agg, order=order, ids=ids, n_nodes=N)
    return out


def pc_bins(bf, paths, samples, n_launch: int, n_stall: int):
    """Group-by definition of the (context, pc, stall) histogram. samples: (launch, pc, stall, count)."""
    valid = [(l, pc, s, c) for (l, pc, s, c) in samples if l < n_launch and s < n_stall and c > 0]
    diag = dict(bad_launch=sum(1 for (l, _, _, _) in samples if l >= n_launch),
                bad_stall=sum(1 for (l, _, s, _) in samples if l < n_launch and s >= n_stall),
                zero=sum(1 for (l, _, s, c) in samples if l < n_launch and s < n_stall and c == 0))
    bins: dict[tuple[int, int, int], int] = {}
    for (l, pc, s, c) in valid:
        ctx = bf["leaf"][l]
        bins[(ctx, pc, s)] = bins.get((ctx, pc, s), 0) + c
    N = bf["n_nodes"]
    pcs = sorted({(ctx, pc) for (ctx, pc, _) in bins})
    pcid = {k: N + i for i, k in enumerate(pcs)}
    cb = sorted((pcid[(ctx, pc)], s, c) for (ctx, pc, s), c in bins.items())
    xs, xst = [0] * N, [[0] * N for _ in range(n_stall)]
    iss, ist = [0] * N, [[0] * N for _ in range(n_stall)]
    for (l, pc, s, c) in valid:
        p = tuple(paths[l])
        ctx = bf["ids"][p]
        xs[ctx] += c
        xst[s][ctx] += c
        for d in range(len(p) + 1):  # every prefix of the context's path
            q = bf["ids"][p[:d]]
            iss[q] += c
            ist[s][q] += c
    return dict(pcs=pcs, bins=cb, xsamples=xs, isamples=iss, xstall=xst, istall=ist, diag=diag)


def topk_nodes(values: list[int], total: int, cand: list[int], threshold: float, k: int):
    if total == 0:
        return []
    keep = [(i, v, v / total) for i, v in ((i, values[i]) for i in cand) if v / total > threshold]
    keep.sort(key=lambda e: (-e[1], e[0]))
    return keep[:k]
