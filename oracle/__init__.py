"""CPU ORACLE (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this package. It wraps oracle/oracle.cpp (plain C++17, std::map tries, literal
propagation; see its header for the PAPER.md passage behind each function) through ctypes
and returns numpy arrays. It shares no code with paper_2411_02797_b200/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")
_lib = None

VIEW_INCLUSIVE, VIEW_EXCLUSIVE, VIEW_BOTTOM_UP, VIEW_STALL = 0, 1, 2, 3
METRIC_SAMPLES = 0xFFFFFFFF
U64_MAX = 0xFFFFFFFFFFFFFFFF


def build(force: bool = False) -> str:
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(_SRC):
        return _SO
    # -ffp-contract=off: no FMA contraction in the derived-float formulas (reading R18)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                           "-o", _SO + ".tmp", _SRC])
    os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        L.or_intern.argtypes = [P, u64, P, P, P]
        L.or_cct_new.restype = P
        L.or_cct_new.argtypes = [u32, u32]
        L.or_cct_free.argtypes = [P]
        L.or_insert.argtypes = [P, P, P, u64, P, u64]
        L.or_pc.argtypes = [P, P, u64, u64]
        L.or_finalize.argtypes = [P]
        L.or_counts.argtypes = [P, P]
        L.or_diag.argtypes = [P, P]
        L.or_get.argtypes = [P, P]
        L.or_topk.argtypes = [P, ctypes.c_int, u32, u32, P, u32, ctypes.c_double, u32, u32, P, P]
        L.or_rule_flags.argtypes = [P, ctypes.c_int, u32, u32, u32, P, u32, ctypes.c_double, ctypes.c_uint64, P, u32, P]
        L.or_stall_issues.argtypes = [P, u32, u32, P, u32, ctypes.c_double, ctypes.c_double, u32, P, u32, P]
        L.or_derived.argtypes = [P, u32, ctypes.c_int, P, P]
        L.or_u256_to_double.argtypes = [P]
        L.or_u256_to_double.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


KEY_DTYPE = np.dtype([("kind", "<u4"), ("str_id", "<u4"), ("addr", "<u8")])
SAMPLE_DTYPE = np.dtype([("launch", "<u4"), ("pc_off", "<u4"), ("stall", "<u2"), ("flags", "<u2"), ("count", "<u4")])
TOPK_DTYPE = np.dtype([("id", "<u4"), ("pad", "<u4"), ("value", "<u8"), ("fraction", "<f8")])
STALL_ISSUE_DTYPE = np.dtype([("node", "<u4"), ("stall", "<u4"), ("count", "<u8")])
RULE_SMALL_KERNELS, RULE_BWD_FWD, RULE_CPU_LATENCY = 2, 3, 5


def as_keys(keys) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(keys))
    if a.dtype != KEY_DTYPE:
        a = np.ascontiguousarray(a.view(np.uint8).reshape(-1)).view(KEY_DTYPE)
    return a


def intern(keys):
    """Raw 16-B keys -> (u32 ids, sorted dictionary of distinct keys)."""
    k = as_keys(keys)
    n = len(k)
    ids = np.zeros(max(n, 1), np.uint32)
    d = np.zeros(max(n, 1), KEY_DTYPE)
    D = ctypes.c_uint64(0)
    lib().or_intern(_p(k), n, _p(ids), _p(d), ctypes.byref(D))
    return ids[:n], d[: D.value]


class OracleCCT:
    """Per-record trie insertion + literal propagation."""

    def __init__(self, n_metrics: int, n_stall: int = 0):
        self.M, self.S = int(n_metrics), int(n_stall)
        self.h = lib().or_cct_new(self.M, self.S)
        self._final = False

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_cct_free(self.h)
            self.h = None

    def insert(self, offsets, frames, metrics):
        off = np.ascontiguousarray(np.asarray(offsets).view(np.uint64) if np.asarray(offsets).dtype == np.int64 else offsets, np.uint64)
        fr = np.ascontiguousarray(np.asarray(frames).view(np.uint32) if np.asarray(frames).dtype == np.int32 else frames, np.uint32)
        X = np.asarray(metrics)
        X = np.ascontiguousarray(X.view(np.uint64) if X.dtype == np.int64 else X, np.uint64).reshape(self.M, -1)
        R = len(off) - 1
        if fr.size == 0:
            fr = np.zeros(1, np.uint32)
        if X.size == 0:
            X = np.zeros((max(self.M, 1), 1), np.uint64)
        assert lib().or_insert(self.h, _p(off), _p(fr), R, _p(X), X.shape[1]) == 0
        return self

    def pc(self, samples, n_launch: int):
        s = np.asarray(samples)
        s = np.ascontiguousarray(np.ascontiguousarray(s).view(np.uint8).reshape(-1)).view(SAMPLE_DTYPE)
        assert lib().or_pc(self.h, _p(s), len(s), int(n_launch)) == 0
        return self

    def finalize(self):
        lib().or_finalize(self.h)
        self._final = True
        return self

    def counts(self):
        c = np.zeros(8, np.uint64)
        lib().or_counts(self.h, _p(c))
        return dict(n_nodes=int(c[0]), n_pc_nodes=int(c[1]), n_bins=int(c[2]), n_records=int(c[3]), max_depth=int(c[4]))

    def diag(self):
        d = np.zeros(4, np.uint64)
        lib().or_diag(self.h, _p(d))
        return dict(empty_paths=int(d[0]), samples_bad_launch=int(d[1]), samples_bad_stall=int(d[2]),
                    samples_zero_count=int(d[3]))

    def arrays(self) -> dict:
        """Canonical CCT as numpy arrays (names as in include/dc.h dc_cct_view)."""
        if not self._final:
            self.finalize()
        c = self.counts()
        N, Np, Nb, R = c["n_nodes"], c["n_pc_nodes"], c["n_bins"], c["n_records"]
        M, S = self.M, self.S
        a = dict(parent=np.zeros(N, np.uint32), frame=np.zeros(N, np.uint32), depth=np.zeros(N, np.uint16),
                 leaf=np.zeros(max(R, 1), np.uint32), xcnt=np.zeros(N, np.uint64), icnt=np.zeros(N, np.uint64))
        for nm in ["xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]:
            a[nm] = np.zeros((max(M, 1), N), np.uint64)
        a["xsamples"] = np.zeros(N, np.uint64)
        a["isamples"] = np.zeros(N, np.uint64)
        a["xstall"] = np.zeros((max(S, 1), N), np.uint64)
        a["istall"] = np.zeros((max(S, 1), N), np.uint64)
        a["pc_ctx"] = np.zeros(max(Np, 1), np.uint32)
        a["pc_off"] = np.zeros(max(Np, 1), np.uint32)
        a["bin_pcnode"] = np.zeros(max(Nb, 1), np.uint32)
        a["bin_stall"] = np.zeros(max(Nb, 1), np.uint16)
        a["bin_count"] = np.zeros(max(Nb, 1), np.uint64)
        order = ["parent", "frame", "depth", "leaf", "xcnt", "icnt", "xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin",
                 "isq_lo", "isq_hi", "xsamples", "isamples", "xstall", "istall", "pc_ctx", "pc_off", "bin_pcnode",
                 "bin_stall", "bin_count"]
        ptrs = (ctypes.c_void_p * len(order))(*[a[k].ctypes.data for k in order])
        assert lib().or_get(self.h, ptrs) == 0
        a["leaf"] = a["leaf"][:R]
        for nm in ["xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]:
            a[nm] = a[nm][:M]
        a["xstall"], a["istall"] = a["xstall"][:S], a["istall"][:S]
        a["pc_ctx"], a["pc_off"] = a["pc_ctx"][:Np], a["pc_off"][:Np]
        a["bin_pcnode"], a["bin_stall"], a["bin_count"] = a["bin_pcnode"][:Nb], a["bin_stall"][:Nb], a["bin_count"][:Nb]
        a.update(n_nodes=N, n_pc_nodes=Np, n_bins=Nb, n_metrics=M, n_stall=S)
        return a

    def topk(self, view: int, metric: int = 0, kind_mask: int = 0xFFFFFFFF, frame_kind=None, threshold: float = 0.0,
             k: int = 10, stall_node: int = 0):
        if not self._final:
            self.finalize()
        out = np.zeros(max(k, 1), TOPK_DTYPE)
        n = ctypes.c_uint32(0)
        fk = None if frame_kind is None else np.ascontiguousarray(frame_kind, np.uint8)
        rc = lib().or_topk(self.h, view, metric & 0xFFFFFFFF, kind_mask & 0xFFFFFFFF, _p(fk),
                           0 if fk is None else len(fk), float(threshold), k, stall_node, _p(out), ctypes.byref(n))
        assert rc == 0, rc
        return out[: n.value]

    def rule_flags(self, rule: int, metric_a: int, metric_b: int = 0, kind_mask: int = 0xFFFFFFFF, frame_kind=None,
                   threshold: float = 0.0, floor: int = 0, cap: int = 1 << 20):
        """Analyses ② (rule 2) / ⑤ (rule 5): flagged canonical node ids in BFS order."""
        if not self._final:
            self.finalize()
        out = np.zeros(max(cap, 1), np.uint32)
        n = ctypes.c_uint32(0)
        fk = None if frame_kind is None else np.ascontiguousarray(frame_kind, np.uint8)
        rc = lib().or_rule_flags(self.h, rule, metric_a, metric_b, kind_mask & 0xFFFFFFFF, _p(fk), 0 if fk is None else len(fk),
                                 float(threshold), int(floor), _p(out), cap, ctypes.byref(n))
        assert rc == 0, rc
        return out[: min(n.value, cap)].tolist()

    def stall_issues(self, metric: int = 0, kind_mask: int = 0xFFFFFFFF, frame_kind=None, hot_threshold: float = 0.0,
                     stall_threshold: float = 0.0, k: int = 3, cap: int = 1 << 16):
        """Analysis ④: (hotspot node, stall, count) entries."""
        if not self._final:
            self.finalize()
        out = np.zeros(max(cap, 1), STALL_ISSUE_DTYPE)
        n = ctypes.c_uint32(0)
        fk = None if frame_kind is None else np.ascontiguousarray(frame_kind, np.uint8)
        rc = lib().or_stall_issues(self.h, metric & 0xFFFFFFFF, kind_mask & 0xFFFFFFFF, _p(fk), 0 if fk is None else len(fk),
                                   float(hot_threshold), float(stall_threshold), k, _p(out), cap, ctypes.byref(n))
        assert rc == 0, rc
        return [(int(e["node"]), int(e["stall"]), int(e["count"])) for e in out[: min(n.value, cap)]]

    def derived(self, metric: int, incl: bool = True):
        if not self._final:
            self.finalize()
        N = self.counts()["n_nodes"]
        mean, std = np.zeros(N), np.zeros(N)
        assert lib().or_derived(self.h, metric, int(incl), _p(mean), _p(std)) == 0
        return mean, std


def run(offsets, frames, metrics, n_metrics, samples=None, n_launch=0, n_stall=0):
    """Convenience: whole oracle pipeline -> OracleCCT (finalized)."""
    o = OracleCCT(n_metrics, n_stall).insert(offsets, frames, metrics)
    if samples is not None:
        o.pc(samples, n_launch)
    return o.finalize()


def u256_to_double(limbs) -> float:
    w = np.ascontiguousarray(limbs, np.uint64)
    return lib().or_u256_to_double(_p(w))


def folded(arrays: dict, metric: int, labels) -> str:
    """SURVEY §8(f) NEXT-3 / SPEC.md export_folded, plain Python over the oracle's canonical
    arrays: one line per non-root node with a non-zero exclusive value, in node order; the
    path from the root (walking parent links) joined by ';' (';' in a label -> ','), a space,
    the integer exclusive value (reading R24: the root has no stack and no line)."""
    parent, frame = arrays["parent"], arrays["frame"]
    xsum = arrays["xsum"][metric]
    out = []
    for n in range(1, int(arrays["n_nodes"])):
        v = int(xsum[n])
        if v == 0:
            continue
        path, a = [], n
        while a != 0:
            path.append(str(labels[int(frame[a])]).replace(";", ","))
            a = int(parent[a])
        out.append(";".join(reversed(path)) + f" {v}\n")
    return "".join(out)


def cpu_intervals(thread, kind, ts):
    """SURVEY §8(f) NEXT-4, PAPER.md:359-363 / SPEC.md attribute_cpu_sample, replayed one sample
    at a time in trace order with the previous timestamp of each (thread, kind) stream: the
    first sample of a stream is the baseline (interval 0, valid False); later ones get
    ts - previous ts. Returns (intervals, valid) as Python lists."""
    prev = {}
    iv, ok = [], []
    for t, k, x in zip(list(map(int, thread)), list(map(int, kind)), list(map(int, ts))):
        key = (t, k)
        if key in prev:
            assert x >= prev[key], "timestamps must not decrease within a stream"
            iv.append(x - prev[key])
            ok.append(True)
        else:
            iv.append(0)
            ok.append(False)
        prev[key] = x
    return iv, ok


def seq_associate(fwd_seq, fwd_paths, bwd_seq, bwd_paths):
    """SURVEY §8(f) NEXT-4, PAPER.md:314-321 / SPEC.md associate_backward, replayed in order: the
    forward registry is a dict sequence id -> the forward op's Python + framework prefix (entries
    with id < 0 are not registered; a later entry replaces an earlier one); a backward record
    with a registered id gets prefix + its own frames, otherwise its own frames (an unknown id is
    counted). Returns (paths, unmatched)."""
    reg = {}
    for s, p in zip(list(map(int, fwd_seq)), fwd_paths):
        if s >= 0:
            reg[s] = list(p)
    out, unmatched = [], 0
    for s, p in zip(list(map(int, bwd_seq)), bwd_paths):
        if s >= 0 and s in reg:
            out.append(reg[s] + list(p))
        else:
            if s >= 0:
                unmatched += 1
            out.append(list(p))
    return out, unmatched



def digest(a: dict, dict_keys) -> str:
    """SURVEY.md §8(c) "Digest (large-config parity)": SHA-256 of the canonical little-endian
    serialisation of the oracle's CCT (this is the oracle's own writer; the CUDA side has a
    separate one). Layout: b"DCCCT1\\0\\0", u64 N, M, S, Npc, Nbins, D; parent u32[N], frame
    u32[N], depth u16[N], xcnt u64[N], icnt u64[N]; per metric xsum, xmin, xsq_lo, xsq_hi, isum,
    imin, isq_lo, isq_hi (u64[N] each); xsamples, isamples u64[N] (zeros without PC samples);
    per stall xstall, istall u64[N]; pc_ctx, pc_off u32[Npc]; bin_pcnode u32[Nb], bin_stall
    u16[Nb], bin_count u64[Nb]; the dictionary's 16-B keys (kind u32, str_id u32, addr u64)."""
    import hashlib
    import struct

    N, M, S = int(a["n_nodes"]), int(a["n_metrics"]), int(a["n_stall"])
    Np, Nb = int(a["n_pc_nodes"]), int(a["n_bins"])
    k = as_keys(dict_keys) if len(dict_keys) else np.zeros(0, KEY_DTYPE)
    h = hashlib.sha256()
    h.update(b"DCCCT1\0\0" + struct.pack("<6Q", N, M, S, Np, Nb, len(k)))

    def put(x, dt):
        h.update(np.ascontiguousarray(np.asarray(x).astype(dt, copy=False)).tobytes())

    put(a["parent"][:N], "<u4")
    put(a["frame"][:N], "<u4")
    put(a["depth"][:N], "<u2")
    put(a["xcnt"][:N], "<u8")
    put(a["icnt"][:N], "<u8")
    for m in range(M):
        for nm in ["xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]:
            put(a[nm][m][:N], "<u8")
    put(a["xsamples"][:N] if S else np.zeros(N, np.uint64), "<u8")
    put(a["isamples"][:N] if S else np.zeros(N, np.uint64), "<u8")
    for s in range(S):
        put(a["xstall"][s][:N], "<u8")
        put(a["istall"][s][:N], "<u8")
    put(a["pc_ctx"][:Np], "<u4")
    put(a["pc_off"][:Np], "<u4")
    put(a["bin_pcnode"][:Nb], "<u4")
    put(a["bin_stall"][:Nb], "<u2")
    put(a["bin_count"][:Nb], "<u8")
    h.update(np.ascontiguousarray(k).tobytes())
    return h.hexdigest()


def leaf_digest(leaf) -> str:
    """SHA-256 of the records' canonical leaf ids (u32 little-endian, trace order)."""
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(np.asarray(leaf).astype("<u4", copy=False)).tobytes()).hexdigest()


def inverted(arrays: dict, metric=0) -> dict:
    """SURVEY §8(f) NEXT-3, the bottom-up (caller-inverted) tree ("switchable
    top-down and bottom-up views"; reading R27), plain Python over the oracle's
    canonical arrays, following the definition: every non-root node n with a non-zero exclusive
    value x(n) contributes x(n) to each prefix of its call path read innermost first (its frame,
    its caller's, ..., the outermost). Inverted nodes = the distinct such prefixes plus a root,
    numbered by (length, lexicographic frame ids) like the CCT itself (reading R2); per node the
    aggregate of the contributing values (count, sum, min, sum of squares); "x" columns: the
    nodes whose whole reversed path ends there. metric: index, or METRIC_SAMPLES."""
    parent, frame = arrays["parent"], arrays["frame"]
    x = arrays["xsamples"] if metric == METRIC_SAMPLES else arrays["xsum"][metric]
    inc, exc = {(): [0, 0, U64_MAX, 0]}, {}
    for n in range(1, int(arrays["n_nodes"])):
        v = int(x[n])
        if v == 0:
            continue
        rev, a = [], n
        while a != 0:
            rev.append(int(frame[a]))
            a = int(parent[a])
        for k in range(len(rev) + 1):
            agg = inc.setdefault(tuple(rev[:k]), [0, 0, U64_MAX, 0])
            agg[0] += 1
            agg[1] += v
            agg[2] = min(agg[2], v)
            agg[3] += v * v
        e = exc.setdefault(tuple(rev), [0, 0, U64_MAX, 0])
        e[0] += 1
        e[1] += v
        e[2] = min(e[2], v)
        e[3] += v * v
    keys = sorted(inc, key=lambda q: (len(q), q))
    ids = {q: i for i, q in enumerate(keys)}
    N = len(keys)
    out = dict(n_nodes=N, parent=np.zeros(N, np.uint32), frame=np.zeros(N, np.uint32), depth=np.zeros(N, np.uint16))
    for nm in ["xcnt", "icnt"]:
        out[nm] = np.zeros(N, np.uint64)
    for nm in ["xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]:
        out[nm] = np.zeros((1, N), np.uint64)
    M64 = (1 << 64) - 1
    for q, i in ids.items():
        out["parent"][i] = 0xFFFFFFFF if i == 0 else ids[q[:-1]]
        out["frame"][i] = 0xFFFFFFFF if i == 0 else q[-1]
        out["depth"][i] = len(q)
        c, s_, m, sq = inc[q]
        out["icnt"][i], out["isum"][0][i], out["imin"][0][i] = c, s_, m
        out["isq_lo"][0][i], out["isq_hi"][0][i] = sq & M64, sq >> 64
        c, s_, m, sq = exc.get(q, [0, 0, U64_MAX, 0])
        out["xcnt"][i], out["xsum"][0][i], out["xmin"][0][i] = c, s_, m
        out["xsq_lo"][0][i], out["xsq_hi"][0][i] = sq & M64, sq >> 64
    return out
