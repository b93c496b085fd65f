"""paper_2411_02797_b200 — B200-native calling-context-tree aggregation (arXiv 2411.02797).

Thin Python binding of libdc.so with the C ABI's names (include/dc.h). Tensors are torch
CUDA tensors (device memory + streams only); every computation runs in libdc's kernels.
No CPU fallback: without the built library or a CUDA device every call raises.

    ctx = Context(0)
    ids, d = dc_intern_frames(ctx, keys)                    # keys: int32 [F, 4] CUDA
    cct, leaf = dc_cct_build(ctx, offsets, ids, d.size, d)  # offsets int64 [R+1], ids int32 [F]
    dc_cct_attribute_metrics(ctx, cct, leaf, metrics)       # metrics int64 [M, R]
    dc_pc_sample_attribute(ctx, cct, samples, leaf, launch_off, n_stall=24)
    dc_cct_rollup(ctx, cct)
    top = dc_hotspots_topk(ctx, cct, DC_VIEW_INCLUSIVE, metric=0, kind_mask=1 << DC_KIND_KERNEL, threshold=0.1, k=5)
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

from ._lib import (DC_KIND_API, DC_KIND_INSTR, DC_KIND_KERNEL, DC_KIND_NATIVE, DC_KIND_OP, DC_KIND_PY,  # noqa: F401
                   DC_METRIC_SAMPLES, DC_NO_NODE, DC_VIEW_BOTTOM_UP, DC_VIEW_EXCLUSIVE, DC_VIEW_INCLUSIVE, DC_VIEW_STALL,
                   DcError, dc_cct_view, dc_diag, dc_paths, dc_topk_entry, lib)

__all__ = ["Context", "Dict", "CCT", "dc_intern_frames", "dc_dict_from_sorted", "dc_cct_build", "dc_cct_attribute_metrics",
           "dc_cct_rollup", "dc_pc_sample_attribute", "dc_hotspots_topk", "dc_cct_derived", "dc_cct_view_get",
           "dc_cct_merge_ranks", "dc_nccl_unique_id", "dc_comm_create", "DcError"]


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libdc takes CUDA tensors (device memory); got a CPU tensor")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """dc_ctx: one device + one stream (default: torch's current stream on that device)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2411_02797_b200 needs a CUDA device (no CPU fallback)")
        self.device = int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        st = lib().dc_ctx_create(self.device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if st != 0:
            raise DcError(st, "dc_ctx_create failed")
        self.h = h

    def check(self, st: int, what: str):
        if st != 0:
            raise DcError(st, f"{what}: {lib().dc_last_error(self.h).decode(errors='replace')}")

    def sync(self):
        self.check(lib().dc_ctx_sync(self.h), "dc_ctx_sync")

    def diag(self) -> dict:
        d = dc_diag()
        self.check(lib().dc_ctx_diag(self.h, ctypes.byref(d)), "dc_ctx_diag")
        return {n: int(getattr(d, n)) for n, _ in dc_diag._fields_}

    @property
    def launches(self) -> int:
        return int(lib().dc_ctx_launch_count(self.h))

    def reserve(self, nbytes: int):
        """Grow the stream-ordered pool to at least nbytes (dc_ctx_reserve)."""
        self.check(lib().dc_ctx_reserve(self.h, int(nbytes)), "dc_ctx_reserve")

    def trim(self, keep_bytes: int = 0):
        """Return the context pool's cached free memory to the device (dc_ctx_trim)."""
        self.check(lib().dc_ctx_trim(self.h, int(keep_bytes)), "dc_ctx_trim")

    def set_timing(self, on: bool):
        self.check(lib().dc_ctx_set_timing(self.h, int(bool(on))), "dc_ctx_set_timing")

    def timer_report(self) -> dict:
        """{name: (count, total_ms)} since the last report (synchronizes)."""
        buf = ctypes.create_string_buffer(1 << 16)
        self.check(lib().dc_ctx_timer_report(self.h, buf, len(buf)), "dc_ctx_timer_report")
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split()
            out[name] = (int(cnt), float(ms))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().dc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Dict:
    def __init__(self, h):
        self.h = h

    @property
    def size(self) -> int:
        return int(lib().dc_dict_size(self.h))

    def kinds(self) -> np.ndarray:
        k = ctypes.c_void_p()
        kd = ctypes.c_void_p()
        lib().dc_dict_arrays(self.h, ctypes.byref(k), ctypes.byref(kd))
        return _dev_to_numpy(kd.value, (self.size,), np.uint8)

    def keys(self) -> np.ndarray:
        k = ctypes.c_void_p()
        lib().dc_dict_arrays(self.h, ctypes.byref(k), None)
        raw = _dev_to_numpy(k.value, (self.size * 16,), np.uint8)
        return raw.view(np.dtype([("kind", "<u4"), ("str_id", "<u4"), ("addr", "<u8")]))

    def __del__(self):
        if getattr(self, "h", None):
            lib().dc_dict_free(self.h)
            self.h = None


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr, "version": 3}


def _dev_to_numpy(ptr, shape, dtype) -> np.ndarray:
    dtype = np.dtype(dtype)
    n = int(np.prod(shape))
    if n == 0 or not ptr:
        return np.zeros(shape, dtype)
    signed = {1: "|u1", 2: "<i2", 4: "<i4", 8: "<i8"}[dtype.itemsize]
    t = torch.as_tensor(_CAI(ptr, (n,), signed), device="cuda")
    return t.cpu().numpy().view(dtype).reshape(shape)


class CCT:
    """dc_cct handle."""

    def __init__(self, h, ctx: Context):
        self.h = h
        self.ctx = ctx

    def view(self, before_rollup: bool = False) -> dc_cct_view:
        """dc_cct_view_get. Before dc_cct_rollup the call reports DC_ERR_STATE (inclusive
        columns NULL); before_rollup=True accepts that and returns the partial view."""
        v = dc_cct_view()
        st = lib().dc_cct_view_get(self.h, ctypes.byref(v))
        if st and not (before_rollup and st == _lib.DC_ERR_STATE):
            raise DcError(st, "dc_cct_view_get")
        return v

    def to_numpy(self) -> dict:
        """Host copies of every view array (names as in the oracle's arrays())."""
        self.ctx.sync()
        v = self.view(before_rollup=True)
        N, Np, Nb, M, S = v.n_nodes, v.n_pc_nodes, v.n_bins, v.n_metrics, v.n_stall
        a = dict(n_nodes=N, n_pc_nodes=Np, n_bins=Nb, n_metrics=M, n_stall=S, max_depth=v.max_depth, state=v.state)
        a["parent"] = _dev_to_numpy(v.parent, (N,), np.uint32)
        a["frame"] = _dev_to_numpy(v.frame, (N,), np.uint32)
        a["depth"] = _dev_to_numpy(v.depth, (N,), np.uint16)
        a["level_off"] = _dev_to_numpy(v.level_off, (v.max_depth + 2,), np.uint32)
        rolled = v.state == 2  # inclusive columns exist only after dc_cct_rollup (None before)
        a["xcnt"] = _dev_to_numpy(v.xcnt, (N,), np.uint64)
        a["icnt"] = _dev_to_numpy(v.icnt, (N,), np.uint64) if rolled else None
        for nm in ["xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]:
            a[nm] = _dev_to_numpy(getattr(v, nm), (M, N), np.uint64) if rolled or nm[0] == "x" else None
        a["xsamples"] = _dev_to_numpy(v.xsamples, (N,), np.uint64) if v.xsamples else np.zeros(N, np.uint64)
        a["isamples"] = (_dev_to_numpy(v.isamples, (N,), np.uint64) if v.isamples else np.zeros(N, np.uint64)) if rolled else None
        a["xstall"] = _dev_to_numpy(v.xstall, (S, N), np.uint64)
        a["istall"] = _dev_to_numpy(v.istall, (S, N), np.uint64) if rolled else None
        a["pc_ctx"] = _dev_to_numpy(v.pc_ctx, (Np,), np.uint32)
        a["pc_off"] = _dev_to_numpy(v.pc_off, (Np,), np.uint32)
        a["bin_pcnode"] = _dev_to_numpy(v.bin_pcnode, (Nb,), np.uint32)
        a["bin_stall"] = _dev_to_numpy(v.bin_stall, (Nb,), np.uint16)
        a["bin_count"] = _dev_to_numpy(v.bin_count, (Nb,), np.uint64)
        return a

    def digest(self, d: "Dict | None") -> str:
        """SHA-256 of the canonical little-endian serialisation of this (rolled-up) tree and its
        dictionary (SURVEY.md §8(c) "Digest"): b"DCCCT1\\0\\0", u64 N, M, S, Npc, Nbins, D, then
        parent, frame, depth (u16), xcnt, icnt, per metric the 8 columns xsum, xmin, xsq_lo,
        xsq_hi, isum, imin, isq_lo, isq_hi, xsamples, isamples, per stall xstall / istall, pc_ctx,
        pc_off, bin_pcnode, bin_stall (u16), bin_count, the dictionary's 16-B keys. Host-side
        formatting of the view's arrays only (for comparing results across runs / with a cached
        reference digest)."""
        import hashlib
        import struct
        a = self.to_numpy()
        N, M, S, Np, Nb = (int(a[k]) for k in ["n_nodes", "n_metrics", "n_stall", "n_pc_nodes", "n_bins"])
        keys = d.keys() if d is not None and d.size else np.zeros(0, np.dtype([("kind", "<u4"), ("str_id", "<u4"), ("addr", "<u8")]))
        h = hashlib.sha256(b"DCCCT1\0\0" + struct.pack("<6Q", N, M, S, Np, Nb, len(keys)))
        cols = [("parent", "<u4"), ("frame", "<u4"), ("depth", "<u2"), ("xcnt", "<u8"), ("icnt", "<u8")]
        for name, dt in cols:
            h.update(np.ascontiguousarray(a[name], dtype=dt).tobytes())
        for m in range(M):
            for name in ["xsum", "xmin", "xsq_lo", "xsq_hi", "isum", "imin", "isq_lo", "isq_hi"]:
                h.update(np.ascontiguousarray(a[name][m], dtype="<u8").tobytes())
        h.update(np.ascontiguousarray(a["xsamples"], dtype="<u8").tobytes())
        h.update(np.ascontiguousarray(a["isamples"], dtype="<u8").tobytes())
        for s in range(S):
            h.update(np.ascontiguousarray(a["xstall"][s], dtype="<u8").tobytes())
            h.update(np.ascontiguousarray(a["istall"][s], dtype="<u8").tobytes())
        for name, dt in [("pc_ctx", "<u4"), ("pc_off", "<u4"), ("bin_pcnode", "<u4"), ("bin_stall", "<u2"),
                         ("bin_count", "<u8")]:
            h.update(np.ascontiguousarray(a[name], dtype=dt).tobytes())
        h.update(np.ascontiguousarray(keys).tobytes())
        return h.hexdigest()

    @property
    def n_nodes(self) -> int:
        # fixed for the handle's lifetime (set by the call that created it): read once
        n = getattr(self, "_n_nodes", None)
        if n is None:
            n = self._n_nodes = int(self.view(before_rollup=True).n_nodes)
        return n

    def free(self):
        if getattr(self, "h", None):
            lib().dc_cct_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ------------------------------------------------------------------ C-ABI names
def dc_intern_frames(ctx: Context, keys: torch.Tensor, out_ids: torch.Tensor | None = None):
    """keys: CUDA int32 [n, 4] (dc_frame_key). Returns (ids int32 [n], Dict)."""
    n = keys.shape[0] if keys.numel() else 0
    if out_ids is None:
        out_ids = torch.empty(max(n, 1), dtype=torch.int32, device=keys.device)
    d = ctypes.c_void_p()
    ctx.check(lib().dc_intern_frames(ctx.h, _ptr(keys) if n else None, n, _ptr(out_ids) if n else None, ctypes.byref(d)),
              "dc_intern_frames")
    return (out_ids if out_ids.numel() == n else out_ids[:n]), Dict(d)


def dc_dict_from_sorted(ctx: Context, keys: torch.Tensor) -> Dict:
    d = ctypes.c_void_p()
    D = keys.shape[0] if keys.numel() else 0
    ctx.check(lib().dc_dict_from_sorted(ctx.h, _ptr(keys) if D else None, D, ctypes.byref(d)), "dc_dict_from_sorted")
    return Dict(d)


def dc_cct_build(ctx: Context, offsets: torch.Tensor, frames: torch.Tensor, n_frames: int, dict: Dict | None = None,
                 want_leaf: bool = True, out_leaf: torch.Tensor | None = None):
    R = offsets.numel() - 1
    if want_leaf and out_leaf is None:
        out_leaf = torch.empty(max(R, 1), dtype=torch.int32, device=offsets.device)
    p = dc_paths(n_records=R, offsets=_ptr(offsets), frames=_ptr(frames) if frames.numel() else None)
    h = ctypes.c_void_p()
    ctx.check(lib().dc_cct_build(ctx.h, ctypes.byref(p), dict.h if dict is not None else None, int(n_frames),
                                 _ptr(out_leaf) if want_leaf else None, ctypes.byref(h)), "dc_cct_build")
    return CCT(h, ctx), ((out_leaf if out_leaf.numel() == R else out_leaf[:R]) if want_leaf else None)


def dc_cct_attribute_metrics(ctx: Context, cct: CCT, leaf: torch.Tensor, metrics: torch.Tensor):
    """metrics: CUDA int64 [M, R] (u64 values, column-major as in dc.h)."""
    M, R = metrics.shape
    ctx.check(lib().dc_cct_attribute_metrics(ctx.h, cct.h, _ptr(leaf) if R else None, R, _ptr(metrics) if R else None, M,
                                             metrics.stride(0) if R else 0), "dc_cct_attribute_metrics")


def dc_cct_rollup(ctx: Context, cct: CCT):
    ctx.check(lib().dc_cct_rollup(ctx.h, cct.h), "dc_cct_rollup")


def dc_pc_sample_attribute(ctx: Context, cct: CCT, samples: torch.Tensor, launch_leaf: torch.Tensor,
                           launch_off: torch.Tensor | None = None, n_stall: int = 24, n_launch: int | None = None):
    """samples: CUDA int32 [n, 4] (dc_pc_sample); launch_leaf int32 [n_launch]; launch_off int64 [n_launch+1] or None."""
    n = samples.shape[0] if samples.numel() else 0
    nl = int(n_launch if n_launch is not None else launch_leaf.numel())
    ctx.check(lib().dc_pc_sample_attribute(ctx.h, cct.h, _ptr(samples) if n else None, n, _ptr(launch_leaf) if nl else None,
                                           nl, _ptr(launch_off), int(n_stall)), "dc_pc_sample_attribute")


def dc_hotspots_topk(ctx: Context, cct: CCT, view: int, metric: int = 0, kind_mask: int = 0xFFFFFFFF,
                     threshold: float = 0.0, k: int = 10, stall_node: int = 0) -> list[tuple[int, int, float]]:
    out = (dc_topk_entry * max(k, 1))()
    n = ctypes.c_uint32(0)
    ctx.check(lib().dc_hotspots_topk(ctx.h, cct.h, int(view), metric & 0xFFFFFFFF, kind_mask & 0xFFFFFFFF, float(threshold),
                                     int(k), int(stall_node), ctypes.cast(out, ctypes.c_void_p), ctypes.byref(n)),
              "dc_hotspots_topk")
    return [(int(out[i].id), int(out[i].value), float(out[i].fraction)) for i in range(n.value)]


DC_RULE_BWD_FWD = 3
DC_RULE_SMALL_KERNELS = 2
DC_RULE_CPU_LATENCY = 5


def dc_analyze_flags(ctx: Context, cct: CCT, rule: int, metric_a: int, metric_b: int = 0, kind_mask: int = 0xFFFFFFFF,
                     threshold: float = 0.0, floor: int = 0, cap: int = 1 << 16) -> list[int]:
    """Analyzer rules ② (small kernels) / ⑤ (CPU latency) as device predicates: flagged node ids,
    breadth-first order (include/dc.h dc_analyze_flags)."""
    prm = _lib.dc_rule_params(metric_a=metric_a, metric_b=metric_b, kind_mask=kind_mask & 0xFFFFFFFF,
                              threshold=float(threshold), floor=int(floor))
    out = (ctypes.c_uint32 * max(cap, 1))()
    n = ctypes.c_uint32(0)
    ctx.check(lib().dc_analyze_flags(ctx.h, cct.h, int(rule), ctypes.byref(prm), ctypes.cast(out, ctypes.c_void_p), int(cap),
                                     ctypes.byref(n)), "dc_analyze_flags")
    return [int(out[i]) for i in range(min(n.value, cap))]


def dc_analyze_stalls(ctx: Context, cct: CCT, metric: int = 0, kind_mask: int = 0xFFFFFFFF, hot_threshold: float = 0.0,
                      stall_threshold: float = 0.0, k: int = 3, cap: int = 1 << 16) -> list[tuple[int, int, int]]:
    """Analysis ④: (hotspot node, stall reason, count) entries (include/dc.h dc_analyze_stalls)."""
    out = (_lib.dc_stall_issue * max(cap, 1))()
    n = ctypes.c_uint32(0)
    ctx.check(lib().dc_analyze_stalls(ctx.h, cct.h, int(metric), kind_mask & 0xFFFFFFFF, float(hot_threshold),
                                      float(stall_threshold), int(k), ctypes.cast(out, ctypes.c_void_p), int(cap),
                                      ctypes.byref(n)), "dc_analyze_stalls")
    return [(int(out[i].node), int(out[i].stall), int(out[i].count)) for i in range(min(n.value, cap))]


def dc_cpu_intervals(ctx: Context, thread: torch.Tensor, kind: torch.Tensor, ts: torch.Tensor):
    """NEXT-4 CPU-sample intervals (include/dc.h dc_cpu_intervals): (interval u64 as int64 tensor,
    valid u8 tensor), trace order. thread int32, kind uint8, ts int64 (device tensors)."""
    n = int(ts.numel())
    iv = torch.empty(max(n, 1), dtype=torch.int64, device=ts.device)
    ok = torch.empty(max(n, 1), dtype=torch.uint8, device=ts.device)
    ctx.check(lib().dc_cpu_intervals(ctx.h, _ptr(thread) if n else None, _ptr(kind) if n else None, _ptr(ts) if n else None, n,
                                     _ptr(iv), _ptr(ok)), "dc_cpu_intervals")
    return iv[:n], ok[:n]


def dc_seq_associate(ctx: Context, fwd_seq: torch.Tensor, fwd_off: torch.Tensor, fwd_frames: torch.Tensor,
                     bwd_seq: torch.Tensor, bwd_off: torch.Tensor, bwd_frames: torch.Tensor):
    """NEXT-4 forward/backward association (include/dc.h dc_seq_associate): integrated backward
    paths as (offsets int64 [nb+1], frames int32) device tensors, and the unmatched count."""
    nf, nb = int(fwd_seq.numel()), int(bwd_seq.numel())
    out_off = torch.empty(nb + 1, dtype=torch.int64, device=bwd_off.device)
    nfr, nun = ctypes.c_uint64(0), ctypes.c_uint64(0)
    q = lambda t: _ptr(t) if t.numel() else None  # noqa: E731
    args = (ctx.h, q(fwd_seq), q(fwd_off), q(fwd_frames), nf, q(bwd_seq), q(bwd_off), q(bwd_frames), nb, _ptr(out_off))
    ctx.check(lib().dc_seq_associate(*args, None, 0, ctypes.byref(nfr), ctypes.byref(nun)), "dc_seq_associate")
    out = torch.empty(max(nfr.value, 1), dtype=torch.int32, device=bwd_off.device)
    ctx.check(lib().dc_seq_associate(*args, _ptr(out), nfr.value, ctypes.byref(nfr), ctypes.byref(nun)), "dc_seq_associate")
    return out_off, out[: nfr.value], int(nun.value)


def dc_export_folded(ctx: Context, cct: CCT, metric: int = 0):
    """Folded flame-graph stacks as arrays: (node ids, exclusive values, list of frame-id paths)
    (include/dc.h dc_export_folded)."""
    nl, nf = ctypes.c_uint64(0), ctypes.c_uint64(0)
    ctx.check(lib().dc_export_folded(ctx.h, cct.h, int(metric), None, None, None, None, 0, 0, ctypes.byref(nl),
                                     ctypes.byref(nf)), "dc_export_folded")
    L, F = nl.value, nf.value
    nodes, vals, offs = np.zeros(max(L, 1), np.uint32), np.zeros(max(L, 1), np.uint64), np.zeros(max(L, 1), np.uint64)
    frames = np.zeros(max(F, 1), np.uint32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    ctx.check(lib().dc_export_folded(ctx.h, cct.h, int(metric), p(nodes), p(vals), p(offs), p(frames), L, F, ctypes.byref(nl),
                                     ctypes.byref(nf)), "dc_export_folded")
    ends = list(offs[1:L].tolist()) + [F]
    paths = [frames[int(o):int(e)].tolist() for o, e in zip(offs[:L].tolist(), ends)]
    return nodes[:L].tolist(), vals[:L].tolist(), paths


def dc_cct_invert(ctx: Context, cct: CCT, metric: int = 0) -> CCT:
    """Bottom-up (caller-inverted) tree of the exclusive values of `metric` (include/dc.h
    dc_cct_invert): roots = frames where the cost is spent, children = their callers. Returns a
    new rolled-up CCT whose metric 0 aggregates the contributing nodes' values."""
    h = ctypes.c_void_p()
    ctx.check(lib().dc_cct_invert(ctx.h, cct.h, metric & 0xFFFFFFFF, ctypes.byref(h)), "dc_cct_invert")
    return CCT(h, ctx)


def folded_text(ctx: Context, cct: CCT, labels, metric: int = 0) -> str:
    """SPEC.md export_folded text: frames joined by ';' (';' inside labels replaced by ','), one
    space, the integer exclusive value; LF line endings. labels[frame id] -> str."""
    _, vals, paths = dc_export_folded(ctx, cct, metric)
    return "".join(";".join(str(labels[f]).replace(";", ",") for f in path) + f" {v}\n" for path, v in zip(paths, vals))


def dc_cct_derived(ctx: Context, cct: CCT, metric: int, incl: bool = True, out: tuple | None = None):
    """mean / population std per node (float64 [N] CUDA). out: optional (mean, std) float64 CUDA
    tensors of at least N elements, written in place (no allocation per call)."""
    N = cct.n_nodes
    if out is not None and out[0].numel() >= N and out[1].numel() >= N:
        mean, std = out
    else:
        mean = torch.empty(max(N, 1), dtype=torch.float64, device=f"cuda:{ctx.device}")
        std = torch.empty_like(mean)
    ctx.check(lib().dc_cct_derived(ctx.h, cct.h, int(metric), int(bool(incl)), _ptr(mean), _ptr(std)), "dc_cct_derived")
    return (mean, std) if mean.numel() == N else (mean[:N], std[:N])


def dc_cct_view_get(cct: CCT) -> dc_cct_view:
    return cct.view()


def dc_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    st = lib().dc_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if st:
        raise DcError(st, "dc_nccl_unique_id")
    return bytes(buf)


class Comm:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().dc_comm_destroy(self.h)
            self.h = None


def dc_comm_create(ctx: Context, uid: bytes, nranks: int, rank: int) -> Comm:
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    ctx.check(lib().dc_comm_create(ctx.h, ctypes.cast(buf, ctypes.c_void_p), int(nranks), int(rank), ctypes.byref(h)),
              "dc_comm_create")
    return Comm(h)


def dc_cct_merge_ranks(ctx: Context, comm: Comm, local: CCT, local_dict: Dict):
    part = ctypes.c_void_p()
    gd = ctypes.c_void_p()
    ctx.check(lib().dc_cct_merge_ranks(ctx.h, comm.h, local.h, local_dict.h, ctypes.byref(part), ctypes.byref(gd)),
              "dc_cct_merge_ranks")
    return CCT(part, ctx), Dict(gd)


def dc_cct_merge_local(ctx: Context, locals_: list, dicts: list):
    """Single-GPU emulation of merge_ranks + gather over len(locals_) logical ranks."""
    P = len(locals_)
    la = (ctypes.c_void_p * P)(*[t.h.value if isinstance(t.h, ctypes.c_void_p) else t.h for t in locals_])
    da = (ctypes.c_void_p * P)(*[d.h.value if isinstance(d.h, ctypes.c_void_p) else d.h for d in dicts])
    out = ctypes.c_void_p()
    gd = ctypes.c_void_p()
    ctx.check(lib().dc_cct_merge_local(ctx.h, P, ctypes.cast(la, ctypes.c_void_p), ctypes.cast(da, ctypes.c_void_p),
                                       ctypes.byref(out), ctypes.byref(gd)), "dc_cct_merge_local")
    return CCT(out, ctx), Dict(gd)


def aggregate_chunks(ctx: Context, chunks):
    """SURVEY §8(f) NEXT-1, chunked / online aggregation: fold an iterable of (rolled-up CCT,
    dictionary) pairs — each built from one chunk of the trace with the dc_* calls — into one
    canonical CCT with dc_cct_merge_local (the cross-rank merge's partition / reduce / verify /
    canonicalise kernels with a loopback exchange). The result equals the CCT of the
    concatenated chunks (reading R19); inputs are freed as they are folded."""
    acc = accd = None
    for cct, d in chunks:
        if acc is None:
            acc, accd = cct, d
            continue
        merged, md = dc_cct_merge_local(ctx, [acc, cct], [accd, d])
        acc.free()
        cct.free()
        acc, accd = merged, md
    return acc, accd


def dc_cct_gather(ctx: Context, comm: Comm, part: CCT, root: int = 0):
    h = ctypes.c_void_p()
    ctx.check(lib().dc_cct_gather(ctx.h, comm.h, part.h, int(root), ctypes.byref(h)), "dc_cct_gather")
    return CCT(h, ctx) if h.value else None
