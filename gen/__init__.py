"""Seeded synthetic trace generator shared by the CPU oracle side and the CUDA side.

TEST/BENCH INPUT ONLY: holds none of the method's arithmetic. Program tables come from
gen/programs.py; bulk per-record draws run in gen/csrc (host loop or device kernel, same
gen_core.h source -> byte-identical traces). Arrays are returned as torch tensors (CPU or
CUDA) whose raw bytes match the C-ABI layouts of include/dc.h:
  keys     int32 [F, 4]    dc_frame_key {u32 kind, u32 str_id, u64 addr}
  ids      int32 [F]       u32 frame ids
  offsets  int64 [R+1]     u64 CSR offsets
  metrics  int64 [M, R]    u64, column-major (metric m is row m)
  samples  int32 [Ns, 4]   dc_pc_sample {u32 launch, u32 pc_off, u16 stall, u16 flags, u32 count}
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import torch

from . import programs
from .programs import Program  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdcgen.so")
_lib = None

NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(force: bool = False) -> str:
    src = [os.path.join(_HERE, "csrc", "dcgen.cu")]
    hdr = os.path.join(_HERE, "csrc", "gen_core.h")
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= max(os.path.getmtime(p) for p in src + [hdr]):
        return _SO
    cmd = ["nvcc", "-O3", "-std=c++17", *NVCC_ARCH, "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
           "-o", _SO + ".tmp", *src]
    subprocess.check_call(cmd)
    os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = ctypes.CDLL(_SO)
    return _lib


P = ctypes.c_void_p
u32, u64 = ctypes.c_uint32, ctypes.c_uint64


class GenProg(ctypes.Structure):
    _fields_ = [("seed", u64), ("mode", u32), ("n_sites", u32), ("site_off", P), ("site_frames", P),
                ("trunc_permille", u32), ("rec_permille", u32), ("max_depth", u32), ("empty_mod", u32),
                ("empty_rem", u32), ("force_record", u64), ("force_site", u32), ("site_rec_k", P),
                ("rec_pos", u32), ("rec_a", u32), ("rec_b", u32), ("dyn_per100k", u32), ("dyn_min", u32),
                ("dyn_max", u32), ("met_kind", u32), ("n_metrics", u32), ("site_base_ns", P),
                ("site_warps", P), ("site_smem", P)]


class GenPcProg(ctypes.Structure):
    _fields_ = [("seed", u64), ("n_launch", u32), ("n_sites", u32), ("launch_off", P), ("site_kernel", P),
                ("kern_off", P), ("pc_thr", P), ("pc_instr", P), ("stall_thr", P), ("stall_id", P),
                ("n_stall", u32), ("bad_per_million", u32)]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _t(a, device):
    if a is None:
        return None
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    elif a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a.copy()).to(device)


class Trace:
    """A generated trace; attributes are torch tensors (see module docstring)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def n_records(self):
        return int(self.offsets.numel() - 1)


def _prog_struct(p: Program, device, keep: list):
    def T(a):
        t = _t(a, device)
        if t is not None:
            keep.append(t)
        return _ptr(t)

    return GenProg(seed=p.seed, mode=p.mode, n_sites=len(p.site_off) - 1, site_off=T(p.site_off),
                   site_frames=T(p.site_frames), trunc_permille=p.trunc_permille, rec_permille=p.rec_permille,
                   max_depth=p.max_depth, empty_mod=p.empty_mod, empty_rem=p.empty_rem,
                   force_record=p.force_record, force_site=p.force_site, site_rec_k=T(p.site_rec_k),
                   rec_pos=p.rec_pos, rec_a=p.rec_a, rec_b=p.rec_b, dyn_per100k=p.dyn_per100k,
                   dyn_min=p.dyn_min, dyn_max=p.dyn_max, met_kind=p.met_kind, n_metrics=p.n_metrics,
                   site_base_ns=T(p.site_base_ns), site_warps=T(p.site_warps), site_smem=T(p.site_smem))


def _stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def make_trace(p: Program, n_records: int | None = None, device: str = "cpu", raw_keys: bool = True,
               ids: bool = True, pc: bool = False, bad_per_million: int = 0, n_launch: int | None = None) -> Trace:
    """Generate records [0, n_records) of program p (default: p.default_records).

    raw_keys -> Trace.keys (16-B raw frame keys, to be interned); ids -> Trace.ids (pool
    ranks, i.e. already-interned canonical ids over the pool dictionary)."""
    L = lib()
    dev = torch.device(device)
    R = int(n_records if n_records is not None else p.default_records)
    keep: list = []
    gp = _prog_struct(p, dev, keep)
    M = p.n_metrics
    if dev.type == "cpu":
        lens = np.zeros(R, np.uint32)
        L.dcgen_lengths_host(ctypes.byref(gp), u64(0), u64(R), lens.ctypes.data_as(P))
        off = np.zeros(R + 1, np.uint64)
        off[1:] = np.cumsum(lens, dtype=np.uint64)
        F = int(off[-1])
        ids_a = np.zeros(max(F, 1), np.uint32) if ids else None
        keys_a = np.zeros((max(F, 1), 4), np.int32) if raw_keys else None
        pool = np.ascontiguousarray(p.pool_keys)
        L.dcgen_frames_host(ctypes.byref(gp), u64(0), u64(R), off.ctypes.data_as(P), pool.ctypes.data_as(P),
                            ids_a.ctypes.data_as(P) if ids else None, keys_a.ctypes.data_as(P) if raw_keys else None)
        met = np.zeros((M, max(R, 1)), np.uint64)
        L.dcgen_metrics_host(ctypes.byref(gp), u64(0), u64(R), met.ctypes.data_as(P), u64(max(R, 1)))
        tr = Trace(program=p, offsets=torch.from_numpy(off.view(np.int64)),
                   ids=torch.from_numpy(ids_a[:F].view(np.int32)) if ids else None,
                   keys=torch.from_numpy(keys_a[:F]) if raw_keys else None,
                   metrics=torch.from_numpy(met[:, :R].view(np.int64).copy()))
    else:
        s = _stream_ptr(dev)
        lens = torch.empty(max(R, 1), dtype=torch.int32, device=dev)
        assert L.dcgen_lengths_dev(ctypes.byref(gp), u64(0), u64(R), _ptr(lens), s) == 0
        off = torch.zeros(R + 1, dtype=torch.int64, device=dev)
        off[1:] = torch.cumsum(lens[:R].to(torch.int64), 0)
        F = int(off[-1].item())
        ids_t = torch.empty(max(F, 1), dtype=torch.int32, device=dev) if ids else None
        keys_t = torch.empty((max(F, 1), 4), dtype=torch.int32, device=dev) if raw_keys else None
        pool_t = torch.from_numpy(np.ascontiguousarray(p.pool_keys).view(np.int32).reshape(-1, 4).copy()).to(dev)
        assert L.dcgen_frames_dev(ctypes.byref(gp), u64(0), u64(R), _ptr(off), _ptr(pool_t), _ptr(ids_t),
                                  _ptr(keys_t), s) == 0
        met = torch.empty((M, max(R, 1)), dtype=torch.int64, device=dev)
        assert L.dcgen_metrics_dev(ctypes.byref(gp), u64(0), u64(R), _ptr(met), u64(max(R, 1)), s) == 0
        tr = Trace(program=p, offsets=off, ids=ids_t[:F] if ids else None, keys=keys_t[:F] if raw_keys else None,
                   metrics=met[:, :R].contiguous())
    tr.n_frames = len(p.pool_keys)
    tr.kinds = torch.from_numpy(np.asarray(p.pool_keys["kind"], np.uint8).copy())
    if pc:
        q = p.pc
        nl = int(n_launch if n_launch is not None else q["n_launch"])
        assert nl <= q["n_launch"]
        launch_off = q["launch_off"][: nl + 1]
        ns = int(launch_off[-1])
        pp = GenPcProg(seed=p.seed, n_launch=nl, n_sites=q["n_sites"], launch_off=None,
                       n_stall=q["n_stall"], bad_per_million=bad_per_million)
        tabs = {k: _t(q[k], dev) for k in ["site_kernel", "kern_off", "pc_thr", "pc_instr", "stall_thr"]}
        tabs["stall_id"] = torch.from_numpy(np.asarray(q["stall_id"], np.uint8).copy()).to(dev)
        tabs["launch_off"] = _t(launch_off, dev)
        for k, v in tabs.items():
            setattr(pp, k, _ptr(v))
        samples = torch.empty((max(ns, 1), 4), dtype=torch.int32, device=dev)
        if dev.type == "cpu":
            L.dcgen_pc_host(ctypes.byref(pp), u32(0), u32(nl), _ptr(samples))
        else:
            assert L.dcgen_pc_dev(ctypes.byref(pp), u32(0), u32(nl), _ptr(samples), _stream_ptr(dev)) == 0
        tr.samples = samples[:ns]
        tr.launch_off = tabs["launch_off"]
        tr.n_launch = nl
        tr.n_stall = q["n_stall"]
        keep.append(tabs)
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()
    tr._keep = keep
    return tr


def make_chunk_host(p: Program, r0: int, n: int, raw_keys: bool = True, ids: bool = False):
    """Records [r0, r0 + n) of program p on the host, as numpy arrays (offsets relative to the
    chunk, starting at 0): (offsets u64 [n+1], ids u32 [F] or None, keys KEY-layout u8 [F, 16]
    or None, metrics u64 [M, n]). Records are generated independently (counter-based), so the
    concatenation of consecutive chunks is byte-identical to make_trace over [0, r0 + n) from r0
    on — used to stream traces too large for host memory through the CPU oracle."""
    L = lib()
    keep: list = []
    gp = _prog_struct(p, torch.device("cpu"), keep)
    lens = np.zeros(max(n, 1), np.uint32)
    L.dcgen_lengths_host(ctypes.byref(gp), u64(r0), u64(n), lens.ctypes.data_as(P))
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens[:n], dtype=np.uint64)
    F = int(off[-1])
    ids_a = np.zeros(max(F, 1), np.uint32) if ids else None
    keys_a = np.zeros((max(F, 1), 16), np.uint8) if raw_keys else None
    pool = np.ascontiguousarray(p.pool_keys)
    L.dcgen_frames_host(ctypes.byref(gp), u64(r0), u64(n), off.ctypes.data_as(P), pool.ctypes.data_as(P),
                        ids_a.ctypes.data_as(P) if ids else None, keys_a.ctypes.data_as(P) if raw_keys else None)
    met = np.zeros((p.n_metrics, max(n, 1)), np.uint64)
    L.dcgen_metrics_host(ctypes.byref(gp), u64(r0), u64(n), met.ctypes.data_as(P), u64(max(n, 1)))
    return off, (ids_a[:F] if ids else None), (keys_a[:F] if raw_keys else None), np.ascontiguousarray(met[:, :n])


def generator_version() -> str:
    """SHA-256 (first 16 hex digits) of the generator's sources: cached oracle results
    (tests/golden/digest_*.json) are keyed by it and go stale when the generator changes."""
    import hashlib
    h = hashlib.sha256()
    for f in ["csrc/gen_core.h", "csrc/dcgen.cu", "programs.py", "rng.py"]:
        with open(os.path.join(_HERE, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]
