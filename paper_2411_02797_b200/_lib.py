"""ctypes binding of libdc.so (include/dc.h). Argument marshalling only: every step of the
path runs in the library's CUDA kernels. There is no CPU fallback: if the extension is
missing or no CUDA device is present, every call raises."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("DC_SO_OVERRIDE") or os.path.join(_HERE, "libdc.so")  # override: A/B builds only

P = ctypes.c_void_p
u8, u16, u32, u64, i32, f64 = ctypes.c_uint8, ctypes.c_uint16, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double

DC_OK, DC_ERR_ARG, DC_ERR_OOM, DC_ERR_CUDA, DC_ERR_NCCL, DC_ERR_CAPACITY, DC_ERR_TRACE, DC_ERR_COLLISION, DC_ERR_STATE = range(9)
STATUS_NAMES = ["DC_OK", "DC_ERR_ARG", "DC_ERR_OOM", "DC_ERR_CUDA", "DC_ERR_NCCL", "DC_ERR_CAPACITY", "DC_ERR_TRACE",
                "DC_ERR_COLLISION", "DC_ERR_STATE"]
DC_VIEW_INCLUSIVE, DC_VIEW_EXCLUSIVE, DC_VIEW_BOTTOM_UP, DC_VIEW_STALL = 0, 1, 2, 3
DC_METRIC_SAMPLES = 0xFFFFFFFF
DC_NO_NODE = 0xFFFFFFFF
DC_KIND_PY, DC_KIND_OP, DC_KIND_NATIVE, DC_KIND_API, DC_KIND_KERNEL, DC_KIND_INSTR = range(6)


class DcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


class dc_paths(ctypes.Structure):
    _fields_ = [("n_records", u64), ("offsets", P), ("frames", P)]


class dc_topk_entry(ctypes.Structure):
    _fields_ = [("id", u32), ("_pad", u32), ("value", u64), ("fraction", f64)]


class dc_rule_params(ctypes.Structure):
    _fields_ = [("metric_a", u32), ("metric_b", u32), ("kind_mask", u32), ("_pad", u32), ("threshold", f64), ("floor", u64)]


class dc_stall_issue(ctypes.Structure):
    _fields_ = [("node", u32), ("stall", u32), ("count", u64)]


class dc_diag(ctypes.Structure):
    _fields_ = [(n, u64) for n in ["empty_paths", "samples_bad_launch", "samples_bad_stall", "samples_zero_count",
                                   "collisions_detected", "levels_built", "max_depth_seen", "bytes_moved_est"]]


class dc_cct_view(ctypes.Structure):
    _fields_ = [("n_nodes", u64), ("n_pc_nodes", u64), ("n_bins", u64), ("n_records", u64), ("n_metrics", u32),
                ("n_stall", u32), ("max_depth", u32), ("n_frames", u32)] + \
               [(n, P) for n in ["parent", "frame", "depth", "level_off", "xcnt", "icnt", "xsum", "xmin", "xsq_lo", "xsq_hi",
                                 "isum", "imin", "isq_lo", "isq_hi", "xsamples", "isamples", "xstall", "istall", "pc_ctx",
                                 "pc_off", "bin_pcnode", "bin_stall", "bin_count"]] + [("state", i32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"libdc.so not built ({SO_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(SO_PATH)
        sig = {
            "dc_ctx_create": (i32, [i32, P, ctypes.POINTER(P)]),
            "dc_ctx_sync": (i32, [P]),
            "dc_ctx_diag": (i32, [P, ctypes.POINTER(dc_diag)]),
            "dc_ctx_destroy": (None, [P]),
            "dc_last_error": (ctypes.c_char_p, [P]),
            "dc_ctx_launch_count": (u64, [P]),
            "dc_ctx_set_timing": (i32, [P, i32]),
            "dc_ctx_reserve": (i32, [P, u64]),
            "dc_ctx_trim": (i32, [P, u64]),
            "dc_ctx_timer_report": (i32, [P, ctypes.c_char_p, ctypes.c_size_t]),
            "dc_intern_frames": (i32, [P, P, u64, P, ctypes.POINTER(P)]),
            "dc_dict_from_sorted": (i32, [P, P, u64, ctypes.POINTER(P)]),
            "dc_dict_size": (u64, [P]),
            "dc_dict_arrays": (i32, [P, ctypes.POINTER(P), ctypes.POINTER(P)]),
            "dc_dict_free": (None, [P]),
            "dc_cct_build": (i32, [P, ctypes.POINTER(dc_paths), P, u32, P, ctypes.POINTER(P)]),
            "dc_cct_attribute_metrics": (i32, [P, P, P, u64, P, u32, u64]),
            "dc_cct_rollup": (i32, [P, P]),
            "dc_pc_sample_attribute": (i32, [P, P, P, u64, P, u64, P, u32]),
            "dc_hotspots_topk": (i32, [P, P, i32, u32, u32, f64, u32, u32, P, ctypes.POINTER(u32)]),
            "dc_cct_derived": (i32, [P, P, u32, i32, P, P]),
            "dc_analyze_flags": (i32, [P, P, i32, ctypes.POINTER(dc_rule_params), P, u32, ctypes.POINTER(u32)]),
            "dc_analyze_stalls": (i32, [P, P, u32, u32, f64, f64, u32, P, u32, ctypes.POINTER(u32)]),
            "dc_cpu_intervals": (i32, [P, P, P, P, u64, P, P]),
            "dc_seq_associate": (i32, [P, P, P, P, u64, P, P, P, u64, P, P, u64, ctypes.POINTER(u64), ctypes.POINTER(u64)]),
            "dc_export_folded": (i32, [P, P, u32, P, P, P, P, u64, u64, ctypes.POINTER(u64), ctypes.POINTER(u64)]),
            "dc_cct_invert": (i32, [P, P, u32, ctypes.POINTER(P)]),
            "dc_cct_view_get": (i32, [P, ctypes.POINTER(dc_cct_view)]),
            "dc_cct_free": (None, [P]),
            "dc_nccl_unique_id": (i32, [P]),
            "dc_merge_plan": (i32, [u32, P, P, P, P, P]),
            "dc_comm_create": (i32, [P, P, i32, i32, ctypes.POINTER(P)]),
            "dc_comm_destroy": (None, [P]),
            "dc_cct_merge_ranks": (i32, [P, P, P, P, ctypes.POINTER(P), ctypes.POINTER(P)]),
            "dc_cct_gather": (i32, [P, P, P, i32, ctypes.POINTER(P)]),
            "dc_cct_merge_local": (i32, [P, u32, P, P, ctypes.POINTER(P), ctypes.POINTER(P)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Names the header declares (checked by the CPU test that the .so exports them)."""
    import re
    hdr = open(os.path.join(os.path.dirname(_HERE), "include", "dc.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)  # drop comments
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dc_[a-z_0-9]+)\s*\(", hdr, flags=re.M)))
