"""Config 3s — the stress variant of config 3 (SURVEY.md §8(d) cfg 3: "20,000 distinct contexts
with samples of 8 concurrent launches interleaved ... exercises the fallback schedule").

TEST/BENCH INPUT ONLY (no method arithmetic): a pure re-arrangement of a generated config-3
trace, done with torch ops on whatever device the trace lives on (so the host copy fed to the
oracle and the device copy fed to the CUDA path are identical):
  * every launch record's call path gets one extra outermost frame unique to that launch (a
    Python frame `stress.py:<launch>`, kind PY), so the 20,000 launches are 20,000 distinct
    contexts;
  * the PC samples of each group of 8 consecutive launches are interleaved round robin (sample i
    of launch 8g + k lands after sample i of launch 8g + k - 1), as 8 concurrent kernels'
    samples arrive in one buffer: samples are no longer contiguous per launch, so no per-launch
    offsets exist and the generic (any-order) schedule runs.
"""
from __future__ import annotations

import torch

STRESS_STR = 0x7FFF0000  # string id range of the per-launch frames (disjoint from the program's)


def make_3s(tr, group: int = 8):
    dev = tr.offsets.device
    R = tr.n_records
    off = tr.offsets
    lens = off[1:] - off[:-1]
    new_lens = lens + 1
    new_off = torch.zeros(R + 1, dtype=torch.int64, device=dev)
    new_off[1:] = torch.cumsum(new_lens, 0)
    F = int(off[-1].item())
    keys = torch.empty((F + R, 4), dtype=torch.int32, device=dev)
    # the unique outermost frame of record r: (kind 0 = PY, str_id = STRESS_STR + r, addr = r)
    r = torch.arange(R, dtype=torch.int64, device=dev)
    uk = torch.zeros((R, 4), dtype=torch.int32, device=dev)
    uk[:, 1] = (STRESS_STR + r).to(torch.int32)
    uk[:, 2] = r.to(torch.int32)  # addr low word (high word 0)
    keys[new_off[:-1]] = uk
    # the original frames shift by their record index + 1
    rec_of = torch.repeat_interleave(r, lens)
    keys[torch.arange(F, device=dev) + rec_of + 1] = tr.keys
    # samples: round robin over each group of `group` launches
    lo = tr.launch_off
    cnt = lo[1:] - lo[:-1]
    s_launch = torch.repeat_interleave(torch.arange(tr.n_launch, dtype=torch.int64, device=dev), cnt)
    idx_in = torch.arange(int(lo[-1].item()), dtype=torch.int64, device=dev) - lo[:-1][s_launch]
    key = ((s_launch // group) << 40) | (idx_in << 8) | (s_launch % group)
    perm = torch.argsort(key, stable=True)
    out = type(tr)(**{k: v for k, v in tr.__dict__.items()})
    out.offsets = new_off
    out.keys = keys
    out.samples = tr.samples[perm].contiguous()
    out.launch_off = None
    out.ids = None
    return out


def make_aggregated(tr):
    """Config 3 with per-PC aggregated records, as CUPTI's PC-sampling API delivers them: per
    launch, one record per distinct (pc_off, stall) with the number of raw samples as its count
    (records stay contiguous per launch, in (pc, stall) order). Same bins as the raw trace."""
    dev = tr.samples.device
    s = tr.samples.to(torch.int64)
    launch, pc, stall = s[:, 0] & 0xFFFFFFFF, s[:, 1] & 0xFFFFFFFF, s[:, 2] & 0xFFFF
    key = (launch << 37) | (pc << 5) | stall  # launch < 2^26, pc_off < 2^32, stall < 32
    uk, cnt = torch.unique(key, sorted=True, return_counts=True)
    out = torch.zeros((uk.numel(), 4), dtype=torch.int64, device=dev)
    out[:, 0] = uk >> 37
    out[:, 1] = (uk >> 5) & 0xFFFFFFFF
    out[:, 2] = uk & 31
    out[:, 3] = cnt
    per_launch = torch.bincount(out[:, 0], minlength=tr.n_launch)
    lo = torch.zeros(tr.n_launch + 1, dtype=torch.int64, device=dev)
    lo[1:] = torch.cumsum(per_launch, 0)
    res = type(tr)(**{k: v for k, v in tr.__dict__.items()})
    res.samples = out.to(torch.int32).contiguous()
    res.launch_off = lo
    return res
