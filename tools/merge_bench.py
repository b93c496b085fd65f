#!/usr/bin/env python
"""Times dc_cct_merge_local (the merge's partition / exchange / reduce / canonicalise kernels
with a loopback exchange) over P logical ranks on one GPU, per phase (library CUDA-event
timers), for config 3 (P traces of 100M PC samples, different seeds), config 5 (P shards of 125M
records) or config 4 with --records (SURVEY's "5m" merge-stress variant: P shards of the cfg-4
shape). Prints one JSON line. Usage: python tools/merge_bench.py [--config 3|4|5] [--P 8] [--records R]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--records", type=int, default=None)
    args = ap.parse_args()
    import bench
    import paper_2411_02797_b200 as dc
    ctx = dc.Context(0)
    parts, dicts, local_ms = [], [], []
    for p in range(args.P):
        prog, tr = bench.make_workload(args.config, p, "cuda:0", args.records)
        F = int(tr.offsets[-1].item())
        tr.ids_buf = torch.empty(F, dtype=torch.int32, device="cuda")
        tr.leaf_buf = torch.empty(tr.n_records, dtype=torch.int32, device="cuda")
        if args.config == 4:  # pre-interned ids: the program's sorted pool is the dictionary (as bench.py)
            import numpy as np
            keys = torch.from_numpy(np.ascontiguousarray(prog.pool_keys).view(np.int32).reshape(-1, 4).copy()).cuda()
            d = tr.dict = dc.dc_dict_from_sorted(ctx, keys)
        else:
            ids, d = dc.dc_intern_frames(ctx, tr.keys, tr.ids_buf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cct, _ = bench.run_step(dc, ctx, tr, args.config, want_views=False)
        ctx.sync()
        parts.append(cct)
        dicts.append(d)
        del tr
        torch.cuda.empty_cache()
    v0 = parts[0].view()
    merged, gd = dc.dc_cct_merge_local(ctx, parts, dicts)  # warm-up
    merged.free()
    ctx.sync()
    ctx.set_timing(True)
    ctx.timer_report()
    times = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        merged, gd = dc.dc_cct_merge_local(ctx, parts, dicts)
        ctx.sync()
        times.append((time.perf_counter() - t0) * 1e3)
        mv = merged.view()
        merged.free()
    rep = ctx.timer_report()
    ctx.set_timing(False)
    phases = {k: round(v[1] / v[0], 3) for k, v in rep.items() if k.startswith("merge") or os.environ.get("MB_ALL")}
    print(json.dumps({"merge_local": {"config": args.config, "P": args.P, "local_nodes": int(v0.n_nodes),
                                      "local_bins": int(v0.n_bins), "merged_nodes": int(mv.n_nodes),
                                      "merged_bins": int(mv.n_bins), "wall_ms_median": round(sorted(times)[len(times) // 2], 3),
                                      "device_phase_ms": phases}}))


if __name__ == "__main__":
    main()
