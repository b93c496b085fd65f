"""Measurement helper: host wall time vs device time of the bench step for a config, with a
cProfile of the binding calls (which call the host spends its time in). Usage:
python tools/host_profile.py [config] [steps]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
import torch  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    bench.spin_waits(0)
    torch.cuda.set_device(0)
    import paper_2411_02797_b200 as dc
    p, tr = bench.make_workload(cfg, 0, "cuda:0")
    ctx = dc.Context(0)
    if cfg == 4:
        keys = torch.from_numpy(np.ascontiguousarray(p.pool_keys).view(np.int32).reshape(-1, 4).copy()).cuda()
        tr.dict = dc.dc_dict_from_sorted(ctx, keys)
    F = int(tr.offsets[-1].item())
    tr.ids_buf = torch.empty(max(F, 1), dtype=torch.int32, device="cuda:0")
    tr.leaf_buf = torch.empty(max(tr.n_records, 1), dtype=torch.int32, device="cuda:0")
    last = None
    for _ in range(3):
        cct, _ = bench.run_step(dc, ctx, tr, cfg)
        if last is not None:
            last.free()
        last = cct
    ctx.sync()
    pr = cProfile.Profile()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(ctx.stream)
    pr.enable()
    for _ in range(steps):
        cct, _ = bench.run_step(dc, ctx, tr, cfg)
        last.free()
        last = cct
    pr.disable()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / steps
    print({"config": cfg, "wall_ms_per_step": round(wall, 4), "device_ms_per_step": round(e0.elapsed_time(e1) / steps, 4)})
    ctx.set_timing(True)
    ctx.timer_report()
    cct, _ = bench.run_step(dc, ctx, tr, cfg)
    print({k: v for k, v in ctx.timer_report().items() if k.startswith("h:") or not k.startswith("k:")})
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)


if __name__ == "__main__":
    main()
