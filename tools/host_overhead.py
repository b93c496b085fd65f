"""Measurement helper: host wall time vs device time of the bench step (config 3), to see how
much of ms_per_step is host orchestration. Prints per-step wall ms and device ms."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402


def main():
    bench.spin_waits(0)
    torch.cuda.set_device(0)
    import paper_2411_02797_b200 as dc
    p, tr = bench.make_workload(3, 0, "cuda:0")
    ctx = dc.Context(0)
    F = int(tr.offsets[-1].item())
    tr.ids_buf = torch.empty(max(F, 1), dtype=torch.int32, device="cuda:0")
    tr.leaf_buf = torch.empty(max(tr.n_records, 1), dtype=torch.int32, device="cuda:0")
    last = None
    for _ in range(5):
        cct, _ = bench.run_step(dc, ctx, tr, 3)
        if last is not None:
            last.free()
        last = cct
    ctx.sync()
    import cProfile
    import pstats
    pr = cProfile.Profile()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(ctx.stream)
    pr.enable()
    for _ in range(20):
        cct, _ = bench.run_step(dc, ctx, tr, 3)
        last.free()
        last = cct
    pr.disable()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / 20
    print({"wall_ms_per_step": round(wall, 4), "device_ms_per_step": round(e0.elapsed_time(e1) / 20, 4)})
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
