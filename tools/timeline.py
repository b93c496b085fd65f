"""Measurement helper: device timeline of the bench step (torch.profiler / CUPTI activity records
of every kernel and memcpy in the process, the library's included). Prints, per profiled step, the
span, the summed kernel busy time and the idle time, then the largest idle gaps with the kernels
on both sides, and per-kernel busy totals. Usage: python tools/timeline.py [config] [steps]"""
import collections
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
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
    n_smp = int(tr.samples.shape[0]) if cfg == 3 else 0
    ctx.reserve(2 * (16 * n_smp + 64 * tr.n_records + 4 * F) + (256 << 20))
    last = None
    for _ in range(4):
        cct, _ = bench.run_step(dc, ctx, tr, cfg)
        if last is not None:
            last.free()
        last = cct
    ctx.sync()
    gc.disable()
    marks = []
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            torch.cuda.synchronize()
            cct, _ = bench.run_step(dc, ctx, tr, cfg)
            ctx.sync()
            last.free()
            last = cct
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev = sorted(ev, key=lambda e: e.time_range.start)
    # split into steps at gaps > 200 us (the host synchronisation between profiled steps)
    groups, cur = [], []
    for e in ev:
        if cur and e.time_range.start - max(x.time_range.end for x in cur[-3:]) > 200:
            groups.append(cur)
            cur = []
        cur.append(e)
    if cur:
        groups.append(cur)
    gaps = collections.Counter()
    gapn = collections.Counter()
    busy_k = collections.Counter()
    for g in groups:
        t0, t1 = g[0].time_range.start, max(e.time_range.end for e in g)
        busy, end = 0.0, t0
        for i, e in enumerate(g):
            s, f = e.time_range.start, e.time_range.end
            if s > end:
                key = (g[i - 1].name[:40] if i else "-") + " -> " + e.name[:40]
                gaps[key] += s - end
                gapn[key] += 1
            busy += max(0.0, f - max(s, end))
            end = max(end, f)
            busy_k[e.name[:60]] += f - s
        print(f"step: span {t1 - t0:8.1f} us  busy {busy:8.1f} us  idle {t1 - t0 - busy:7.1f} us  kernels {len(g)}")
    n = steps
    print("largest idle gaps (us per step, count per step):")
    for k, v in gaps.most_common(25):
        print(f"  {v / n:7.1f}  {gapn[k] / n:4.1f}  {k}")
    print("busy per kernel (us per step):")
    for k, v in busy_k.most_common(40):
        print(f"  {v / n:7.1f}  {k}")


if __name__ == "__main__":
    main()
