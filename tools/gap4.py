import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench
import paper_2411_02797_b200 as dc
bench.spin_waits(0); torch.cuda.set_device(0)
p, tr = bench.make_workload(4, 0, "cuda:0")
ctx = dc.Context(0)
keys = torch.from_numpy(np.ascontiguousarray(p.pool_keys).view(np.int32).reshape(-1, 4).copy()).cuda()
tr.dict = dc.dc_dict_from_sorted(ctx, keys)
s = ctx.stream
for it in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    h = []
    ev[0].record(s); h.append(time.perf_counter())
    cct, leaf = dc.dc_cct_build(ctx, tr.offsets, tr.ids, tr.n_frames, tr.dict)
    ev[1].record(s); h.append(time.perf_counter())
    dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics)
    ev[2].record(s); h.append(time.perf_counter())
    dc.dc_cct_rollup(ctx, cct)
    ev[3].record(s); h.append(time.perf_counter())
    hot = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_INCLUSIVE, 0, 1 << dc.DC_KIND_KERNEL, 0.01, 10)
    ev[4].record(s); h.append(time.perf_counter())
    dc.dc_cct_derived(ctx, cct, 0, True)
    ev[5].record(s); h.append(time.perf_counter())
    cct.free()
    ev[6].record(s); h.append(time.perf_counter())
    torch.cuda.synchronize()
    print([round(ev[i].elapsed_time(ev[i+1]),3) for i in range(6)], [round((h[i+1]-h[i])*1e3,3) for i in range(6)])
ctx.set_timing(True)
ctx.timer_report()
for it in range(2):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(s)
    cct, leaf = dc.dc_cct_build(ctx, tr.offsets, tr.ids, tr.n_frames, tr.dict)
    ev[1].record(s)
    torch.cuda.synchronize()
    print("timed", round(ev[0].elapsed_time(ev[1]), 3), {k: v for k, v in ctx.timer_report().items()})
    cct.free()
