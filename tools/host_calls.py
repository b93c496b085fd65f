"""Measurement helper: host wall time of each public API call of the config-3 bench step
(perf_counter around each call, averaged over steps; calls without a readback are pure host
cost: Python binding + C host code + launches). Usage: python tools/host_calls.py [steps]"""
import collections
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    bench.spin_waits(0)
    torch.cuda.set_device(0)
    import paper_2411_02797_b200 as dc
    p, tr = bench.make_workload(3, 0, "cuda:0")
    ctx = dc.Context(0)
    F = int(tr.offsets[-1].item())
    tr.ids_buf = torch.empty(max(F, 1), dtype=torch.int32, device="cuda:0")
    tr.leaf_buf = torch.empty(max(tr.n_records, 1), dtype=torch.int32, device="cuda:0")
    ctx.reserve(2 * (16 * int(tr.samples.shape[0]) + 64 * tr.n_records + 4 * F) + (256 << 20))
    acc = collections.Counter()
    gc.disable()
    last = None
    for it in range(steps + 3):
        T = [time.perf_counter()]
        ids, d = dc.dc_intern_frames(ctx, tr.keys, tr.ids_buf); T.append(time.perf_counter())
        n_fr = d.size; T.append(time.perf_counter())
        cct, leaf = dc.dc_cct_build(ctx, tr.offsets, ids, n_fr, d, out_leaf=tr.leaf_buf); T.append(time.perf_counter())
        dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics); T.append(time.perf_counter())
        dc.dc_pc_sample_attribute(ctx, cct, tr.samples, leaf, tr.launch_off, n_stall=tr.n_stall); T.append(time.perf_counter())
        dc.dc_cct_rollup(ctx, cct); T.append(time.perf_counter())
        hot = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_INCLUSIVE, 0, 1 << dc.DC_KIND_KERNEL, 0.01, 10); T.append(time.perf_counter())
        dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_STALL, k=5, stall_node=hot[0][0]); T.append(time.perf_counter())
        dc.dc_cct_derived(ctx, cct, 0, True); T.append(time.perf_counter())
        if last is not None:
            last.free()
        last = cct
        T.append(time.perf_counter())
        if it >= 3:
            for i, nm in enumerate(["intern", "d.size", "build", "attribute", "pc", "rollup", "topk", "topk_stall", "derived", "free"]):
                acc[nm] += (T[i + 1] - T[i]) * 1e6
            acc["total"] += (T[-1] - T[0]) * 1e6
    ctx.sync()
    print({k: round(v / steps, 1) for k, v in acc.items()})


if __name__ == "__main__":
    main()
