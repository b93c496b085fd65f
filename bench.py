#!/usr/bin/env python
"""bench.py — device-timed throughput of the CCT aggregation hot path on B200.

One step = one pass of the whole hot path over one synthetic trace
already resident in HBM: dc_intern_frames (raw 16-B frame keys) -> dc_cct_build ->
dc_cct_attribute_metrics -> dc_pc_sample_attribute -> dc_cct_rollup -> dc_hotspots_topk
(hotspot kernels + stall top-k of the top hotspot) -> dc_cct_derived.

Default workload (N=1): BASELINE.json config 3 — "LLM-inference-shaped PC-sampling trace:
100M samples attributed to (context, pc, stall reason), ~20k kernels" — the 100M-record
trace on which north_star sets the >= 50 % HBM-roofline target. At N>1 every rank runs its
own 100M-sample trace (different seed): weak scaling, no data-path collective yet.
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "profile records/sec into aggregated CCT (device-timed) and HBM GB/s vs peak at 1/2/4/8"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_for(kernel: str, cfg: int):
    """dram bytes per launch of `kernel` on config `cfg` from the committed ncu --set full
    summary (profiles/ncu_traffic.json, written by tools/ncu_summary.py), if captured."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t.get(f"cfg{cfg}:k_{kernel}")
    except Exception:
        return None


class Clocks:
    """Polls NVML (SM clock, max clock, throttle reasons) in a thread during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle", 0x2: "applications_clocks_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = float(os.environ.get("DC_BENCH_CLOCK_MS", "5")) / 1000.0  # measurement experiments only
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        if PINNED:  # keep the sampler off the core the timed host thread is pinned to
            try:
                others = set(os.sched_getaffinity(0) if not ALL_CORES else ALL_CORES) - PINNED
                if others:
                    os.sched_setaffinity(0, others)
            except Exception:
                pass
        while not self.stop:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        self.stop = False
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "n_samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "n_samples": len(self.samples)}


PINNED: set = set()
ALL_CORES: set = set()


def pin_host_thread(local: int):
    """The step's host round trips make its time sensitive to host-thread wake-up and migration:
    the launching thread is pinned to one core (rank-distinct), threads started later by the bench
    (the clock sampler) move themselves off it. Measured: 30-step medians 0.813-0.841 vs
    0.836-0.839 ms unpinned. BENCH_NOPIN=1 disables it."""
    global PINNED, ALL_CORES
    if os.environ.get("BENCH_NOPIN"):
        return
    try:
        cores = sorted(os.sched_getaffinity(0))
        ALL_CORES = set(cores)
        if len(cores) > 1:
            c = cores[(2 * local + 1) % len(cores)]
            os.sched_setaffinity(0, {c})
            PINNED = {c}
    except Exception:
        pass


def spin_waits(device: int):
    """The hot path's few host round trips (sizes read back between kernels) wait on the stream;
    spin-waiting (CU_CTX_SCHED_SPIN on the primary context, set before it is created) wakes the
    host within microseconds instead of after a yield/blocking wake-up, which otherwise adds
    box-dependent idle gaps to every step. Best effort: ignored if the context already exists."""
    try:
        from cuda.bindings import driver as cu
        cu.cuInit(0)
        _, dev = cu.cuDeviceGet(device)
        cu.cuDevicePrimaryCtxSetFlags(dev, cu.CUctx_flags.CU_CTX_SCHED_SPIN)
    except Exception:
        pass


# --------------------------------------------------------------------------- workloads
def make_workload(cfg: int, rank: int, device: str, n_records: int | None = None, stress: bool = False,
                  aggregated: bool = False):
    import gen
    from gen import programs
    if cfg == 3:
        p = programs.config3()
    elif cfg == 2:
        p = programs.config2()
    elif cfg == 4:
        p = programs.config4()
    elif cfg == 5:
        p = programs.config5(shard=rank)  # rank p builds shard p (its own seed and rank-local frames)
    else:
        p = programs.config1()
    if cfg != 5:
        p.seed = p.seed + 7919 * rank  # weak scaling: each rank its own draws of the same program
    tr = gen.make_trace(p, n_records=n_records, device=device, raw_keys=(cfg != 4), ids=(cfg == 4), pc=(cfg == 3))
    if stress and cfg == 3:  # variant 3s: 20k distinct contexts, samples of 8 launches interleaved
        from gen import stress as st
        tr = st.make_3s(tr)
    if aggregated and cfg == 3:  # per-PC aggregated records (count > 1), as CUPTI delivers them
        from gen import stress as st
        tr = st.make_aggregated(tr)
    return p, tr


def run_step(dc, ctx, tr, cfg: int, want_views: bool = True, comm=None):
    """One pass of the hot path; returns (cct, views). With a communicator (N > 1) the step is
    the local rows a1-a6 + a5 followed by the cross-rank merge a9 (NCCL exchange), and returns
    this rank's partition of the merged CCT; the views run on a single GPU's complete CCT."""
    if cfg == 4:
        d = tr.dict
        cct, leaf = dc.dc_cct_build(ctx, tr.offsets, tr.ids, tr.n_frames, tr.dict)
    else:
        ids, d = dc.dc_intern_frames(ctx, tr.keys, tr.ids_buf)
        cct, leaf = dc.dc_cct_build(ctx, tr.offsets, ids, d.size, d, out_leaf=tr.leaf_buf)
    dc.dc_cct_attribute_metrics(ctx, cct, leaf, tr.metrics)
    if cfg == 3:
        dc.dc_pc_sample_attribute(ctx, cct, tr.samples, leaf, tr.launch_off, n_stall=tr.n_stall)
    dc.dc_cct_rollup(ctx, cct)
    views = {}
    if comm is not None:
        lv = cct.view()
        views["local"] = (int(lv.n_nodes), int(lv.n_bins))
        part, _gd = dc.dc_cct_merge_ranks(ctx, comm, cct, d)
        cct.free()
        return part, views
    if want_views:
        # derived columns first: no readback, so its kernel runs while the host waits on the views
        buf = getattr(tr, "derived_buf", None)
        if buf is None or buf[0].numel() < cct.n_nodes:  # output columns allocated once (first warm-up step)
            n = max(cct.n_nodes, 1)
            buf = tr.derived_buf = (torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}"),
                                    torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}"))
        dc.dc_cct_derived(ctx, cct, 0, True, out=buf)
        hot = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_INCLUSIVE, 0, 1 << dc.DC_KIND_KERNEL, 0.01, 10)
        views["hotspots"] = hot
        if cfg == 3 and hot:
            views["stall"] = dc.dc_hotspots_topk(ctx, cct, dc.DC_VIEW_STALL, k=5, stall_node=hot[0][0])
    return cct, views


def records_of(tr, cfg):
    return tr.n_records + (int(tr.samples.shape[0]) if cfg == 3 else 0)


def alg_bytes_pc_hist(n_samples: int, n_bins: int) -> int:
    # SURVEY §8(d) a6 per unit: 16 B per sample read once + 16 B per bin written once
    return 16 * n_samples + 16 * n_bins


# --------------------------------------------------------------------------- oracle (CPU) legs
def oracle_sample(cfg: int, n_launch: int, rank: int = 0, stress: bool = False):
    """Bounded sample of the workload on the host: the first n_launch launch records and their
    PC samples (config 3), generated by the same generator."""
    import gen
    from gen import programs
    p = programs.config3() if cfg == 3 else programs.program(cfg)
    p.seed = p.seed + 7919 * rank
    tr = gen.make_trace(p, n_records=n_launch, pc=(cfg == 3), n_launch=n_launch if cfg == 3 else None)
    if stress and cfg == 3:
        from gen import stress as st
        tr = st.make_3s(tr)
    return p, tr


def oracle_time(p, tr, cfg: int) -> tuple[float, int]:
    import oracle
    t0 = time.perf_counter()
    ids, d = oracle.intern(tr.keys.numpy())
    o = oracle.OracleCCT(p.n_metrics, 24).insert(tr.offsets.numpy(), ids, tr.metrics.numpy())
    if cfg == 3:
        o.pc(tr.samples.numpy(), tr.n_launch)
    o.finalize()
    hot = o.topk(oracle.VIEW_INCLUSIVE, 0, 1 << 4, np.asarray(d["kind"], np.uint8), 0.01, 10)
    if cfg == 3 and len(hot):
        o.topk(oracle.VIEW_STALL, k=5, stall_node=int(hot[0]["id"]))
    o.derived(0, True)
    dt = time.perf_counter() - t0
    return dt, records_of(tr, cfg)


def cpu_baseline(cfg: int, n_launch: int, stress: bool = False):
    p, tr = oracle_sample(cfg, n_launch, stress=stress)
    dt, recs = oracle_time(p, tr, cfg)
    desc = (f"first {n_launch} launch records of config {cfg} and their {recs - n_launch} PC samples "
            f"(of 20,000 / 100,000,000{': the whole trace' if n_launch >= 20000 else ''})" if cfg == 3
            else f"first {n_launch} records of config {cfg}")
    return {"value": recs / dt, "unit": "records/s", "cores": 1, "kind": "oracle", "sample": desc,
            "seconds": round(dt, 3)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    n_launch = args.ref_launches
    p, tr = oracle_sample(args.config, n_launch)
    for _ in range(args.warmup):
        oracle_time(p, tr, args.config)
    ts, recs = [], 0
    for _ in range(args.steps):
        dt, recs = oracle_time(p, tr, args.config)
        ts.append(dt)
    tot = sum(ts)
    v = recs * len(ts) / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "records/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / len(ts), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"config{args.config}-sample", "launches": n_launch, "records_per_step": recs},
            "cpu_baseline": {"value": v, "unit": "records/s", "cores": 1, "kind": "oracle",
                             "sample": f"first {n_launch} launch records of config {args.config} + their PC samples"},
            "e2e": {"value": v, "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dc", choices=["dc", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--records", type=int, default=None, help="override record count (configs 2/4)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-launches", type=int, default=None,
                    help="oracle sample (launch records); default: config 3 whole (20,000 launches, 100M samples, ~20 s "
                         "on one core), else the first 4,000 records")
    ap.add_argument("--ref-launches", type=int, default=200)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--stress", action="store_true", help="config 3s: 20k distinct contexts, interleaved samples (generic schedule)")
    ap.add_argument("--aggregated", action="store_true", help="config 3 with per-PC aggregated records (counts > 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    spin_waits(local)
    pin_host_thread(local)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    import paper_2411_02797_b200 as dc
    dev = f"cuda:{local}"
    p, tr = make_workload(args.config, rank, dev, args.records, stress=args.stress, aggregated=args.aggregated)
    if args.config == 4:
        keys = torch.from_numpy(np.ascontiguousarray(p.pool_keys).view(np.int32).reshape(-1, 4).copy()).to(dev)
    ctx = dc.Context(local)
    comm = None
    if world > 1:
        from paper_2411_02797_b200 import dist as dcdist
        comm = dcdist.make_comm(ctx, world, rank)
    if args.config == 4:
        tr.dict = dc.dc_dict_from_sorted(ctx, keys)
    F = int(tr.offsets[-1].item())
    tr.ids_buf = torch.empty(max(F, 1), dtype=torch.int32, device=dev)
    tr.leaf_buf = torch.empty(max(tr.n_records, 1), dtype=torch.int32, device=dev)
    tr.derived_buf = None
    stream = ctx.stream
    recs = records_of(tr, args.config)

    def barrier():
        if dist is not None:
            dist.barrier()

    # setup: grow the library's stream-ordered pool past one step's peak (scratch of the PC
    # histogram ~12 B/sample, records and frames ~64 B/record, plus the live previous tree) so
    # no timed step maps new memory (dc_ctx_reserve; measured: a 5th-step stall of up to 30 ms)
    n_smp = int(tr.samples.shape[0]) if args.config == 3 else 0
    ctx.reserve(2 * (16 * n_smp + 64 * tr.n_records + 4 * F) + (256 << 20))
    # warm-up exactly like the timed loop (the previous step's CCT stays alive while the next one
    # is built), so the memory pool has grown to its steady-state size before timing
    last = None
    for _ in range(args.warmup):
        cct, _ = run_step(dc, ctx, tr, args.config, comm=comm)
        if last is not None:
            last.free()
        last = cct
    last.free()
    ctx.sync()
    # ---------------- timed region (device time, CUDA events on the library stream; the
    # library's own per-stage timers are off here and measured in a separate pass below)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # no Python garbage collection inside the timed region: a full collection over torch's heap
    # takes milliseconds and stalls the host between the step's launches
    gc.collect()
    gc.disable()
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    b0 = ctx.diag()["bytes_moved_est"]
    clk = Clocks(local)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with clk:
        e0.record(stream)
        last = None
        for i in range(args.steps):
            cct, views = run_step(dc, ctx, tr, args.config, comm=comm)
            if last is not None:
                last.free()
            last = cct
            step_ev[i].record(stream)  # per-step boundaries (distribution of step times)
        e1.record(stream)
        torch.cuda.synchronize()
    gc.enable()
    per_step = [e0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i]) for i in range(1, args.steps)]
    if os.environ.get("DC_BENCH_DUMP_STEPS"):
        print(json.dumps({"per_step_ms": [round(x, 3) for x in per_step]}), file=sys.stderr)
    barrier()
    launches = (ctx.launches - l0) // args.steps
    step_bytes = (ctx.diag()["bytes_moved_est"] - b0) / args.steps
    ms = e0.elapsed_time(e1) / args.steps
    if "local" in views:
        n_nodes, n_bins = views["local"]
    else:
        nv = last.view()
        n_bins, n_nodes = int(nv.n_bins), int(nv.n_nodes)
    last.free()
    # ---------------- instrumented pass: per-stage / per-kernel CUDA-event timers
    ctx.set_timing(True)
    ctx.timer_report()
    for _ in range(max(2, min(args.steps, 5))):
        cct, _ = run_step(dc, ctx, tr, args.config, comm=comm)
        cct.free()
    timers = ctx.timer_report()
    ctx.set_timing(False)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = recs * world / (ms / 1000.0)

    # ---------------- roofline of the dominant kernel (SURVEY §8(d) algorithmic bytes per launch)
    peak, peak_src = peaks()
    R_, F_ = tr.n_records, F
    alg = {  # kernel timer -> algorithmic bytes of one launch
        "k:pc_owner": alg_bytes_pc_hist(n_smp, n_bins) if args.config == 3 else 0,  # 16 B/sample + 16 B/bin
        "k:pc_table": alg_bytes_pc_hist(n_smp, n_bins) if args.config == 3 else 0,  # generic schedule (3s)
        "k:intern_insert": 20 * F_,                          # 16-B raw key read + 4-B id written per key
        "k:path_hash": 8 * (R_ + 1) + 4 * F_ + 8 * R_,       # offsets + frames read, 8-B path hash written
        "k:path_group": 8 * (R_ + 1) + 4 * F_ + 12 * R_,     # offsets + frames (exact verify) + hash read, slot written
    }
    cand = [k for k in alg if k in timers and alg[k] and (args.config != 3 or k in ("k:pc_owner", "k:pc_table"))]
    kname = max(cand, key=lambda k: timers[k][1] / timers[k][0]) if cand else None
    roof = None
    if kname:
        cnt, tot_ms = timers[kname]
        kms = tot_ms / cnt
        ab = alg[kname]
        ach = ab / (kms / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": kname[2:], "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": (traffic_for(kname[2:], args.config) if args.records is None and not args.stress
                            and not args.aggregated else None),  # captures are of the default workloads
                "alg_bytes_per_launch": ab,
                "kernel_ms": round(kms, 4), "peak_source": peak_src,
                "share_of_step": round(kms / ms, 4)}
    stages = {k: round(v[1] / v[0], 4) for k, v in timers.items()}

    # ---------------- e2e through the public API with host buffers
    e2e = None
    if args.e2e_steps > 0 and args.config in (1, 2, 3, 5):
        host = {"keys": tr.keys.cpu().pin_memory(), "offsets": tr.offsets.cpu().pin_memory(),
                "metrics": tr.metrics.cpu().pin_memory()}
        if args.config == 3:
            host["samples"] = tr.samples.cpu().pin_memory()
            if tr.launch_off is not None:
                host["launch_off"] = tr.launch_off.cpu().pin_memory()
        devb = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
        h2d = sum(v.numel() * v.element_size() for v in host.values())
        d2h = 0

        class T:
            pass
        t2 = T()
        t2.ids_buf, t2.leaf_buf, t2.derived_buf, t2.n_stall = tr.ids_buf, tr.leaf_buf, None, getattr(tr, "n_stall", 24)
        t2.n_records = tr.n_records
        t2.launch_off = None
        for k, v in devb.items():
            setattr(t2, k, v)
        gc.collect()
        gc.disable()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            f0.record(stream)
            for _ in range(args.e2e_steps):
                for k in host:
                    devb[k].copy_(host[k], non_blocking=True)
                cct, views = run_step(dc, ctx, t2, args.config, comm=comm)
                # results read back to the host every step: the top-k entries (24 B each)
                d2h = 24 * (len(views.get("hotspots", [])) + len(views.get("stall", [])))
                cct.free()
            f1.record(stream)
        torch.cuda.synchronize()
        gc.enable()
        barrier()
        ems = f0.elapsed_time(f1) / args.e2e_steps
        if dist is not None:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": recs * world / (ems / 1000.0), "unit": "records/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(ems, 3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, args.cpu_launches or (20000 if args.config == 3 else 4000), stress=args.stress)

    if rank == 0:
        wl = {3: "config3: LLM-inference PC-sampling trace, 20k launch records (raw 16-B frame keys, mean depth ~42) "
                 "+ 100M PC samples (16 B each), 24 stall reasons",
              2: "config2: ResNet-50-training-shaped trace, 1M launch records, 5 metrics, raw frame keys",
              1: "config1: tiny 10k-record trace", 4: "config4: JAX-shaped pre-interned trace, depth <= 256",
              5: "config5: one DDP shard per rank (config-2 program, rank-local frames, own raw-key dictionary), "
                 "125M records per rank; merged across ranks at N > 1"}[args.config]
        if args.aggregated and args.config == 3:
            wl = ("config3 aggregated: config 3's 100M raw samples as per-launch per-(pc, stall) records with counts "
                  f"({int(tr.samples.shape[0])} records, as CUPTI's PC-sampling API delivers them)")
        if args.stress and args.config == 3:
            wl = ("config3s (stress variant): config 3 with a per-launch outermost frame (20k distinct contexts) and the "
                  "samples of each 8 consecutive launches interleaved round robin (no per-launch offsets: generic schedule)")
        line = {"metric": METRIC, "value": value, "unit": "records/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic (counter-based generator, gen/)",
                "config": {"workload": wl, "config_id": args.config, "variant": "3s" if args.stress else ("aggregated" if args.aggregated else None),
                           "records_per_gpu_step": recs,
                           "pc_samples": int(tr.samples.shape[0]) if args.config == 3 else 0,
                           "launch_records": tr.n_records, "nodes": n_nodes, "bins": n_bins,
                           "l2": (f"inputs larger than L2 ({step_bytes / 1e9:.2f} GB read per step); no flush"
                                  if step_bytes > 126e6 else
                                  f"inputs fit in L2 ({step_bytes / 1e6:.1f} MB per step, not flushed: tiny "
                                  f"latency-bound config, not a bandwidth figure)"),
                           "parallelism": (f"dp{world}: per-rank shard, local CCT + NCCL cross-rank merge "
                                           "(dc_cct_merge_ranks), weak scaling") if world > 1 else "dp1"},
                "roofline": roof, "stages_ms": stages, "gpu_launches": int(launches),
                "step_hbm": {"alg_bytes_per_step": int(step_bytes), "gbs": round(step_bytes / (ms / 1e3) / 1e9, 1),
                             "frac_of_peak": round(step_bytes / (ms / 1e3) / 1e9 / peak, 4)},
                "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
                "step_ms_dist": {"min": round(min(per_step), 4), "median": round(statistics.median(per_step), 4),
                                 "max": round(max(per_step), 4)}}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
