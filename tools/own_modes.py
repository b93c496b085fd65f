"""Measurement helper: cost breakdown of the context-owner PC histogram kernel on config 3.

DC_OWN_MODE=2 streams the samples through shared memory only (TMA + mbarriers), =1 also
classifies them and forms keys, =0 is the real kernel. Results of modes 1/2 are not valid
CCTs (measurement only). Prints one JSON line per mode with the average kernel time.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2411_02797_b200 as dc  # noqa: E402


def main():
    p = gen.programs.config3()
    tr = gen.make_trace(p, pc=True, device="cuda")
    ctx = dc.Context(0)
    ids, d = dc.dc_intern_frames(ctx, tr.keys)
    for mode in sys.argv[1:] or ["2", "1", "0"]:
        os.environ["DC_OWN_MODE"] = mode
        for it in range(8):
            if it == 3:
                ctx.set_timing(True)
                ctx.timer_report()
            cct, leaf = dc.dc_cct_build(ctx, tr.offsets, ids, d.size, d)
            try:
                dc.dc_pc_sample_attribute(ctx, cct, tr.samples, leaf, tr.launch_off, n_stall=24)
            except dc.DcError:
                pass
            cct.free()
        t = ctx.timer_report()
        ctx.set_timing(False)
        k = t.get("k:pc_owner", (1, float("nan")))
        ms = k[1] / k[0]
        print(json.dumps({"mode": int(mode), "kernel_ms": round(ms, 4), "GBps": round(1.6e9 / (ms / 1e3) / 1e9, 1),
                          "pc_ms": round(t["pc"][1] / t["pc"][0], 4)}), flush=True)
        if mode == "0":
            print(json.dumps({k: round(v[1] / v[0], 4) for k, v in sorted(t.items())}), flush=True)
    os.environ["DC_OWN_MODE"] = "0"
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
