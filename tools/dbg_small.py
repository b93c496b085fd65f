"""Debug helper: small-P builders (lexicographic rank vs level loop) on a config-2 prefix."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2411_02797_b200 as dc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
R = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
p = gen.programs.program(cfg) if cfg != 3 else gen.programs.config3(n_samples=100_000)
tr = gen.make_trace(p, n_records=R)
ctx = dc.Context(0)
kk = torch.from_numpy(tr.keys.numpy().view(np.int32).reshape(-1, 4)).cuda()
off = torch.from_numpy(tr.offsets.numpy().view(np.int64)).cuda()
ids, d = dc.dc_intern_frames(ctx, kk)
res = {}
for mode in ["rank", "levels"]:
    if mode == "levels":
        os.environ["DC_TEST_BUILD_LEVELS"] = "1"
    try:
        cct, leaf = dc.dc_cct_build(ctx, off, ids, d.size, d)
        a = cct.to_numpy()
        a["leaf"] = leaf.cpu().numpy().view(np.uint32)
        res[mode] = a
        print(mode, "N", a["n_nodes"], "maxdepth", len(a["level_off"]) - 2, ctx.diag())
    except Exception as e:  # noqa: BLE001
        print(mode, "error", e)
if len(res) == 2:
    a, b = res["rank"], res["levels"]
    for k in ["parent", "frame", "depth", "level_off", "leaf"]:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        if x.shape != y.shape or not np.array_equal(x, y):
            bad = np.argwhere(x[: min(len(x), len(y))] != y[: min(len(x), len(y))])[:10].ravel()
            print(k, "DIFF", x.shape, y.shape, bad.tolist(), x[bad].tolist(), y[bad].tolist())
        else:
            print(k, "same")
