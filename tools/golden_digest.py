#!/usr/bin/env python
"""Writes tests/golden/digest_cfg{4,5}.json: the CPU oracle's canonical CCT digest for the
full-size configs 4 (200M records, depth <= 256) and 5 (8 shards x 125M records, per-shard
raw-key dictionaries, merged = CCT of the concatenated trace, reading R19).

Calls only oracle/ (the arithmetic) and gen/ (the seeded inputs): no expected value comes
from the CUDA path. The traces are far larger than host memory, so records are generated in
chunks (gen.make_chunk_host; records are drawn independently, so the chunks concatenate to
the exact trace) and fed to ONE oracle trie in trace order (OracleCCT.insert per chunk: the
per-record insertion is unchanged, only the loop over records is split).

Config 5 needs interning over the raw keys of all shards. The oracle's intern ranks the
distinct keys; with the trace streamed this takes two passes: (1) the distinct keys of every
chunk (oracle.intern of the chunk), their union ranked by oracle.intern once more; (2) per
chunk, oracle.intern again for the chunk-local ids, mapped to the global rank of each local
dictionary entry (a plain dict lookup over <= 1k keys). Chunk generation + interning runs in
worker processes; the trie insertion runs in the main process, in trace order.

Usage: python tools/golden_digest.py [4] [5] [--chunk 1000000] [--workers 7]
The JSON records the generator version (gen.generator_version()); the GPU tests refuse a
stale file.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def sample_nodes(N: int, k: int = 256) -> list[int]:
    return sorted(set([0] + np.linspace(0, N - 1, k).astype(np.int64).tolist()))


def derived_samples(o, N: int, M: int) -> dict:
    nodes = sample_nodes(N)
    out = {"nodes": nodes}
    for m in range(M):
        for incl in (True, False):
            mean, std = o.derived(m, incl)
            out[f"m{m}_{'incl' if incl else 'excl'}"] = [[float(mean[n]), float(std[n])] for n in nodes]
    return out


def summary(o, a, dict_keys, extra: dict) -> dict:
    d = {"generator_version": gen.generator_version(), "n_nodes": int(a["n_nodes"]), "n_metrics": int(a["n_metrics"]),
         "n_stall": int(a["n_stall"]), "n_pc_nodes": int(a["n_pc_nodes"]), "n_bins": int(a["n_bins"]),
         "n_frames": int(len(dict_keys)), "max_depth": int(a["depth"].max()) if a["n_nodes"] else 0,
         "sha256": oracle.digest(a, dict_keys), "root_icnt": int(a["icnt"][0]),
         "root_isum": [int(a["isum"][m][0]) for m in range(int(a["n_metrics"]))]}
    d.update(extra)
    d["derived"] = derived_samples(o, int(a["n_nodes"]), int(a["n_metrics"]))
    return d


# ----------------------------------------------------------------------------- config 4
def run_config4(chunk: int) -> dict:
    p = gen.programs.config4()
    R = p.default_records
    o = oracle.OracleCCT(p.n_metrics, 0)
    t0 = time.time()
    for r0 in range(0, R, chunk):
        n = min(chunk, R - r0)
        off, ids, _, met = gen.make_chunk_host(p, r0, n, raw_keys=False, ids=True)
        o.insert(off, ids, met)
        if (r0 // chunk) % 20 == 0:
            print(f"cfg4: {r0 + n:,}/{R:,} records, {time.time() - t0:.0f} s", flush=True)
    o.finalize()
    secs = time.time() - t0
    a = o.arrays()
    extra = {"config": 4, "seed": p.seed, "records": R, "oracle_seconds": round(secs, 1), "oracle_cores": 1,
             "leaf_sha256": oracle.leaf_digest(a["leaf"]),
             "note": "pre-interned ids; dictionary = the program's sorted pool keys (dc_dict_from_sorted)"}
    return summary(o, a, p.pool_keys, extra)


# ----------------------------------------------------------------------------- config 5
_W: dict = {}


def _w_init():
    _W["progs"] = {}


def _prog5(s):
    if s not in _W["progs"]:
        _W["progs"][s] = gen.programs.config5(s)
    return _W["progs"][s]


def _pass1(job):
    s, r0, n = job
    _, _, keys, _ = gen.make_chunk_host(_prog5(s), r0, n, raw_keys=True)
    _, d = oracle.intern(keys)
    return d


def _pass2(job):
    s, r0, n, gkeys = job
    off, _, keys, met = gen.make_chunk_host(_prog5(s), r0, n, raw_keys=True)
    ids, d = oracle.intern(keys)
    rank = {(int(k["kind"]), int(k["str_id"]), int(k["addr"])): i for i, k in enumerate(gkeys)}
    remap = np.array([rank[(int(k["kind"]), int(k["str_id"]), int(k["addr"]))] for k in d], np.uint32)
    return off, remap[ids] if len(ids) else ids, met


def run_config5(chunk: int, workers: int, shards: int = 8) -> dict:
    progs = [gen.programs.config5(s) for s in range(shards)]
    jobs = [(s, r0, min(chunk, progs[s].default_records - r0)) for s in range(shards)
            for r0 in range(0, progs[s].default_records, chunk)]
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_w_init) as pool:
        dicts = pool.map(_pass1, jobs, chunksize=1)
    gkeys = oracle.intern(np.concatenate(dicts))[1]
    print(f"cfg5 pass 1: {len(gkeys)} distinct keys over {len(jobs)} chunks, {time.time() - t0:.0f} s", flush=True)
    o = oracle.OracleCCT(2, 0)
    with ctx.Pool(workers, initializer=_w_init) as pool:
        for i, (off, ids, met) in enumerate(pool.imap(_pass2, [j + (gkeys,) for j in jobs], chunksize=1)):
            o.insert(off, ids, met)
            if i % 50 == 0:
                print(f"cfg5 pass 2: chunk {i}/{len(jobs)}, {time.time() - t0:.0f} s", flush=True)
    o.finalize()
    secs = time.time() - t0
    a = o.arrays()
    extra = {"config": 5, "seeds": [p.seed for p in progs], "records": sum(p.default_records for p in progs),
             "shards": shards, "oracle_seconds": round(secs, 1), "oracle_cores": workers + 1,
             "note": "oracle over the concatenation of shards 0..7 in order; chunk generation + interning in "
                     f"{workers} worker processes, trie insertion single-threaded"}
    return summary(o, a, gkeys, extra)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[4, 5])
    ap.add_argument("--chunk", type=int, default=1_000_000)
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    args = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    for cfg in args.configs:
        d = run_config4(args.chunk) if cfg == 4 else run_config5(args.chunk, args.workers)
        d["written_by"] = "tools/golden_digest.py (oracle/ + gen/ only)"
        path = os.path.join(GOLDEN, f"digest_cfg{cfg}.json")
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print(f"wrote {path}: N={d['n_nodes']} sha256={d['sha256'][:16]}… in {d['oracle_seconds']} s", flush=True)


if __name__ == "__main__":
    main()
