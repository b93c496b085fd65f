"""Program tables for the synthetic traces (TEST/BENCH INPUT ONLY — none of the method's
arithmetic lives here).

Each config is a *program model*: a list of launch sites, each with a fixed unified call
path Python -> framework op(s) -> native -> GPU API -> kernel (§4.1 "call
path"), per-site base GPU times, and (config 3) per-kernel PC / stall-reason
distributions. Floating point (log-normal, Zipf) is used only here, while building the
tables; per-record draws are integer-only (gen/csrc/gen_core.h). Shapes follow SURVEY.md
§8(d) "Configs as concrete synthetic inputs"; the recipe is restated in DESIGN.md.
"""
from __future__ import annotations

import numpy as np

KIND_PY, KIND_OP, KIND_NATIVE, KIND_API, KIND_KERNEL, KIND_INSTR = 0, 1, 2, 3, 4, 5
KIND_NAMES = ["PY", "OP", "NATIVE", "API", "KERNEL", "INSTR"]

# Stall-reason ids (24, CUPTI-like); 3 = math_dep and 7 = const_mem_miss are the ones the
# paper's Llama3 case study names.
STALL_NAMES = ["selected", "not_selected", "long_scoreboard", "math_dep", "short_scoreboard",
               "mio_throttle", "lg_throttle", "const_mem_miss", "barrier", "membar", "branch_resolving",
               "dispatch", "drain", "imc_miss", "no_instruction", "pipe_busy", "sleeping",
               "tex_throttle", "wait", "misc", "sync", "tmem", "gmma", "other"]
N_STALL = 24


class Pool:
    """Raw frame keys (kind, str_id, addr) + string table; index = insertion order until
    finalize() sorts it (then index = rank of the key in the sorted pool)."""

    def __init__(self):
        self.strings: list[str] = []
        self.str_ix: dict[str, int] = {}
        self.keys: list[tuple[int, int, int]] = []
        self.key_ix: dict[tuple[int, int, int], int] = {}
        self.labels: list[str] = []

    def s(self, name: str) -> int:
        if name not in self.str_ix:
            self.str_ix[name] = len(self.strings)
            self.strings.append(name)
        return self.str_ix[name]

    def key(self, kind: int, sname: str, addr: int, label: str | None = None) -> int:
        k = (kind, self.s(sname), int(addr))
        if k not in self.key_ix:
            self.key_ix[k] = len(self.keys)
            self.keys.append(k)
            if not label:
                label = f"{sname}+{addr:#x}" if kind >= KIND_NATIVE else f"{sname}:{addr}"
            self.labels.append(label)
        return self.key_ix[k]

    def py(self, file: str, line: int, func: str = "") -> int:
        return self.key(KIND_PY, file, line, f"{func or file}@{file}:{line}")

    def op(self, name: str) -> int:
        return self.key(KIND_OP, name, 0, name)

    def native(self, module: str, pc: int, kind: int = KIND_NATIVE, label: str = "") -> int:
        return self.key(kind, module, pc, label or f"{module}+{pc:#x}")

    def finalize(self, site_paths: list[list[int]]):
        """Sort keys lexicographically; remap the site paths to sorted indices."""
        order = sorted(range(len(self.keys)), key=lambda i: self.keys[i])
        rank = np.empty(len(order), np.int64)
        rank[np.asarray(order, np.int64)] = np.arange(len(order))
        keys = np.zeros(len(order), dtype=[("kind", "<u4"), ("str_id", "<u4"), ("addr", "<u8")])
        for new, old in enumerate(order):
            keys[new] = self.keys[old]
        labels = [self.labels[old] for old in order]
        paths = [[int(rank[f]) for f in p] for p in site_paths]
        return keys, labels, paths


def _pack_sites(paths: list[list[int]]):
    off = np.zeros(len(paths) + 1, np.uint32)
    off[1:] = np.cumsum([len(p) for p in paths])
    frames = np.asarray([f for p in paths for f in p], np.uint32)
    if frames.size == 0:
        frames = np.zeros(1, np.uint32)
    return off, frames


class Program:
    """Everything gen_core.h needs for one config, as numpy arrays + scalars."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


# ------------------------------------------------------------------------------------------
# Config 1: tiny random template tree (SURVEY §8(d) cfg 1)
# ------------------------------------------------------------------------------------------
def config1(seed: int = 1, n_templates: int = 400) -> Program:
    rng = np.random.default_rng(seed)
    pool = Pool()
    # exactly 1000 raw keys: 40% PY, 10% OP, 35% native, 5% API, 10% kernel
    ids = []
    for i in range(400):
        ids.append(pool.py(f"src{i % 40}.py", 1 + int(rng.integers(1, 2000)) * 41 + i, f"fn{i}"))
    for i in range(100):
        ids.append(pool.op(f"aten::op{i}"))
    for i in range(350):
        ids.append(pool.native(f"lib{i % 10}.so", 0x1000 + 16 * i + int(rng.integers(0, 8)) * 0x100000))
    for i in range(50):
        ids.append(pool.native("libcudart.so", 0x400 + 8 * i, KIND_API))
    for i in range(100):
        ids.append(pool.native(f"kern{i % 4}.cubin", 0x10 * i, KIND_KERNEL))
    assert len(pool.keys) == 1000
    by_kind = [np.asarray([f for f in ids if pool.keys[f][0] == k]) for k in range(5)]
    kind_p = np.array([0.40, 0.10, 0.35, 0.05, 0.10])

    def frame():
        k = int(rng.choice(5, p=kind_p))
        return int(rng.choice(by_kind[k]))

    paths: list[list[int]] = []
    for t in range(n_templates):
        L = 32 if t == 1 else int(rng.integers(4, 25))
        p: list[int] = []
        if paths and rng.random() < 0.7:
            src = paths[int(rng.integers(0, len(paths)))]
            p = list(src[: int(rng.integers(1, len(src) + 1))])[:L]
        while len(p) < L:
            p.append(frame())
        paths.append(p)
    keys, labels, paths = pool.finalize(paths)
    off, frames = _pack_sites(paths)
    return Program(name="cfg1", seed=seed, mode=1, site_off=off, site_frames=frames, pool_keys=keys,
                   labels=labels, strings=pool.strings, trunc_permille=200, rec_permille=10, max_depth=32,
                   empty_mod=3331, empty_rem=7, force_record=1, force_site=1, site_rec_k=None,
                   rec_pos=0, rec_a=0, rec_b=0, dyn_per100k=0, dyn_min=0, dyn_max=0,
                   met_kind=1, n_metrics=2, site_base_ns=None, site_warps=None, site_smem=None,
                   default_records=10_000)


# ------------------------------------------------------------------------------------------
# Config 2: PyTorch ResNet-50 training-shaped (SURVEY §8(d) cfg 2)
# ------------------------------------------------------------------------------------------
def _resnet_sites(pool: Pool, rng, local_tag: int | None = None):
    """Returns a list of (path, kind-of-op) for one training iteration, program order."""
    prefix = [pool.py("train.py", 212, "main"), pool.py("train.py", 150, "train_epoch"),
              pool.py("train.py", 97, "train_step")]
    fwd_call = pool.py("train.py", 61, "train_step")
    wrapped = pool.py("torch/nn/modules/module.py", 1736, "_wrapped_call_impl")
    callimpl = pool.py("torch/nn/modules/module.py", 1747, "_call_impl")
    dispatch = [pool.native("libtorch_cpu.so", 0x2A0000 + 0x140 * i) for i in range(int(rng.integers(4, 9)))]
    api = pool.native("libcudart.so", 0x6E0D0, KIND_API, "cudaLaunchKernel")
    eval_fn = pool.op("autograd::engine::evaluate_function")
    sites: list[list[int]] = []
    op_natives: dict[str, list[int]] = {}

    chains = {
        "conv": ["aten::conv2d", "aten::convolution", "aten::_convolution", "aten::cudnn_convolution"],
        "bn": ["aten::batch_norm", "aten::_batch_norm_impl_index", "aten::cudnn_batch_norm"],
        "relu": ["aten::relu_"], "maxpool": ["aten::max_pool2d", "aten::max_pool2d_with_indices"],
        "add": ["aten::add_"], "avgpool": ["aten::adaptive_avg_pool2d", "aten::mean"],
        "fc": ["aten::linear", "aten::addmm"], "loss": ["aten::cross_entropy_loss", "aten::log_softmax", "aten::nll_loss"],
    }
    nkern_fwd = {"conv": 2, "bn": 1, "relu": 1, "maxpool": 1, "add": 1, "avgpool": 1, "fc": 1, "loss": 3}
    nkern_bwd = {"conv": 3, "bn": 1, "relu": 1, "maxpool": 1, "add": 1, "avgpool": 1, "fc": 2, "loss": 3}
    func_line = {"conv": 454, "bn": 2478, "relu": 1500, "maxpool": 796, "add": 0, "avgpool": 1214, "fc": 116, "loss": 3086}

    def natives(opk, bwd):
        key = opk + ("_bwd" if bwd else "")
        if key not in op_natives:
            base = 0x900000 + 0x10000 * len(op_natives)
            op_natives[key] = [pool.native("libtorch_cuda.so", base + 0x60 * i) for i in range(int(rng.integers(4, 9)))]
        return op_natives[key]

    def kernels(opk, bwd, n):
        return [pool.native(f"{opk}_kernels.cubin", (0x8000 if bwd else 0) + 0x400 * i, KIND_KERNEL) for i in range(n)]

    leaf_calls = []  # (module py frames, opk)

    def module_frames(stack):
        fr = []
        for (file, line, fn) in stack:
            fr += [wrapped, callimpl, pool.py(file, line, fn)]
        return fr

    model = ("torchvision/models/resnet.py", 285, "ResNet.forward")
    leaf_calls.append(([model], "conv", 268))
    leaf_calls.append(([model], "bn", 269))
    leaf_calls.append(([model], "relu", 270))
    leaf_calls.append(([model], "maxpool", 271))
    for li, nblocks in enumerate([3, 4, 6, 3]):
        layer = ("torchvision/models/resnet.py", 273 + li, f"layer{li+1}")
        seq = ("torch/nn/modules/container.py", 250, "Sequential.forward")
        for b in range(nblocks):
            blk = ("torchvision/models/resnet.py", 140 + 0 * b, "Bottleneck.forward")
            st = [model, layer, seq, blk]
            for (opk, line) in [("conv", 143), ("bn", 144), ("relu", 145), ("conv", 147), ("bn", 148),
                                ("relu", 149), ("conv", 151), ("bn", 152)]:
                leaf_calls.append((st, opk, line + 1000 * b + 10000 * li))
            if b == 0:
                leaf_calls.append((st, "conv", 155 + 10000 * li))
                leaf_calls.append((st, "bn", 156 + 10000 * li))
            leaf_calls.append((st, "add", 158 + 1000 * b + 10000 * li))
            leaf_calls.append((st, "relu", 159 + 1000 * b + 10000 * li))
    leaf_calls.append(([model], "avgpool", 278))
    leaf_calls.append(([model], "fc", 280))
    loss_call = ([("train.py", 63, "loss_fn")], "loss", 64)

    def path(stack, opk, line, bwd):
        p = list(prefix) + [fwd_call]
        p += module_frames(stack[:-1])
        file, _, fn = stack[-1]
        p += [wrapped, callimpl, pool.py(file, line, fn)]
        p += [pool.py("torch/nn/functional.py", func_line[opk], opk)] if opk != "add" else []
        if bwd:
            p += [eval_fn, pool.op(f"{chains[opk][0].split('::')[1].capitalize()}Backward0")]
            p += [pool.op(c + "_backward") for c in chains[opk][-2:]]
        else:
            p += [pool.op(c) for c in chains[opk]]
        p += dispatch + natives(opk, bwd) + [api]
        return p

    for stack, opk, line in leaf_calls:
        for k in kernels(opk, False, nkern_fwd[opk]):
            sites.append(path(stack, opk, line, False) + [k])
    lp = list(prefix) + [pool.py("train.py", 62, "train_step"), pool.py("train.py", 64, "loss_fn")]
    for c, k in zip(chains["loss"], kernels("loss", False, 3)):
        sites.append(lp + [pool.op(c)] + dispatch + natives("loss", False) + [api, k])
    bw = list(prefix) + [pool.py("train.py", 66, "train_step"), pool.py("torch/_tensor.py", 581, "backward"),
                         pool.py("torch/autograd/__init__.py", 347, "backward")]
    for c, k in zip(chains["loss"], kernels("loss", True, 3)):
        sites.append(bw + [eval_fn, pool.op(c + "_backward")] + dispatch + natives("loss", True) + [api, k])
    for stack, opk, line in reversed(leaf_calls):
        for k in kernels(opk, True, nkern_bwd[opk]):
            sites.append(path(stack, opk, line, True) + [k])
    opt = list(prefix) + [pool.py("train.py", 68, "train_step"), pool.py("torch/optim/sgd.py", 135, "step"),
                          pool.py("torch/optim/sgd.py", 370, "_single_tensor_sgd")]
    for p_ in range(161):
        for j, opn in enumerate(["aten::add_", "aten::mul_"]):
            sites.append(opt + [pool.py("torch/optim/sgd.py", 380 + j, "_single_tensor_sgd"), pool.op(opn)]
                         + dispatch + natives("opt", False) + [api, pool.native("opt_kernels.cubin", 0x400 * j, KIND_KERNEL)])
    if local_tag is not None:
        # rank-local frames (data loader / logging): prepended to 5% of the sites
        n_local = max(1, len(sites) // 20)
        # same file names on every rank (string ids stay consistent across shards), rank-specific
        # lines: these keys differ between the per-shard dictionaries
        dl = [pool.py("dataloader.py", 1000 + local_tag, "fetch"), pool.py("logging.py", 2000 + local_tag, "log")]
        for i in range(n_local):
            j = (i * 20 + 3) % len(sites)
            sites[j] = sites[j][:3] + dl + sites[j][3:]
    return sites


def config2(seed: int = 2) -> Program:
    rng = np.random.default_rng(seed)
    pool = Pool()
    sites = _resnet_sites(pool, rng)
    keys, labels, paths = pool.finalize(sites)
    off, frames = _pack_sites(paths)
    n = len(paths)
    base = np.maximum(1000, np.exp(np.log(20_000.0) + 1.2 * rng.standard_normal(n))).astype(np.uint64)
    warps = (1 << rng.integers(0, 6, n)).astype(np.uint32)
    smem = np.where(rng.random(n) < 0.3, 0, 1024 * rng.integers(1, 229, n)).astype(np.uint32)
    return Program(name="cfg2", seed=seed, mode=0, site_off=off, site_frames=frames, pool_keys=keys,
                   labels=labels, strings=pool.strings, trunc_permille=0, rec_permille=0, max_depth=1024,
                   empty_mod=0, empty_rem=0, force_record=2**63, force_site=0, site_rec_k=None,
                   rec_pos=0, rec_a=0, rec_b=0, dyn_per100k=0, dyn_min=0, dyn_max=0,
                   met_kind=2, n_metrics=5, site_base_ns=base, site_warps=warps, site_smem=smem,
                   default_records=1_000_000)


# ------------------------------------------------------------------------------------------
# Config 3: LLM-decode-shaped PC sampling (SURVEY §8(d) cfg 3)
# ------------------------------------------------------------------------------------------
LLM_SITES = [("input_layernorm", "rmsnorm", 0.6), ("input_layernorm", "to_fp16", 0.3),
             ("q_proj", "gemm", 3.0), ("k_proj", "gemm", 1.0), ("v_proj", "gemm", 1.0),
             ("rotary", "rope", 0.4), ("attn", "flash_attn", 4.0), ("attn", "softmax_lse", 0.3),
             ("o_proj", "gemm", 3.0), ("residual", "add", 0.3), ("post_attention_layernorm", "rmsnorm", 0.6),
             ("post_attention_layernorm", "to_fp16", 0.3), ("gate_proj", "gemm", 6.0), ("up_proj", "gemm", 6.0),
             ("act", "silu_mul", 0.5), ("down_proj", "gemm", 6.0), ("residual2", "add", 0.3),
             ("kv_cache", "copy", 0.4), ("quant", "fp8_quant", 0.5), ("dequant", "fp8_dequant", 0.5)]


def config3(seed: int = 3, n_launch: int = 20_000, n_samples: int = 100_000_000, n_layers: int = 32) -> Program:
    rng = np.random.default_rng(seed)
    pool = Pool()
    prefix = [pool.py("serve.py", 40, "main"), pool.py("serve.py", 88, "serve_loop"),
              pool.py("engine.py", 301, "step"), pool.py("engine.py", 212, "execute_model"),
              pool.py("model_runner.py", 1450, "execute_model"), pool.py("model_runner.py", 1301, "_model_forward"),
              pool.py("torch/utils/_contextlib.py", 116, "decorate_context"), pool.py("llama.py", 512, "LlamaModel.forward")]
    wrapped = pool.py("torch/nn/modules/module.py", 1736, "_wrapped_call_impl")
    callimpl = pool.py("torch/nn/modules/module.py", 1747, "_call_impl")
    dispatch = [pool.native("libtorch_cpu.so", 0x2A0000 + 0x140 * i) for i in range(12)]
    api = pool.native("libcudart.so", 0x6E0D0, KIND_API, "cudaLaunchKernel")
    kern_names = sorted({k for _, k, _ in LLM_SITES})
    kern_ix = {k: i for i, k in enumerate(kern_names)}
    sites, site_kernel, weight = [], [], []
    for layer in range(n_layers):
        lf = pool.py("llama.py", 520, "LlamaModel.forward.layer")  # loop body line
        dec = pool.py("llama.py", 2000 + layer, f"decoder_layer_{layer}")  # unrolled per-layer graph frame
        for si, (mod, kern, w) in enumerate(LLM_SITES):
            p = list(prefix) + [lf, wrapped, callimpl, dec, wrapped, callimpl,
                                pool.py("llama.py", 300 + 7 * si, f"{mod}.forward")]
            p += [pool.py("torch/nn/functional.py", 100 + si, mod)]
            nops = 1 + (si % 3)
            p += [pool.op(f"vllm::{kern}_op{j}") for j in range(nops)]
            p += dispatch + [pool.native("libvllm_C.so", 0x10000 * kern_ix[kern] + 0x80 * j) for j in range(8 + si % 5)]
            p += [api, pool.native(f"{kern}.cubin", 0x100, KIND_KERNEL, kern)]
            sites.append(p)
            site_kernel.append(kern_ix[kern])
            weight.append(w * float(np.exp(0.5 * rng.standard_normal())))
    keys, labels, paths = pool.finalize(sites)
    off, frames = _pack_sites(paths)
    ns = len(paths)
    # per-kernel PC tables: code size U[64,4096], Zipf(1.2) over a random permutation of the
    # instructions, 2-4 dominant stall reasons per PC including const_mem_miss / math_dep.
    kern_off = [0]
    pc_thr, pc_instr, stall_thr, stall_id = [], [], [], []
    for k in range(len(kern_names)):
        n = int(rng.integers(64, 4097))
        pr = 1.0 / np.arange(1, n + 1) ** 1.2
        cdf = np.cumsum(pr / pr.sum())
        thr = np.minimum((cdf * 2**31).astype(np.int64), 2**31 - 1).astype(np.uint32)
        thr = np.maximum.accumulate(thr)
        pc_thr.append(thr)  # entry n-1 unused by the search (upper bound = n-1)
        pc_instr.append(rng.permutation(n).astype(np.uint32))
        for _ in range(n):
            nd = int(rng.integers(2, 5))
            ch = list(rng.choice(N_STALL, size=nd, replace=False))
            if rng.random() < 0.3 and 7 not in ch:
                ch[0] = 7
            if rng.random() < 0.4 and 3 not in ch:
                ch[-1] = 3
            w = rng.dirichlet(np.ones(nd))
            c = np.cumsum(w)[:-1]
            t = np.full(3, 0xFFFFFFFF, np.uint32)
            t[: nd - 1] = np.minimum((c * 2**31).astype(np.int64), 2**31 - 1)
            ids = np.zeros(4, np.uint8)
            ids[:nd] = ch
            stall_thr.append(t)
            stall_id.append(ids)
        kern_off.append(kern_off[-1] + n)
    # launch run lengths: proportional to launch duration (site weight), jitter +-25 %,
    # scaled so that the total is exactly n_samples
    wt = np.asarray(weight)
    site_len = wt / wt.sum() * ns * (n_samples / n_launch)
    from .rng import rnd_np
    jit = 750 + (rnd_np(seed, 15, np.arange(n_launch, dtype=np.uint64)) % np.uint64(501)).astype(np.int64)
    lens = np.maximum(1, (site_len[np.arange(n_launch) % ns] * jit / 1000).astype(np.int64))
    lens = np.maximum(1, lens * n_samples // int(lens.sum()))
    rem = n_samples - int(lens.sum())
    lens[:rem] += 1  # 0 <= rem < n_launch + n_launch (floor losses + the max(1) floor)
    lens[-1] += n_samples - int(lens.sum())
    assert lens.min() >= 1 and int(lens.sum()) == n_samples
    launch_off = np.zeros(n_launch + 1, np.uint64)
    launch_off[1:] = np.cumsum(lens).astype(np.uint64)
    base = (np.asarray(weight) * 5_000).astype(np.uint64) + 2000
    return Program(name="cfg3", seed=seed, mode=0, site_off=off, site_frames=frames, pool_keys=keys,
                   labels=labels, strings=pool.strings, trunc_permille=0, rec_permille=0, max_depth=1024,
                   empty_mod=0, empty_rem=0, force_record=2**63, force_site=0, site_rec_k=None,
                   rec_pos=0, rec_a=0, rec_b=0, dyn_per100k=0, dyn_min=0, dyn_max=0,
                   met_kind=3, n_metrics=2, site_base_ns=base, site_warps=None, site_smem=None,
                   default_records=n_launch,
                   pc=dict(n_launch=n_launch, n_sites=ns, launch_off=launch_off,
                           site_kernel=np.asarray(site_kernel, np.uint32),
                           kern_off=np.asarray(kern_off, np.uint32), pc_thr=np.concatenate(pc_thr),
                           pc_instr=np.concatenate(pc_instr), stall_thr=np.concatenate(stall_thr),
                           stall_id=np.concatenate(stall_id), n_stall=N_STALL, kern_names=kern_names))


# ------------------------------------------------------------------------------------------
# Config 4: JAX-compiled-graph-shaped, deep recursion (SURVEY §8(d) cfg 4)
# ------------------------------------------------------------------------------------------
def config4(seed: int = 4, n_exe: int = 16, leaves=(500, 5001), n_records: int = 200_000_000) -> Program:
    rng = np.random.default_rng(seed)
    pool = Pool()
    rec_a = pool.py("jax/_src/tree_util.py", 1023, "tree_map")
    rec_b = pool.py("jax/_src/tree_util.py", 1031, "<lambda>")
    pjit = [pool.native("libjax_pjit.so", 0x10000 + 0x80 * i) for i in range(int(rng.integers(10, 21)))]
    api = pool.native("libcuda.so", 0x2F00, KIND_API, "cuLaunchKernel")
    sites, rec_k = [], []
    for e in range(n_exe):
        pre = [pool.py(f"exe{e}.py", 10 + 3 * i, f"fn{i}") for i in range(int(rng.integers(6, 21)))]
        thunk = [pool.native("libxla_runtime.so", 0x40000 * (1 + e % 4) + 0x40 * i) for i in range(int(rng.integers(4, 11)))]
        nl = int(rng.integers(*leaves))
        first_rec = True
        for j in range(nl):
            p = pre + pjit + thunk + [pool.native(f"xla_exe{e}.so", 0x10 * j, KIND_API, f"thunk_{j}"), api,
                                      pool.native(f"exe{e}.cubin", 0x100 * j, KIND_KERNEL, f"fusion.{j}")]
            sites.append(p)
            if rng.random() < 0.05 or (first_rec and j == nl - 1):
                target = 256 if first_rec else int(rng.integers(64, 257))
                first_rec = False
                rec_k.append(max(0, target - len(p)))
            else:
                rec_k.append(0)
    keys, labels, paths = pool.finalize(sites)
    # recursion frames after remap
    rank = {k: i for i, k in enumerate(map(tuple, keys.tolist()))}
    ra, rb = rank[tuple(pool.keys[rec_a])], rank[tuple(pool.keys[rec_b])]
    off, frames = _pack_sites(paths)
    n = len(paths)
    base = np.maximum(500, np.exp(np.log(8_000.0) + 1.0 * rng.standard_normal(n))).astype(np.uint64)
    return Program(name="cfg4", seed=seed, mode=0, site_off=off, site_frames=frames, pool_keys=keys,
                   labels=labels, strings=pool.strings, trunc_permille=0, rec_permille=0, max_depth=1024,
                   empty_mod=0, empty_rem=0, force_record=2**63, force_site=0,
                   site_rec_k=np.asarray(rec_k, np.uint32), rec_pos=4, rec_a=ra, rec_b=rb,
                   dyn_per100k=100, dyn_min=64, dyn_max=256,
                   met_kind=3, n_metrics=2, site_base_ns=base, site_warps=None, site_smem=None,
                   default_records=n_records)


# ------------------------------------------------------------------------------------------
# Config 5: DDP-style shards of the config-2 program (SURVEY §8(d) cfg 5)
# ------------------------------------------------------------------------------------------
def config5(shard: int, seed_base: int = 50) -> Program:
    seed = seed_base + shard
    rng = np.random.default_rng(2)  # same program on every rank ...
    pool = Pool()
    sites = _resnet_sites(pool, rng, local_tag=shard)  # ... plus 5 % rank-local frames
    keys, labels, paths = pool.finalize(sites)
    off, frames = _pack_sites(paths)
    n = len(paths)
    r2 = np.random.default_rng(2)
    base = np.maximum(1000, np.exp(np.log(20_000.0) + 1.2 * r2.standard_normal(n))).astype(np.uint64)
    return Program(name=f"cfg5.{shard}", seed=seed, mode=0, site_off=off, site_frames=frames, pool_keys=keys,
                   labels=labels, strings=pool.strings, trunc_permille=0, rec_permille=0, max_depth=1024,
                   empty_mod=0, empty_rem=0, force_record=2**63, force_site=0, site_rec_k=None,
                   rec_pos=0, rec_a=0, rec_b=0, dyn_per100k=0, dyn_min=0, dyn_max=0,
                   met_kind=3, n_metrics=2, site_base_ns=base, site_warps=None, site_smem=None,
                   default_records=125_000_000)


def program(cfg: int, **kw) -> Program:
    if cfg == 5:
        return config5(**({"shard": 0} | kw))
    return {1: config1, 2: config2, 3: config3, 4: config4}[cfg](**kw)
