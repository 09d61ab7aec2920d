#!/usr/bin/env python
"""Benchmark: TP transformer fwd+bwd tokens/s on 1/2/4/8 B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): BERT-large DistributedTransformer — 24 layers,
hidden 1024, 16 heads x 64, FFN 4096, seq 512, post-LN, GeLU(erf), dropout 0.1,
bf16 storage / fp32 accumulate — forward + backward, speed mode, TP degree =
number of GPUs, TP across data-parallel ranks with 8 sequences per GPU (weak
scaling: the gathered GEMM M is 4096*T, per-GPU work fixed).  Synthetic
hidden states and random-init weights (no dataset / checkpoint).

One JSON line on rank 0:
  value      whole-job tokens/s, inputs resident in HBM, device-timed (CUDA events, max over ranks)
  e2e        same metric through the public API with pinned-host inputs copied in and the
             loss read back every step
  roofline   the dominant kernel family (smpk tcgen05 GEMMs): algorithmic FLOPs / their device time
             (CUPTI records of graph replays, each launch charged from max(start, end of its stream
             predecessor) -- programmatic dependent launch starts records early)
  cpu_baseline  the CPU oracle (oracle/tp.py, torch fp32 on the host cores) on a bounded sample
``--impl reference`` times only the CPU reference path (the reference has no TP
code; its algorithm is restated in oracle/).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "TP transformer fwd+bwd tokens/sec at 1/2/4/8 B200; % of bf16 tensor-core peak"
UNIT = "tokens/s"
CFG = dict(num_layers=24, num_attention_heads=16, attention_head_size=64, hidden_size=1024, intermediate_size=4096,
           attention_dropout_prob=0.1, hidden_dropout_prob=0.1, activation="gelu", layernorm_epsilon=1e-5,
           pre_layernorm=False, post_layernorm=True)
SEQ = 512
BATCH_PER_GPU = 8
# BASELINE.json configs[2] (the north_star's ">= 60% of peak" target): GPT-3 1.3B with the
# vocab-parallel embedding, tied LM head and vocab-parallel cross-entropy; 8 sequences of 2048
# tokens per GPU (the paper's prescaled TP=8 batch, is 8 sequences per step)
GPT_CFG = dict(num_layers=24, num_attention_heads=16, attention_head_size=128, hidden_size=2048,
               intermediate_size=8192, vocab_size=50257, num_positions=2048, attention_dropout_prob=0.1,
               hidden_dropout_prob=0.1, activation="gelu_tanh", layernorm_epsilon=1e-5, causal_mask_size=2048,
               pre_layernorm=True, post_layernorm=False)
GPT_SEQ = 2048
GPT_BATCH_PER_GPU = 8


def flops_per_token_layer(H=1024, s=SEQ, causal=False):
    """fwd+bwd algorithmic FLOPs per token per layer: 72 H^2 + 12 s H (non-causal)."""
    return 72 * H * H + (6 if causal else 12) * s * H


def flops_per_token(workload: str) -> float:
    """fwd+bwd algorithmic FLOPs per token of the whole model: BERT-large 1.963 GFLOP
    (24 layers); GPT-1.3B 8.469 GFLOP (24 causal layers + the tied LM head's 6 H V)."""
    if workload == "gpt1.3b":
        c = GPT_CFG
        return (c["num_layers"] * flops_per_token_layer(c["hidden_size"], GPT_SEQ, causal=True)
                + 6 * c["hidden_size"] * c["vocab_size"])
    return flops_per_token_layer() * CFG["num_layers"]


def gemm_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per GEMM launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            return json.load(f)["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [v for v in sm if mx and v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (the oracle restatement; the reference has no TP code)
# ---------------------------------------------------------------------------

def cpu_reference_sample(max_seconds=15.0, min_iters=2, workload="bert-large"):
    """The CPU oracle (oracle/tp.py, torch fp32 on all host cores) on a bounded sample: one layer
    fwd+bwd on one sequence (BERT-large: 512 tokens; GPT-1.3B: 2048 causal tokens, plus the tied
    LM head + CE on the same tokens), scaled to the whole model's per-token cost.
    Returns (tokens/s of the whole model, threads, seconds, iterations)."""
    from oracle import tp
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    gpt = workload == "gpt1.3b"
    c = GPT_CFG if gpt else CFG
    seq = GPT_SEQ if gpt else SEQ
    cfg = tp.LayerConfig(num_attention_heads=c["num_attention_heads"], attention_head_size=c["attention_head_size"],
                         hidden_size=c["hidden_size"], intermediate_size=c["intermediate_size"],
                         attention_dropout_prob=0.1, hidden_dropout_prob=0.1, activation=c["activation"],
                         causal_mask_size=seq if gpt else None, pre_layernorm=c["pre_layernorm"],
                         post_layernorm=c["post_layernorm"])
    p = {k: v.requires_grad_(True) for k, v in tp.init_layer_params(cfg, 1, dtype=torch.float32).items()}
    H = c["hidden_size"]
    x = torch.randn(1, seq, H, requires_grad=True)
    dy = torch.randn(1, seq, H)
    dctx = tp.DropoutCtx(seed=0, layer=0, torch_rng=True)
    E = (torch.randn(c["vocab_size"], H) * 0.02).requires_grad_(True) if gpt else None
    tgt = torch.randint(0, c["vocab_size"], (seq,)) if gpt else None

    def one():
        tp.transformer_layer_ref(x, p, cfg, None, dctx).backward(dy)

    def head():
        logits = x.detach().reshape(seq, H) @ E.t()
        tp.cross_entropy_ref(logits, tgt, c["vocab_size"]).sum().backward()

    one()  # untimed warm-up
    t0 = time.perf_counter()
    it = 0
    while it < min_iters or (time.perf_counter() - t0 < max_seconds and it < 50):
        one()
        it += 1
    dt = time.perf_counter() - t0
    sec_per_tok = dt / (seq * it) * c["num_layers"]
    if gpt:
        head()
        t1 = time.perf_counter()
        head()
        sec_per_tok += (time.perf_counter() - t1) / seq
        dt += time.perf_counter() - t1
    return 1.0 / sec_per_tok, threads, dt, it


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cpu_sample_text(workload, it, dt):
    reps = f" x {it} iters ({dt:.1f} s)" if it else ""
    if workload == "gpt1.3b":
        return (f"1 GPT-1.3B layer fwd+bwd{reps} on 1x{GPT_SEQ} causal tokens + the tied LM head and CE on the "
                f"same tokens, torch fp32 CPU oracle (oracle/tp.py), scaled to 24 layers + head")
    return (f"1 BERT-large layer fwd+bwd{reps} on 1x{SEQ} tokens, torch fp32 CPU oracle (oracle/tp.py), "
            f"scaled to the 24-layer stack")


def _config(workload, world, args):
    if workload == "gpt1.3b":
        return {"workload": "gpt3-1.3b-24L-vocab-parallel-lm (BASELINE.json configs[2] shapes)",
                "model": "GPT-3 1.3B: 24L H2048 16x128 FFN8192 causal pre-LN gelu_tanh dropout0.1, vocab-parallel "
                         "embedding V=50257->50304 + tied LM head + vocab-parallel CE",
                "global_batch": GPT_BATCH_PER_GPU * world, "per_gpu_batch": GPT_BATCH_PER_GPU, "seq_len": GPT_SEQ,
                "parallelism": f"tp{world} ({args.optimize} mode, TP across DP ranks)",
                "tp_comm": args.tp_comm, "l2": "inputs larger than L2 (logits alone 1.6 GB per step)"}
    return {"workload": "bert-large-24L-tp-layer-stack (BASELINE.json configs[1])",
            "model": "BERT-large DistributedTransformer 24L H1024 16x64 FFN4096 post-LN gelu dropout0.1",
            "global_batch": BATCH_PER_GPU * world, "per_gpu_batch": BATCH_PER_GPU, "seq_len": SEQ,
            "parallelism": f"tp{world} ({args.optimize} mode, TP across DP ranks)",
            "tp_comm": args.tp_comm, "l2": "inputs larger than L2 (saved activations ~6 GB per step)"}


def run_reference(args, rank):
    if rank != 0:
        return
    steps = []
    for i in range(args.warmup + args.steps):
        v, threads, dt, it = cpu_reference_sample(max_seconds=args.ref_seconds, min_iters=1,
                                                  workload=args.workload)
        if i >= args.warmup:
            steps.append(v)
    value = statistics.median(steps)
    sample = _cpu_sample_text(args.workload, None, None) + f"; {cpu_model()}"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": _config(args.workload, args.gpus, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU path
# ---------------------------------------------------------------------------

def barrier():
    if dist.is_initialized():
        dist.barrier()


def max_over_ranks(v: float) -> float:
    if not dist.is_initialized():
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def exclusive_us(events) -> list:
    """(event, exclusive device us) for CUDA kernel records: the span from max(start, end of the
    previous kernel on the same stream) to end.  With programmatic dependent launch a kernel's
    CTAs are scheduled (and its CUPTI record starts) while its predecessor still runs; its own
    work begins only when the predecessor ends, so the overlap is not charged to it twice."""
    cuda = [ev for ev in events if ev.device_type == torch.autograd.DeviceType.CUDA]
    last_end = {}
    out = []
    for ev in sorted(cuda, key=lambda e: e.time_range.start):
        sid = getattr(ev, "device_resource_id", -1)
        t0, t1 = ev.time_range.start, ev.time_range.end
        begin = max(t0, last_end.get(sid, t0))
        out.append((ev, max(t1 - begin, 0.0)))
        last_end[sid] = max(t1, last_end.get(sid, t1))
    return out


def kernel_ms_per_step(run, name_part: str, steps: int = 3) -> float:
    """Device time (CUPTI kernel records, exclusive per stream) per step of the kernels whose name
    contains name_part."""
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            run()
        torch.cuda.synchronize()
    us = sum(d for ev, d in exclusive_us(prof.events()) if name_part in ev.name)
    return us / steps / 1e3


def trace_kernels(run, path_prefix: str, rank: int, steps: int = 2) -> None:
    """Diagnostics only (never the bench value): CUPTI kernel trace of `steps` steps,
    aggregated per kernel name, written to <prefix>_rank<r>.txt."""
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            run()
        torch.cuda.synchronize()
    agg = {}
    for ev, us in exclusive_us(prof.events()):  # exclusive per stream (see exclusive_us)
        a = agg.setdefault(ev.name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    seq = [(ev.name, ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total,
            ev.time_range.start, getattr(ev, "device_resource_id", -1))
           for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
    first = seq[:len(seq) // steps]
    t0 = min(t for _, _, t, _ in first) if first else 0
    with open(f"{path_prefix}_rank{rank}_seq.txt", "w") as f:  # the first step: duration, start, stream
        for name, us, t, sid in sorted(first, key=lambda e: e[2]):
            f.write(f"{us:9.1f} {t - t0:10.1f} {sid:4d}  {name[:100]}\n")
    with open(f"{path_prefix}_rank{rank}.txt", "w") as f:
        f.write(f"# {steps} steps, total kernel time {tot / steps / 1e3:.3f} ms/step\n")
        for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{us / steps:10.1f} us/step {n // steps:5d} launches/step  {us / n:8.2f} us/launch  {name[:150]}\n")


STATE_OVERLAP: dict = {}


def run_gpu(args, rank, world, local):
    import paper_2111_05972_b200 as smp
    from paper_2111_05972_b200 import _lib, kernels

    torch.cuda.set_device(local)
    smp.init({"tensor_parallel_degree": world, "optimize": args.optimize, "seed": 1234, "tp_comm": args.tp_comm,
              "tp_rs": args.tp_rs, "tp_exchange": args.tp_exchange,
              "tp_overlap_sms": args.tp_overlap_sms if args.tp_overlap_sms >= 0 else (96 if world >= 4 else 0)})
    STATE_OVERLAP["sms"] = smp.state.STATE.config.get("tp_overlap_sms", 0) if world > 1 else 0
    torch.manual_seed(1000 + rank)
    gpt = args.workload == "gpt1.3b"
    if gpt:
        # token ids in, per-token CE out: the LM objective (mean over valid tokens) is backpropagated
        model = smp.nn.DistributedTransformerLMHead(**GPT_CFG)
        B, s, H = GPT_BATCH_PER_GPU, GPT_SEQ, GPT_CFG["hidden_size"]
        g = torch.Generator().manual_seed(7 + rank)
        ids_h = torch.randint(0, GPT_CFG["vocab_size"], (B, s), generator=g)
        lab_h = torch.full_like(ids_h, -100)
        lab_h[:, :-1] = ids_h[:, 1:]  # next-token targets of uniform-random tokens
        x, dy = ids_h.cuda(), lab_h.cuda()
    else:
        model = smp.nn.DistributedTransformer(**CFG)
        B, s, H = BATCH_PER_GPU, SEQ, CFG["hidden_size"]
        x = torch.randn(B, s, H, device="cuda", dtype=torch.bfloat16, requires_grad=True)
        dy = torch.randn(B, s, H, device="cuda", dtype=torch.bfloat16)
    model.train()
    n_valid = B * (s - 1)

    def step(inp, grad):
        for prm in model.parameters():
            prm.grad = None
        if gpt:
            loss = model(inp, labels=grad).sum() / n_valid
            loss.backward()
            return loss
        y = model(inp)
        y.backward(grad)
        return y

    run = lambda: step(x, dy)  # noqa: E731
    if args.graph:
        # capture the whole fwd+bwd step (every smpk launch + NCCL) in one CUDA graph:
        # removes the host launch path from the step
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(max(args.warmup, 2)):
                step(x, dy)
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        launches_g0 = _lib.launch_count
        kernels.PROFILER = graph_prof = kernels.GemmProfiler(count_only=True)  # GEMM FLOPs of one step
        with torch.cuda.graph(graph):
            static_y = step(x, dy)
        kernels.PROFILER = None
        graph_launches = _lib.launch_count - launches_g0
        run = graph.replay
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    barrier()

    # -------- timed region: inputs resident in HBM (activations >> 126 MB L2)
    sampler = ClockSampler(local)
    sampler.start()
    kernels.PROFILER = None if args.graph else kernels.GemmProfiler()
    launches0 = _lib.launch_count
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = (_lib.launch_count - launches0) // args.steps
    prof, kernels.PROFILER = kernels.PROFILER, None
    gemm_flops, gemm_ms, gemm_launches = prof.flops_and_ms() if prof else (0.0, 0.0, 0)
    if args.graph:
        # Event brackets cannot sit inside the replayed graph without adding event-record nodes
        # (measured: +~10 us per GEMM), so the GEMM durations come from the device-side kernel
        # records (CUPTI) of replays of the same graph right after the timed region.
        launches = graph_launches
        gemm_ms = kernel_ms_per_step(run, "gemm_bf16_tcgen05", steps=3)
        gemm_launches = len(graph_prof.records)
        gemm_flops, gemm_ms, gemm_launches = (graph_prof.flops() * args.steps, gemm_ms * args.steps,
                                              gemm_launches * args.steps)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    tokens_step = B * s * world
    if args.trace:
        trace_kernels(run, args.trace, rank)
    value = tokens_step / (ms / 1e3)

    # -------- e2e through the public API: pinned host input + upstream grad in, loss out
    if gpt:  # token ids + targets in, the mean loss out
        xh, dyh = ids_h.pin_memory(), lab_h.pin_memory()
    else:
        xh = torch.randn(B, s, H, dtype=torch.bfloat16).pin_memory()
        dyh = torch.randn(B, s, H, dtype=torch.bfloat16).pin_memory()
    lossh = torch.empty(1, dtype=torch.float32).pin_memory()
    xd = torch.empty_like(x)
    dyd = torch.empty_like(dy)

    # input pipeline of a training loop: step k+1's pinned host inputs are copied to a device
    # staging buffer on a copy stream while step k runs; step k+1 then starts with a device copy
    # into its inputs.  Every step's H2D copy is inside the timed region (the first one exposed).
    copy_stream = torch.cuda.Stream()
    stage = [(torch.empty_like(xd), torch.empty_like(dyd)) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def h2d(k):
        bx, bdy = stage[k % 2]
        copy_stream.wait_event(free[k % 2])  # the step that used this buffer copied it out
        with torch.cuda.stream(copy_stream):
            bx.copy_(xh, non_blocking=True)
            bdy.copy_(dyh, non_blocking=True)
            ready[k % 2].record(copy_stream)

    def e2e_step(k, n):
        if k + 1 < n:
            h2d(k + 1)
        main = torch.cuda.current_stream()
        main.wait_event(ready[k % 2])
        bx, bdy = stage[k % 2]
        if args.graph:
            with torch.no_grad():  # the graph's static input buffers
                x.copy_(bx)
                dy.copy_(bdy)
            free[k % 2].record(main)
            run()
            y, g = static_y, dy
        else:
            xd.copy_(bx)
            dyd.copy_(bdy)
            free[k % 2].record(main)
            y = step(xd if gpt else xd.detach().requires_grad_(True), dyd)
            g = dyd
        out = y.detach().float().reshape(1) if gpt else (y.detach().float() * g.float()).sum().reshape(1)
        lossh.copy_(out, non_blocking=True)

    h2d(0)
    e2e_step(0, 1)
    torch.cuda.synchronize()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    h2d(0)
    for k in range(args.steps):
        e2e_step(k, args.steps)
    t1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1) / args.steps)
    barrier()

    if rank != 0:
        return
    peaks, peak_kind = load_peaks()
    peak_sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    peak_burst = peaks["bf16_tflops"]
    # the roofline denominator follows the clocks the kernels actually ran at: a short bench at
    # the maximum SM clock is compared with the BURST peak (measured at max clock); only a run whose
    # median SM clock under load sat clearly below max uses the sustained figure
    at_max = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    peak_roof = peak_burst if (at_max or clocks.get("sm_mhz") is None) else peak_sus
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    flops_tok = flops_per_token(args.workload)
    model_tflops = value / world * flops_tok / 1e12  # per GPU
    cpu = None
    if not args.skip_cpu_baseline and world == 1:  # the CPU baseline is timed on rank 0 at N=1 only
        v, threads, dt, it = cpu_reference_sample(max_seconds=args.ref_seconds, workload=args.workload)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": _cpu_sample_text(args.workload, it, dt) + f"; {cpu_model()}"}
    cfg_line = _config(args.workload, world, args)
    cfg_line["tp_overlap_sms"] = STATE_OVERLAP.get("sms", 0)
    cfg_line["tp_exchange"] = args.tp_exchange
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": ("synthetic uniform-random token ids, random-init weights" if gpt else
                 "synthetic tokens' hidden states, random-init weights"),
        "config": cfg_line,
        "mfu": {"model_tflops_per_gpu": model_tflops, "flops_per_token": flops_tok,
                "frac_of_sustained": model_tflops / peak_sus, "frac_of_burst": model_tflops / peaks["bf16_tflops"],
                "peak_kind": peak_kind},
        "roofline": {"bound": "tensor", "kernel": "smpk gemm_bf16_tcgen05 (all GEMM launches of the step)",
                     "timing": ("CUPTI kernel records (exclusive per stream) of replays of the step graph" if args.graph
                                else "CUDA events around each GEMM launch (eager)"),
                     "achieved": achieved, "peak": peak_roof, "unit": "TFLOP/s", "frac": achieved / peak_roof,
                     "peak_kind": (f"{peak_kind} bf16_tflops (burst: SM clock at max during the timed region)"
                                   if peak_roof == peak_burst else
                                   f"{peak_kind} bf16_tflops_sustained (SM clock below max under load)"),
                     "frac_of_burst": achieved / peak_burst, "frac_of_sustained": achieved / peak_sus,
                     "launches_per_step": gemm_launches // args.steps,
                     "gemm_ms_per_step": gemm_ms / args.steps, "traffic": gemm_traffic(),
                     "traffic_unit": "DRAM bytes per GEMM launch (ncu, profiles/gemm_traffic.json)"},
        "cpu_baseline": cpu,
        "e2e": {"value": tokens_step / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 2 * xh.numel() * xh.element_size(), "d2h_bytes_per_step": 4,
                "input_pipeline": "pinned host -> device staging on a copy stream one step ahead (the first "
                                  "step's copy exposed), device copy into the step's inputs, loss read back"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="smpk", choices=["smpk", "reference"])
    ap.add_argument("--workload", default="bert-large", choices=["bert-large", "gpt1.3b"],
                    help="bert-large: BASELINE.json configs[1] (the metric's config, default); gpt1.3b: configs[2] "
                         "shapes (the north_star's >= 60%% of peak target) with embedding + LM head + CE")
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--graph", type=int, default=1, help="capture the step in a CUDA graph (1) or run eagerly (0)")
    ap.add_argument("--optimize", default="speed", choices=["speed", "memory"],
                    help="smp optimize mode of the TP layers (PAPER.md:763); the headline is speed")
    ap.add_argument("--tp-comm", default="peer", choices=["peer", "nccl"],
                    help="TP collectives: fused NVLink peer stores (default) or NCCL calls")
    ap.add_argument("--tp-exchange", default="barrier", choices=["overlap", "chunks", "barrier"],
                    help="peer exchanges: copy-engine mailboxes with two overlapped micro-batches, per-owner chunks "
                         "over the mailboxes, or SM pull/push behind one barrier per exchange")
    ap.add_argument("--tp-rs", default="pull", choices=["pull", "push"],
                    help="peer reduce-scatter: consumer pulls partials over NVLink, or GEMM epilogue pushes")
    ap.add_argument("--tp-overlap-sms", type=int, default=int(os.environ.get("SMPK_TP_OVERLAP_SMS", "-1")),
                    help="T>1: SMs for the backward weight-gradient GEMMs beside the exchange (0 = serial; "
                         "-1 = 96 at T >= 4, where it measured faster, else 0)")
    ap.add_argument("--trace", default="", help="diagnostics: write a per-kernel CUPTI trace summary to PREFIX_rankR.txt")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    run_gpu(args, rank, world, local)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
