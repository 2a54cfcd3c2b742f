#!/usr/bin/env python
"""bench.py -- COMET fused MoE layer forward on B200 (BASELINE.json metric).

Metric: MoE layer forward latency in ms (max over ranks), lower is better,
and its fraction of the roofline.  Workload (BASELINE.json configs[1]):
Mixtral-8x7B MoE layer (E=8, top-2, N=4096, K=14336), bf16, 8192 tokens,
EP = number of GPUs (N=1 -> EP=1, the largest config that fits one GPU).
A step is one full layer forward of every rank: GPU index build from the
router output, dispatch (local HBM rows + NVLink pulls), fused GroupGEMM FC1
+ activation, fused GroupGEMM FC2 + top-k combine (+ remote combine).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

``value``: tokens already resident in HBM (the symmetric token buffer, where
the previous layer would have written them).  ``e2e``: the same forward
through the public per-rank API with HOST (pinned) buffers -- the tokens and
the router output cross PCIe to the GPU and the result back inside the timed
region (one GPU: the zero-copy forward, dispatch CTAs read the tokens from
pinned host memory and the fused combine writes the output there; multi-GPU:
copy, forward, copy).
``--impl reference`` times the reference algorithm on the host cores (the
numpy oracle port; the reference package itself is pure Python and cannot
run a Mixtral layer in bounded time) on a bounded token sample per step,
extrapolated to the full workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPES = {  # E, topk, N, K, tp
    "mixtral-8x7b": (8, 2, 4096, 14336, 1),
    "phi-3.5-moe": (16, 2, 4096, 6400, 2),
    "qwen2-style": (64, 8, 3584, 2560, 1),
}
BF16_PEAK_TFLOPS_FALLBACK = 1590.0
HBM_PEAK_GBS_FALLBACK = 6650.0
NVLINK_GBS = 900.0


def load_peaks():
    """(burst TF/s, sustained TF/s, HBM GB/s, source) from MEASURED_PEAKS.json."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return (float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)")
    except Exception:
        return BF16_PEAK_TFLOPS_FALLBACK, 1400.0, HBM_PEAK_GBS_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.lines, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def wait_started(self, timeout: float = 5.0):
        """Block until nvidia-smi produced its first sample, so the timed
        region is covered by samples."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sms)}


def dist_setup(gpus: int):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    from paper_2502_19811_b200.distributed import local_device
    local = local_device()  # LOCAL_RANK (COMET_SAME_DEVICE=1: every rank on GPU 0, test mode)
    if world != gpus:
        raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}")
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("COMET_DIST_BACKEND", "nccl")  # gloo: ranks sharing one GPU (test mode)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def cpu_reference_sample(model, routing, sample_tokens: int, steps: int, warmup: int):
    """Reference algorithm (oracle.moe_oracle.layer_forward: execute_naive
    restated with one GEMM pair per expert) on the host cores, fp32, over the
    first ``sample_tokens`` tokens; returns (ms per full-workload step, info)."""
    import numpy as np
    from oracle import moe_oracle as O
    rng = np.random.default_rng(11)
    w0 = rng.standard_normal((model.E, model.N, model.K), dtype=np.float32) / np.float32(math.sqrt(model.N))
    w1 = rng.standard_normal((model.E, model.K, model.N), dtype=np.float32) / np.float32(math.sqrt(model.N))
    x = rng.standard_normal((sample_tokens, model.N), dtype=np.float32)
    ex = routing.as_array()[:sample_tokens]
    # every host core for the BLAS pool (torchrun exports OMP_NUM_THREADS=1 to
    # multi-rank jobs, which OpenBLAS would otherwise honour)
    import contextlib
    limits, threads = contextlib.nullcontext(), os.cpu_count()
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        n_host = len(os.sched_getaffinity(0))
        limits = threadpool_limits(limits=n_host, user_api="blas")
        threads = max([i["num_threads"] for i in threadpool_info() if i.get("user_api") == "blas"] or [n_host])
    except Exception:
        pass
    with limits:
        for _ in range(max(0, warmup)):
            O.layer_forward(x, w0, w1, ex, dtype=np.float32)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            O.layer_forward(x, w0, w1, ex, dtype=np.float32)
            times.append(time.perf_counter() - t0)
    scale = routing.workload.M / sample_tokens
    ms = statistics.median(times) * 1e3 * scale
    try:
        import torch
        torch_threads = torch.get_num_threads()
    except Exception:
        torch_threads = None
    return ms, {"cores": os.cpu_count(), "threads": threads, "torch_threads": torch_threads,
                "sample": f"{sample_tokens} of {routing.workload.M} tokens (all experts, full N/K), fp32 numpy "
                          f"(OpenBLAS), median of {steps} steps, scaled x{scale:g} to the full workload"}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    from paper_2502_19811_b200 import ModelConfig, ParallelSpec, WorkloadSpec, build_routing
    E, topk, N, K, tp = SHAPES[args.shape]
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    ep = max(1, args.gpus // tp) if args.gpus >= tp else 1
    routing = build_routing(model, ParallelSpec(tp=1, ep=1), WorkloadSpec(M=args.M, seed=0, std=args.std))
    ms, info = cpu_reference_sample(model, routing, args.cpu_sample, args.steps, args.warmup)
    out = {
        "impl": "reference", "metric": "moe_layer_fwd_latency", "value": round(ms, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, model, ep, tp),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": info["threads"], "kind": "port",
                         "sample": info["sample"], "host_cpu_count": info["cores"], "blas_threads": info["threads"],
                         "torch_threads": info["torch_threads"]},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def workload_config(args, model, ep, tp):
    return {"workload": f"{args.shape} MoE layer forward, {args.M} tokens, EP={ep} x TP={tp}, routing std "
                        f"{args.std} (build_routing seed 0), random-init bf16 weights",
            "tokens": args.M, "experts": model.E, "topk": model.topk, "embed": model.N, "hidden": model.K,
            "ep": ep, "tp": tp, "std": args.std,
            "l2": "inputs larger than L2 (expert weights + token rows >> 126 MB)"}


def rank_weights_random(model, parallel, rank, device):
    """Random-init bf16 weights of this rank's experts only (N(0,1)/sqrt(N))."""
    import torch
    from paper_2502_19811_b200.executor import RankWeights, _ceil
    e_per = model.E // parallel.ep
    kl = model.K // parallel.tp
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    n_pad, k_pad = _ceil(model.N, 64), _ceil(kl, 64)
    w0t = torch.zeros(e_per, k_pad, n_pad, dtype=torch.bfloat16, device=device)
    w1t = torch.zeros(e_per, n_pad, k_pad, dtype=torch.bfloat16, device=device)
    s = 1.0 / math.sqrt(model.N)
    for e in range(e_per):
        w0t[e, :kl, :model.N] = (torch.randn(kl, model.N, device=device, generator=g) * s).to(torch.bfloat16)
        w1t[e, :model.N, :kl] = (torch.randn(model.N, kl, device=device, generator=g) * s).to(torch.bfloat16)
    return RankWeights(w0t, w1t)


def run_ours(args):
    import numpy as np
    import torch
    rank, world, local = dist_setup(args.gpus)
    from paper_2502_19811_b200 import (LayerKnobs, ModelConfig, MoELayer, ParallelSpec, WorkloadSpec,
                                       build_routing, distributed)
    from paper_2502_19811_b200.executor import index_flags
    E, topk, N, K, tp = SHAPES[args.shape]
    if world % tp:
        tp = 1
    ep = world // tp
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec(tp=tp, ep=ep)
    routing = build_routing(model, par, WorkloadSpec(M=args.M, seed=0, std=args.std))
    M = args.M
    dev = torch.device("cuda", local)
    # the dispatch CTAs must leave compute pairs: a reduced grid (COMET_GRID,
    # the ranks-sharing-one-GPU test mode) caps them at half of it
    grid = int(os.environ.get("COMET_GRID", torch.cuda.get_device_properties(local).multi_processor_count))
    n_comm0 = max(2, min(args.n_comm0, (grid // 2) // 2 * 2))
    knobs = LayerKnobs(n_comm0=n_comm0, n_comm1=args.n_comm1,
                       group0=args.group0, wave1=args.wave1)
    weights = rank_weights_random(model, par, rank, dev)
    layer = distributed.init_layer(model, par, M, weights, knobs=knobs) if world > 1 else \
        MoELayer(model, par, rank, M, weights, device=local, knobs=knobs)
    lo, hi = layer.token_range(M)
    g = torch.Generator(device="cuda").manual_seed(7 + rank)
    x_local = torch.randn(hi - lo, N, device=dev, generator=g).to(torch.bfloat16)
    ex = torch.from_numpy(routing.as_array().copy()).to(dev)
    y = torch.empty(hi - lo, layer.n_pad, dtype=torch.bfloat16, device=dev)
    layer.place_tokens(x_local, M)
    stream = torch.cuda.current_stream()

    def step():
        layer.run(ex, M, y)

    for _ in range(args.warmup):
        step()
    barrier(world)
    # ---- timed region (device events, max over ranks) ----
    with ClockSampler(local) as clk:
        clk.wait_started()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        s.record(stream)
        for _ in range(args.steps):
            step()
        e.record(stream)
        barrier(world)
        ms_local = s.elapsed_time(e) / args.steps
        # per-kernel durations (same stream), for the roofline of the dominant kernel
        from paper_2502_19811_b200.executor import fused_launch
        ctx = layer.ctx
        fused = fused_launch(world, layer.n_comm1())
        n_prof = max(3, min(args.steps, 10))
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_prof)]
        for i in range(n_prof):
            ctx.index_build(ex, M, flags=index_flags(world, layer.n_comm1()))
            ev[i][0].record(stream)
            if fused:
                ctx.layers(layer.weights.w0t, layer.weights.w1t, None, y, layer.act,
                           knobs.n_comm0 if world > 1 else 0, knobs.group0, knobs.wave1)
                ev[i][1].record(stream)
            else:
                ctx.layer0(layer.weights.w0t, layer.act, knobs.n_comm0 if world > 1 else 0, knobs.group0)
                ev[i][1].record(stream)
                ctx.layer1(layer.weights.w1t, None, y, layer.n_comm1(), knobs.wave1)
            ev[i][2].record(stream)
            ctx.combine_finish(y)
            ev[i][3].record(stream)
        barrier(world)
    ms = max_over_ranks(ms_local, world)
    t_l0 = statistics.median(ev[i][0].elapsed_time(ev[i][1]) for i in range(n_prof))
    t_l1 = statistics.median(ev[i][1].elapsed_time(ev[i][2]) for i in range(n_prof))
    meta = ctx.index_meta()
    rows = int(meta[0])
    kl = K // tp
    flops_layer = 2.0 * rows * N * kl  # one GEMM of the pair (algorithmic, unpadded rows)

    # ---- e2e: public per-rank API with host (pinned) buffers ----
    x_host = x_local.cpu().pin_memory()
    ex_host = torch.from_numpy(routing.as_array().copy()).pin_memory()
    y_host = torch.empty(hi - lo, N, dtype=torch.bfloat16).pin_memory()
    for _ in range(max(1, args.warmup // 2)):
        layer.forward_host(x_host, ex_host, out=y_host)
    barrier(world)
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record(stream)
    for _ in range(args.steps):
        layer.forward_host(x_host, ex_host, out=y_host)
    e2.record(stream)
    barrier(world)
    e2e_ms = max_over_ranks(s2.elapsed_time(e2) / args.steps, world)
    h2d = x_host.numel() * 2 + ex_host.numel() * 4
    d2h = y_host.numel() * 2

    # ---- unfused comparison path: NCCL all-to-all + cuBLAS grouped GEMM ----
    unfused_ms, unfused_error = None, None
    if tp == 1 and not args.no_unfused:
        # a comparison point, not the product: a failure (e.g. a collective
        # backend without all_to_all on CUDA tensors) is reported, not fatal
        try:
            from paper_2502_19811_b200.unfused import UnfusedLayer
            ul = UnfusedLayer(model, par, rank, layer.weights.w0t[:, :kl, :N].transpose(1, 2).contiguous(),
                              layer.weights.w1t[:, :N, :kl].transpose(1, 2).contiguous())
            for _ in range(3):
                ul.forward(x_local, ex, M=M)
            barrier(world)
            s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n_u = max(5, args.steps // 4)
            s3.record(stream)
            for _ in range(n_u):
                ul.forward(x_local, ex, M=M)
            e3.record(stream)
            barrier(world)
            unfused_ms = max_over_ranks(s3.elapsed_time(e3) / n_u, world)
            del ul
        except Exception as exc:  # noqa: BLE001
            unfused_error = repr(exc)[:200]

    # ---- roofline ----
    peak_burst, peak_sust, hbm_gbs, peak_src = load_peaks()
    rows_max = max_over_ranks(float(rows), world)
    t_flops_ms = 2 * (2.0 * rows_max * N * kl) / (peak_burst * 1e12) * 1e3
    t_flops_sust_ms = 2 * (2.0 * rows_max * N * kl) / (peak_sust * 1e12) * 1e3
    # the per-kernel timing runs right after the long timed loop: sustained peak
    peak_tf = peak_sust
    if fused:  # one launch runs both GEMMs (layer0 + layer1)
        dominant, t_dom, flops_dom = "layers", t_l0, 2 * flops_layer
    else:
        dominant = "layer1" if t_l1 >= t_l0 else "layer0"
        t_dom, flops_dom = max(t_l0, t_l1), flops_layer
    achieved_tf = flops_dom / (t_dom * 1e-3) / 1e12
    traffic = load_traffic(dominant)
    launches_per_step = (4 if fused else 5) - (0 if (world == 1 and knobs.n_comm1 == 0) else 1) + \
        (1 if world > 1 else 0)
    clocks = clk.summary()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cms, info = cpu_reference_sample(model, routing, args.cpu_sample, 3, 1)
        cpu = {"value": round(cms, 3), "unit": "ms", "cores": info["threads"], "kind": "port",
               "sample": info["sample"], "host_cpu_count": info["cores"], "blas_threads": info["threads"],
               "torch_threads": info["torch_threads"]}

    if rank == 0:
        out = {
            "metric": "moe_layer_fwd_latency", "value": round(ms, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens, random-init weights", "config": workload_config(args, model, ep, tp),
            "pct_of_roofline": round(100.0 * t_flops_ms / ms, 2),
            "roofline_ms": round(t_flops_ms, 4),
            "pct_of_roofline_sustained": round(100.0 * t_flops_sust_ms / ms, 2),
            "pct_of_roofline_spec_2250tf": round(100.0 * t_flops_ms * peak_burst / 2250.0 / ms, 2),
            "roofline_note": "roofline_ms = 2 GEMMs x 2*rows*N*K/tp FLOP at the measured burst bf16 peak "
                             "(BASELINE.md); pct_of_roofline_sustained uses the measured sustained peak",
            "roofline": {"bound": "tensor",
                         "kernel": "moe_layer_kernel (" + ("layer0 + layer1, one launch" if fused else dominant) + ")",
                         "achieved": round(achieved_tf, 1), "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": round(achieved_tf / peak_tf, 4), "traffic": traffic,
                         "peak_source": peak_src + ", sustained figure (kernel timed inside a long step)",
                         "flops_per_launch": flops_dom, "ms_per_launch": round(t_dom, 4)},
            "kernels_ms": ({"layers": round(t_l0, 4)} if fused else {"layer0": round(t_l0, 4), "layer1": round(t_l1, 4)}),
            "unfused_ms": None if unfused_ms is None else round(unfused_ms, 4),
            "speedup_vs_unfused": None if unfused_ms is None else round(unfused_ms / ms, 3),
            **({"unfused_error": unfused_error} if unfused_error else {}),
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": ("MoELayer.forward_host -> comet_forward_zerocopy (pinned host buffers read / written "
                             "over PCIe by the layer kernel)" if world == 1 and os.environ.get("COMET_E2E", "zerocopy")
                             == "zerocopy" else "MoELayer.forward_host (H2D, forward, D2H)")},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "knobs": {"n_comm0": knobs.n_comm0, "n_comm1": knobs.n_comm1, "group0": knobs.group0,
                      "wave1": knobs.wave1},
        }
        if cpu is not None:
            out["cpu_baseline"] = cpu
        print(json.dumps(out))
    layer.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def load_traffic(dominant):
    """dram read+write bytes per launch of the dominant kernel from the
    committed ncu --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_layer_summary.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data[dominant]["dram_bytes"]
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--shape", choices=sorted(SHAPES), default="mixtral-8x7b")
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--std", type=float, default=0.0)
    ap.add_argument("--n-comm0", type=int, default=None,
                    help="layer0 dispatch CTAs (default 8 per rank of the group, max 64: measured best at EP=2/4/8)")
    ap.add_argument("--n-comm1", type=int, default=0)
    ap.add_argument("--group0", type=int, default=None,
                    help="layer0 pair-group raster (default: 8 at EP=1 and EP>=8, 4 at EP=2/4; measured)")
    ap.add_argument("--wave1", type=int, default=4)
    ap.add_argument("--cpu-sample", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unfused", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.n_comm0 is None:
        # measured (gpu_run106.sh, tools/matrix.py): EP=2 16 vs 64 CTAs
        # 1.396 vs 1.409 ms, EP=4 32 vs 64 0.734 vs 0.742 ms, EP=8 64 best
        args.n_comm0 = min(64, 8 * args.gpus)
    if args.group0 is None:
        # measured (tools/gpu_runs/gpu_run105.sh, 3 reps): 8-pair groups win at
        # EP=1 and EP=8 (all 8 pairs of a rank in one group: 0.423 -> 0.417 ms),
        # 4-pair groups at EP=2/4 (1.386 vs 1.404, 0.737 vs 0.744 ms)
        args.group0 = 8 if args.gpus == 1 or args.gpus >= 8 else 4
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
