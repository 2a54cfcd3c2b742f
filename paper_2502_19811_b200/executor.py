"""MoE layer execution: the reference's executor API on the B200 kernels.

Mirror of `pkg/src/moepipe/executor.py`.  ``ExpertWeights``,
``random_weights`` and the three entry points keep the reference's names,
argument meaning and error behaviour (executor.py:30-246):

* ``execute_naive(x, weights, routing, activation=None, combine_weights=None)``
* ``execute_scheduled(x, weights, routing, scheds0, scheds1, ...)``
* ``execute_tp_sharded(x, weights, routing, tp, ...)``

All three run the same fused GPU path -- index build, NVLink dispatch +
GroupGEMM FC1 + activation (layer0), GroupGEMM FC2 + top-k combine (layer1)
-- with every EP/TP rank of the routing's ``ParallelSpec`` emulated in this
process on one GPU (the reference simulates ranks in-process too; multi-GPU
deployments use ``MoELayer`` per rank, see ``distributed.py``).  Arithmetic
is bf16 in, fp32 accumulate, bf16 between the GEMMs: results match the
reference's fp64 oracle within the tolerance stated in DESIGN.md, not
bitwise.  There is no CPU fallback.

The per-rank form for real deployments is ``MoELayer`` (device tensors in,
device tensors out, no host synchronisation).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Union

import numpy as np

from . import _lib
from .config import ConfigurationError, ModelConfig, ParallelSpec
from .resolver import TileSchedule, validate_schedule
from .routing import RoutingTable

Activation = Optional[Union[str, Callable[[np.ndarray], np.ndarray]]]


@dataclass(frozen=True, eq=False)
class ExpertWeights:
    """``w0[e]`` (N, K) and ``w1[e]`` (K, N), stacked (ref executor.py:30-74).
    Identity-hashed so prepared device copies can be cached per instance."""

    w0: np.ndarray
    w1: np.ndarray

    def __post_init__(self) -> None:
        if self.w0.ndim != 3 or self.w1.ndim != 3:
            raise ConfigurationError("expert weights must be stacked [E, ., .] arrays")
        e0, n, k = self.w0.shape
        e1, k1, n1 = self.w1.shape
        if e0 != e1 or n != n1 or k != k1:
            raise ConfigurationError(f"inconsistent weight shapes {self.w0.shape} / {self.w1.shape}")

    @property
    def num_experts(self) -> int:
        return self.w0.shape[0]

    def check_model(self, model: ModelConfig) -> None:
        e, n, k = self.w0.shape
        if (e, n, k) != (model.E, model.N, model.K):
            raise ConfigurationError(
                f"weights shaped for (E={e}, N={n}, K={k}), model wants "
                f"(E={model.E}, N={model.N}, K={model.K})")

    def shard_along_k(self, tp: int) -> List["ExpertWeights"]:
        """``tp`` contiguous K shards; concatenation reconstructs the weights."""
        k = self.w0.shape[2]
        if k % tp != 0:
            raise ConfigurationError(f"K={k} is not divisible by tp={tp}")
        size = k // tp
        return [ExpertWeights(w0=self.w0[:, :, s * size:(s + 1) * size].copy(),
                              w1=self.w1[:, s * size:(s + 1) * size, :].copy()) for s in range(tp)]


def random_weights(model: ModelConfig, seed: int = 0) -> ExpertWeights:
    """N(0,1)/sqrt(N) weights, same PCG64 stream as the reference
    (executor.py:77-83)."""
    rng = np.random.default_rng(seed)
    scale = 1.0 / np.sqrt(model.N)
    w0 = rng.standard_normal((model.E, model.N, model.K)) * scale
    w1 = rng.standard_normal((model.E, model.K, model.N)) * scale
    return ExpertWeights(w0=w0, w1=w1)


def activation_code(activation: Activation) -> int:
    """Map the reference's activation hook (executor.py:86-90) to a fused
    epilogue.  Callables are recognised when they are the numpy function of
    a supported activation; anything else is rejected (no host fallback)."""
    if activation is None or isinstance(activation, str):
        key = activation.lower() if isinstance(activation, str) else None
        if key not in _lib.ACTIVATIONS:
            raise ConfigurationError(f"unsupported activation {activation!r}; "
                                     f"choose from {sorted(k for k in _lib.ACTIVATIONS if k)}")
        return _lib.ACTIVATIONS[key]
    if activation is np.tanh:
        return _lib.ACTIVATIONS["tanh"]
    name = getattr(activation, "comet_activation", None)
    if isinstance(name, str) and name in _lib.ACTIVATIONS:
        return _lib.ACTIVATIONS[name]
    raise ConfigurationError(
        f"activation {activation!r} has no fused GPU epilogue; pass one of "
        f"{sorted(k for k in _lib.ACTIVATIONS if k)} (or np.tanh)")


def _ceil(v: int, m: int) -> int:
    return -(-v // m) * m


# ---------------------------------------------------------------------------
# Per-rank layer (device tensors) -- the B200 form of the reference layer.
# ---------------------------------------------------------------------------

class RankWeights:
    """One rank's experts on the GPU: ``w0t [E_r, K_l, N]`` and
    ``w1t [E_r, N, K_l]`` bf16, K-major for TMA, zero-padded to multiples of
    64 (padding contributes exact zeros).  Built once, outside any timed
    region (the reference keeps fp64 [E, N, K] / [E, K, N])."""

    def __init__(self, w0t, w1t):
        self.w0t, self.w1t = w0t, w1t

    @classmethod
    def from_full(cls, w0, w1, model: ModelConfig, parallel: ParallelSpec, rank: int, device: int = 0):
        import torch
        e_per = model.E // parallel.ep
        e_lo = parallel.ep_group_of_rank(rank) * e_per
        kl = model.K // parallel.tp
        s = parallel.tp_index_of_rank(rank)
        n_pad, k_pad = _ceil(model.N, 64), _ceil(kl, 64)
        dev = torch.device("cuda", device)
        w0s = torch.as_tensor(np.asarray(w0[e_lo:e_lo + e_per, :, s * kl:(s + 1) * kl])) \
            if not isinstance(w0, torch.Tensor) else w0[e_lo:e_lo + e_per, :, s * kl:(s + 1) * kl]
        w1s = torch.as_tensor(np.asarray(w1[e_lo:e_lo + e_per, s * kl:(s + 1) * kl, :])) \
            if not isinstance(w1, torch.Tensor) else w1[e_lo:e_lo + e_per, s * kl:(s + 1) * kl, :]
        w0t = torch.zeros(e_per, k_pad, n_pad, dtype=torch.bfloat16, device=dev)
        w1t = torch.zeros(e_per, n_pad, k_pad, dtype=torch.bfloat16, device=dev)
        w0t[:, :kl, :model.N] = w0s.to(dev).transpose(1, 2).to(torch.bfloat16)
        w1t[:, :model.N, :kl] = w1s.to(dev).transpose(1, 2).to(torch.bfloat16)
        return cls(w0t, w1t)


@dataclass
class LayerKnobs:
    """Kernel knobs.  n_comm0/n_comm1 are the paper's communication-block
    counts n_c (simulator.py:45-65), chosen by ``assigner.select_split`` from
    measured timings; group0 / wave1 set the layer0 L2 grouping and the
    layer1 column-wave width."""

    n_comm0: int = 64
    n_comm1: int = 0
    group0: int = 4
    wave1: int = 4

    @classmethod
    def for_world(cls, world: int) -> "LayerKnobs":
        """Measured defaults (bench.py / tools/gpu_runs/gpu_run105-106.sh): 8
        dispatch CTAs per rank of the group (max 64); 8-pair layer0 groups at
        EP=1 and EP>=8, 4-pair groups at EP=2/4."""
        return cls(n_comm0=min(64, 8 * max(1, world)), group0=8 if world == 1 or world >= 8 else 4)


class MoELayer:
    """One rank's fused MoE layer forward on its GPU.

    ``forward(x_local, experts, combine_w=None)``: ``x_local`` bf16
    ``[M_r, N]`` (this rank's contiguous tokens, routing.py:97-104),
    ``experts`` int32 ``[M, topk]`` global router output (ascending per
    token), ``combine_w`` fp32 ``[M, topk]`` or None.  Returns bf16 ``[M_r, N]``.
    Asynchronous on the current stream.  Multi-GPU: call ``connect`` once
    with the IPC handles of all ranks (see distributed.py)."""

    def __init__(self, model: ModelConfig, parallel: ParallelSpec, rank: int, m_cap: int,
                 weights: RankWeights, device: int = 0, activation: Activation = None,
                 knobs: Optional[LayerKnobs] = None):
        self.model, self.parallel, self.rank, self.m_cap = model, parallel, rank, m_cap
        self.n_pad = _ceil(model.N, 64)
        self.k_pad = _ceil(model.K // parallel.tp, 64) * parallel.tp
        self.ctx = _lib.Context(rank=rank, world=parallel.world_size, tp=parallel.tp, ep=parallel.ep,
                                device=device, E=model.E, topk=model.topk, N=self.n_pad, K=self.k_pad,
                                m_cap=m_cap)
        self.torch = self.ctx.torch
        self.weights = weights
        self.act = activation_code(activation)
        self.knobs = knobs or LayerKnobs.for_world(parallel.world_size)
        self.device = device
        self._xbuf = self.ctx.token_buffer()

    def token_range(self, M: int):
        w = self.parallel.world_size
        base = M // w
        lo = self.rank * base
        return lo, (M if self.rank == w - 1 else lo + base)

    def place_tokens(self, x_local, M: int) -> None:
        """Copy this rank's tokens into its symmetric token buffer."""
        lo, hi = self.token_range(M)
        if x_local.shape[0] != hi - lo:
            raise ConfigurationError(f"rank {self.rank} owns {hi - lo} tokens, got {x_local.shape[0]}")
        self._xbuf[lo:hi, :x_local.shape[1]].copy_(x_local, non_blocking=True)

    def n_comm1(self) -> int:
        """Combine CTAs layer1 launches with.  world > 1: rows of tokens with a
        single hosted expert are pushed by the epilogue; the combine CTAs reduce
        tokens with >= 2 hosted experts, so they may be 0 only when no token can
        have two (one expert per EP group, or top-1)."""
        k, world = self.knobs, self.parallel.world_size
        if world == 1:
            return k.n_comm1
        if self.model.E // self.parallel.ep == 1 or self.model.topk == 1:
            return k.n_comm1
        return max(2, k.n_comm1)

    def run(self, experts, M: int, y_local, combine_w=None, stream=None) -> None:
        """Index build + layer0 + layer1 (+ remote combine) on ``stream``;
        tokens must already be in place (``place_tokens``)."""
        k = self.knobs
        world = self.parallel.world_size
        self.ctx.forward(experts, M, self.weights.w0t, self.weights.w1t, combine_w, y_local,
                         activation=self.act, n_comm0=k.n_comm0 if world > 1 else 0,
                         n_comm1=self.n_comm1(),
                         group0=k.group0, wave1=k.wave1, stream=stream)

    def forward(self, x_local, experts, combine_w=None, M: Optional[int] = None):
        torch = self.torch
        M = int(experts.shape[0]) if M is None else M
        if M > self.m_cap:
            raise ConfigurationError(f"M={M} exceeds the layer capacity m_cap={self.m_cap}")
        dev = torch.device("cuda", self.device)
        if x_local.device != dev:
            x_local = x_local.to(dev, non_blocking=True)
        if x_local.dtype != torch.bfloat16:
            x_local = x_local.to(torch.bfloat16)
        ex = experts if (experts.device == dev and experts.dtype == torch.int32) else \
            experts.to(dev, non_blocking=True).to(torch.int32)
        cw = None
        if combine_w is not None:
            cw = combine_w if combine_w.device == dev and combine_w.dtype == torch.float32 else \
                combine_w.to(dev, non_blocking=True).float()
            cw = cw.contiguous()
        self.place_tokens(x_local, M)
        lo, hi = self.token_range(M)
        y = torch.empty(hi - lo, self.n_pad, dtype=torch.bfloat16, device=dev)
        self.run(ex.contiguous(), M, y, cw)
        return y if self.n_pad == self.model.N else y[:, :self.model.N]

    def forward_host(self, x_host, experts_host, combine_w=None, out=None, chunks: Optional[int] = None):
        """End-to-end form on HOST buffers (pinned for overlap): H2D of the
        tokens and router output, the forward, D2H of the result into ``out``
        (allocated pinned when None); asynchronous on the current stream like
        ``forward`` (synchronise it before reading ``out``).

        Single GPU, default (COMET_E2E=zerocopy; pinned ``x_host``/``out``):
        ONE launch with the host as the token-owning peer
        (``comet_forward_zerocopy``): dispatch CTAs read each token row once
        from pinned host memory over PCIe in the compute claim order and the
        fused combine writes output rows straight to ``out``.

        Single GPU, COMET_E2E=stream: ONE streamed launch
        (``comet_forward_host``): the token upload runs in 1024-token chunks
        whose landing the dispatch CTAs wait for, and the download of each
        chunk starts as soon as the fused combine finished its rows.  Correct
        (tests) but not yet faster: at world 1 the fused combine's folder
        waits for its sibling row's unit, which runs concurrently (layer1
        units 150 -> 220 us; 4.2 vs 4.1 ms, tools/stream_probe.py).  Default:
        the M tokens run as
        consecutive forwards over token chunks with the H2D of chunk c+1 and
        the D2H of chunk c-1 on two copy streams under the forward of chunk
        c.  Only the first chunk's upload and the last chunk's download stay
        exposed (COMET_E2E=chunks or an explicit ``chunks``; default 3 equal
        chunks for M >= 6144; ``chunks`` = an int for equal chunks or a list
        of sizes).  Multi-GPU ranks copy, run, copy."""
        torch = self.torch
        M = int(experts_host.shape[0])
        N = self.model.N
        lo_r, hi_r = self.token_range(M)
        if out is None:
            out = torch.empty(hi_r - lo_r, N, dtype=torch.bfloat16, pin_memory=True)
        world = self.parallel.world_size
        import os
        e2e_mode = os.environ.get("COMET_E2E", "zerocopy")
        if (world == 1 and chunks is None and e2e_mode == "zerocopy" and self.n_pad == N
                and N % 512 == 0 and self.model.topk <= 8 and x_host.is_pinned() and out.is_pinned()
                and out.is_contiguous()):
            # one launch, the host as the token-owning peer (comet_forward_zerocopy)
            ex = experts_host if experts_host.dtype == torch.int32 else experts_host.to(torch.int32)
            cw = None if combine_w is None else combine_w.float().contiguous()
            xb = x_host if x_host.dtype == torch.bfloat16 else x_host.to(torch.bfloat16)
            k = self.knobs
            # 16-pair groups, layer1 one group behind (PCIe-paced dispatch: a
            # group spans two experts' tiles, whose token rows land together
            # with the per-token dedup; 3.50 -> 3.40 ms vs 8-pair groups, lag 3)
            self.ctx.forward_zerocopy(xb.contiguous(), ex.contiguous(), cw, out, M, self.weights.w0t,
                                      self.weights.w1t, self.act, n_comm0=int(os.environ.get("COMET_ZC_NC", 16)),
                                      group0=int(os.environ.get("COMET_ZC_G0", 16)), wave1=k.wave1)
            return out
        if (world == 1 and chunks is None and e2e_mode == "stream"
                and self.n_pad == N and x_host.is_pinned() and out.is_pinned() and out.is_contiguous()):
            # one launch streaming the upload / download (comet_forward_host)
            ex = experts_host if experts_host.dtype == torch.int32 else experts_host.to(torch.int32)
            cw = None if combine_w is None else combine_w.float().contiguous()
            xb = x_host if x_host.dtype == torch.bfloat16 else x_host.to(torch.bfloat16)
            k = self.knobs
            # the dispatch CTAs also reduce the combine (they do not join the
            # GEMMs here): a small count
            self.ctx.forward_host(xb.contiguous(), ex.contiguous(), cw, out, M, self.weights.w0t, self.weights.w1t,
                                  self.act, n_comm0=int(os.environ.get("COMET_STREAM_NC", 16)), group0=k.group0,
                                  wave1=k.wave1, chunks=max(1, min(64, M // 1024)))
            return out
        sizes = _chunk_sizes(M, chunks)
        if world > 1 or len(sizes) <= 1:
            y = self.forward(x_host, experts_host, combine_w, M=M)
            out.copy_(y, non_blocking=True)
            return out
        dev = torch.device("cuda", self.device)
        C = len(sizes)
        bounds = [0]
        for n in sizes:
            bounds.append(bounds[-1] + n)
        mc = max(sizes)
        st = getattr(self, "_pipe", None)
        if st is None or st["mc"] < mc:
            bf, i32, f32 = torch.bfloat16, torch.int32, torch.float32
            st = {"mc": mc, "h2d": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                  "x": [torch.empty(mc, N, dtype=bf, device=dev) for _ in range(2)],
                  "ex": [torch.empty(mc, self.model.topk, dtype=i32, device=dev) for _ in range(2)],
                  "cw": [torch.empty(mc, self.model.topk, dtype=f32, device=dev) for _ in range(2)],
                  "y": [torch.empty(mc, self.n_pad, dtype=bf, device=dev) for _ in range(2)],
                  "done": [None, None], "down": [None, None]}
            self._pipe = st
        comp = torch.cuda.current_stream(dev)
        h2d, d2h = st["h2d"], st["d2h"]
        start = torch.cuda.Event()  # uploads begin after the caller's prior work (honest step timing)
        start.record(comp)
        h2d.wait_event(start)
        last = None
        for c in range(C):
            lo, hi = bounds[c], bounds[c + 1]
            m, b = hi - lo, c % 2
            with torch.cuda.stream(h2d):
                if st["done"][b] is not None:  # staging slot b consumed by its last forward
                    h2d.wait_event(st["done"][b])
                st["x"][b][:m].copy_(x_host[lo:hi], non_blocking=True)
                st["ex"][b][:m].copy_(experts_host[lo:hi], non_blocking=True)
                if combine_w is not None:
                    st["cw"][b][:m].copy_(combine_w[lo:hi], non_blocking=True)
                up = torch.cuda.Event()
                up.record(h2d)
            comp.wait_event(up)
            if st["down"][b] is not None:  # output slot b downloaded
                comp.wait_event(st["down"][b])
            self._xbuf[:m, :N].copy_(st["x"][b][:m], non_blocking=True)
            self.run(st["ex"][b][:m], m, st["y"][b][:m], st["cw"][b][:m] if combine_w is not None else None)
            done = torch.cuda.Event()
            done.record(comp)
            st["done"][b] = done
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                out[lo:hi].copy_(st["y"][b][:m, :N], non_blocking=True)
                last = torch.cuda.Event()
                last.record(d2h)
            st["down"][b] = last
        comp.wait_event(last)
        return out

    def close(self) -> None:
        self.ctx.close()


def _chunk_sizes(M: int, chunks=None) -> List[int]:
    """Token chunks of the host pipeline (see MoELayer.forward_host)."""
    if isinstance(chunks, (list, tuple)):
        if sum(chunks) != M or any(c <= 0 for c in chunks):
            raise ConfigurationError(f"chunk sizes {chunks} must be positive and sum to M={M}")
        return list(chunks)
    if chunks is not None:
        C = max(1, min(int(chunks), M))
        return [M * (c + 1) // C - M * c // C for c in range(C)]
    # measured (tools/e2e_probe.py, M=8192): 3 equal chunks 4.18 ms, 2: 4.24,
    # 4: 4.55, uneven (M/8, 3M/8, 3M/8, M/8): 4.53, 1: 5.28 -- every chunk
    # re-reads all expert weights, so fewer, larger chunks win
    C = max(1, min(3, M // 2048))
    return [M * (c + 1) // C - M * c // C for c in range(C)]


# ---------------------------------------------------------------------------
# Reference-compatible global entry points (all ranks emulated in-process).
# ---------------------------------------------------------------------------

_weight_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_group_cache: Dict[tuple, list] = {}


def _check_input(x, routing: RoutingTable):
    shape = tuple(x.shape)
    if shape != (routing.workload.M, routing.model.N):
        raise ConfigurationError(
            f"input must be shaped (M={routing.workload.M}, N={routing.model.N}), got {shape}")


def _rank_weights(weights: ExpertWeights, model: ModelConfig, parallel: ParallelSpec) -> List[RankWeights]:
    key = (model, parallel)
    per = _weight_cache.get(weights)
    if per is None:
        per = {}
        _weight_cache[weights] = per
    if key not in per:
        per[key] = [RankWeights.from_full(weights.w0, weights.w1, model, parallel, r)
                    for r in range(parallel.world_size)]
    return per[key]


def _layers(model: ModelConfig, parallel: ParallelSpec, m_cap: int, rw: List[RankWeights], act: int):
    key = (model, parallel, m_cap)
    layers = _group_cache.get(key)
    if layers is None:
        if len(_group_cache) > 8:
            for group in _group_cache.values():
                for layer in group:
                    layer.close()
            _group_cache.clear()
        layers = [MoELayer(model, parallel, r, m_cap, rw[r]) for r in range(parallel.world_size)]
        if parallel.world_size > 1:
            _lib.Context.link_local([layer.ctx for layer in layers])
        _group_cache[key] = layers
    for r, layer in enumerate(layers):
        layer.weights = rw[r]
        layer.act = act
    return layers


def run_emulated(x, weights: ExpertWeights, routing: RoutingTable, parallel: ParallelSpec,
                 activation: Activation = None, combine_weights=None, knobs: Optional[LayerKnobs] = None):
    """Execute the layer with every rank of ``parallel`` on this GPU (shared
    by the three reference entry points).  Returns a torch fp32 [M, N]."""
    torch = _lib.require_device()
    model = routing.model
    act = activation_code(activation)
    M = routing.workload.M
    rw = _rank_weights(weights, model, parallel)
    layers = _layers(model, parallel, max(1, M), rw, act)
    dev = torch.device("cuda", 0)
    xt = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float32))
    xt = xt.to(dev).to(torch.bfloat16)
    ex = torch.from_numpy(routing.as_array().copy()).to(dev)
    cw = None
    if combine_weights is not None:
        cw = (combine_weights if isinstance(combine_weights, torch.Tensor)
              else torch.as_tensor(np.asarray(combine_weights, dtype=np.float32))).to(dev).float().contiguous()
    out = torch.zeros(M, layers[0].n_pad, dtype=torch.bfloat16, device=dev)
    if M == 0:
        return out[:, :model.N].float()
    for layer in layers:
        if knobs is not None:
            layer.knobs = knobs
        lo, hi = layer.token_range(M)
        layer.place_tokens(xt[lo:hi], M)
    _phase_forward(layers, ex, M, [out[slice(*layer.token_range(M))] for layer in layers], cw)
    torch.cuda.synchronize()
    return out[:, :model.N].float()


def index_flags(world: int, n_comm1: int) -> int:
    """Index-build flags of the forward hot path (index.cuh): combine token
    list only for world-1 combine CTAs; x_ready signal when world > 1."""
    return (2 if world == 1 and n_comm1 > 0 else 0) | (4 if world > 1 else 0)


def fused_launch(world: int, n_comm1: int) -> bool:
    """Both layers in one persistent launch (comet_layers) -- the default,
    as in comet_forward -- unless world-1 combine CTAs are asked for or
    COMET_FUSED=0."""
    import os
    return os.environ.get("COMET_FUSED", "1") != "0" and not (world == 1 and n_comm1 > 0)


def _phase_forward(layers, ex, M: int, outs, cw, stream=None) -> None:
    """Enqueue a forward of every emulated rank, phase by phase, on one
    stream: each in-kernel wait is on work enqueued before it, so ranks that
    share a device cannot deadlock (index -> token signal -> layer0 ->
    layer1 -> remote combine)."""
    world = layers[0].parallel.world_size
    for layer in layers:
        # hot path: the kernels' tables only (+ the combine list for world-1
        # combine CTAs); world > 1: the build also publishes the x_ready epoch
        layer.ctx.index_build(ex, M, stream=stream, flags=index_flags(world, layer.n_comm1()))
    if fused_launch(world, layers[0].n_comm1()):
        for layer, y in zip(layers, outs):
            k = layer.knobs
            layer.ctx.layers(layer.weights.w0t, layer.weights.w1t, cw, y, layer.act,
                             k.n_comm0 if world > 1 else 0, k.group0, k.wave1, stream=stream)
    else:
        for layer in layers:
            k = layer.knobs
            layer.ctx.layer0(layer.weights.w0t, layer.act, k.n_comm0 if world > 1 else 0, k.group0, stream=stream)
        for layer, y in zip(layers, outs):
            k = layer.knobs
            layer.ctx.layer1(layer.weights.w1t, cw, y, layer.n_comm1(), k.wave1,
                             stream=stream)
    if world > 1:
        for layer, y in zip(layers, outs):
            layer.ctx.combine_finish(y, stream=stream)


def _to_numpy(y) -> np.ndarray:
    return y.double().cpu().numpy()


def execute_naive(x, weights: ExpertWeights, routing: RoutingTable, activation: Activation = None,
                  combine_weights=None) -> np.ndarray:
    """Layer forward (ref executor.py:132-148), on the GPU path."""
    _check_input(x, routing)
    weights.check_model(routing.model)
    return _to_numpy(run_emulated(x, weights, routing, routing.parallel, activation, combine_weights))


def _as_list(scheds: Union[TileSchedule, Sequence[TileSchedule]]) -> List[TileSchedule]:
    return [scheds] if isinstance(scheds, TileSchedule) else list(scheds)


def _check_schedules(scheds0, scheds1, routing: RoutingTable) -> None:
    """Schedules must validate clean and cover each EP group once
    (ref executor.py:159-177)."""
    par = routing.parallel
    for sched in (*scheds0, *scheds1):
        bad = validate_schedule(sched, routing)
        if bad:
            raise ConfigurationError(f"schedule for rank {sched.rank} is invalid: {bad[0].message}")
    for scheds, layer in ((scheds0, 0), (scheds1, 1)):
        groups = sorted(par.ep_group_of_rank(s.rank) for s in scheds)
        if groups != list(range(par.ep)):
            raise ConfigurationError(
                f"layer{layer} schedules must cover each EP group exactly once, got groups {groups}")


def execute_scheduled(x, weights: ExpertWeights, routing: RoutingTable,
                      scheds0: Union[TileSchedule, Sequence[TileSchedule]],
                      scheds1: Union[TileSchedule, Sequence[TileSchedule]],
                      activation: Activation = None, combine_weights=None) -> np.ndarray:
    """Tile-order execution (ref executor.py:180-218).  The schedules are
    validated exactly like the reference; the GPU then runs its own
    device-built schedule for the same tiles (results do not depend on tile
    order)."""
    _check_input(x, routing)
    weights.check_model(routing.model)
    _check_schedules(_as_list(scheds0), _as_list(scheds1), routing)
    return _to_numpy(run_emulated(x, weights, routing, routing.parallel, activation, combine_weights))


def execute_tp_sharded(x, weights: ExpertWeights, routing: RoutingTable, tp: int,
                       activation: Activation = None, combine_weights=None) -> np.ndarray:
    """K split into ``tp`` shards, partials summed rank-ascending
    (ref executor.py:221-246): runs tp x ep emulated ranks."""
    _check_input(x, routing)
    weights.check_model(routing.model)
    if routing.model.K % tp:
        raise ConfigurationError(f"K={routing.model.K} is not divisible by tp={tp}")
    par = ParallelSpec(tp=tp, ep=routing.parallel.ep)
    return _to_numpy(run_emulated(x, weights, routing, par, activation, combine_weights))


_RANK_LAYERS: Dict[tuple, "MoELayer"] = {}


def execute_scheduled_rank(x_local, w_local: RankWeights, routing: RoutingTable, sched0: Optional[TileSchedule] = None,
                           sched1: Optional[TileSchedule] = None, activation: Activation = None,
                           combine_weights=None, layer: Optional["MoELayer"] = None, knobs: Optional[LayerKnobs] = None):
    """Per-rank form of ``execute_scheduled`` (ref executor.py:
    180-218) for one process per GPU: this rank's tokens ``x_local``
    [M_r, N] (the rows ``routing.parallel``'s contiguous pre-distribution
    gives it, routing.py:86-104) in, this rank's output rows [M_r, N] out, as
    a bf16 tensor on this rank's GPU.  ``sched0`` / ``sched1`` are this
    rank's schedules (optional), validated like the reference's.  The first
    call creates the rank's ``MoELayer`` with ``distributed.init_layer``
    (collective: every rank calls it, same routing shape) and caches it;
    ``layer`` passes an existing one.  ``combine_weights`` are the global
    [M, topk] weights (a rank's combine reads any token's)."""
    from . import distributed
    par = routing.parallel
    rank, world, _ = distributed.world_info()
    distributed.check_world(par, world)
    for sched, lay in ((sched0, 0), (sched1, 1)):
        if sched is None:
            continue
        if sched.rank != rank or sched.layer != lay:
            raise ConfigurationError(f"schedule (rank {sched.rank}, layer {sched.layer}) given to rank {rank} "
                                     f"as its layer{lay} schedule")
        bad = validate_schedule(sched, routing, rank)
        if bad:
            raise ConfigurationError(f"schedule for rank {rank} is invalid: {bad[0].message}")
    M = routing.workload.M
    if layer is not None and layer.act != activation_code(activation):
        raise ConfigurationError("activation differs from the one the given layer was built with")
    if layer is None:
        key = (routing.model, par, M, id(w_local), activation_code(activation))
        layer = _RANK_LAYERS.get(key)
        if layer is None:
            layer = distributed.init_layer(routing.model, par, M, w_local, activation=activation, knobs=knobs)
            _RANK_LAYERS[key] = layer
    torch = layer.torch
    ex = torch.from_numpy(routing.as_array().copy())
    cw = None if combine_weights is None else torch.as_tensor(np.asarray(combine_weights, np.float32))
    if not isinstance(x_local, torch.Tensor):
        x_local = torch.from_numpy(np.ascontiguousarray(np.asarray(x_local, np.float32)))
    lo, hi = layer.token_range(M)
    if x_local.shape[0] != hi - lo or x_local.shape[1] != routing.model.N:
        raise ConfigurationError(f"x_local must be [{hi - lo}, {routing.model.N}] on rank {rank}, "
                                 f"got {tuple(x_local.shape)}")
    return layer.forward(x_local, ex, cw, M=M)
