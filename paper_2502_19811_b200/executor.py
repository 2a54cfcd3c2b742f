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
        # (numpy: a private copy of this rank's slice -- cached weights are read-only)
        w0s = torch.from_numpy(np.array(w0[e_lo:e_lo + e_per, :, s * kl:(s + 1) * kl])) \
            if not isinstance(w0, torch.Tensor) else w0[e_lo:e_lo + e_per, :, s * kl:(s + 1) * kl]
        w1s = torch.from_numpy(np.array(w1[e_lo:e_lo + e_per, s * kl:(s + 1) * kl, :])) \
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
    layer1 column-wave width.  ``zc_*`` / ``stream_n_comm`` size the
    single-GPU host-buffer forwards.  The remaining fields are the context
    options of include/comet_b200.h (COMET_OPT_*, ``_lib.OPTIONS``): None
    keeps the library's measured default.  Nothing is read from the
    environment."""

    n_comm0: Optional[int] = None  # None: the adaptive chooser (assigner.choose_split) per token count
    n_comm1: int = 0
    group0: Optional[int] = None  # None: measured with n_c by the chooser (assigner.choose_knobs)
    wave1: int = 4
    zc_n_comm: int = 16
    zc_group0: int = 16
    stream_n_comm: int = 16
    fused: Optional[bool] = None
    ksplit_max: Optional[int] = None
    split_tail0: Optional[bool] = None
    split1: Optional[int] = None
    dedup: Optional[int] = None
    pull_local: Optional[bool] = None
    fold_order: Optional[bool] = None
    group1: Optional[int] = None
    chunk_rows: Optional[int] = None
    pdl: Optional[int] = None
    grid: Optional[int] = None
    fuse1: Optional[bool] = None
    spin_timeout_ms: Optional[int] = None
    zc_dedup: Optional[bool] = None
    zc_interleave: Optional[int] = None
    zc_download: Optional[int] = None
    zc_order: Optional[bool] = None
    zc_fold_order: Optional[bool] = None
    stream_fuse: Optional[bool] = None
    sequential: Optional[bool] = None
    streamk: Optional[bool] = None
    fold_stride: Optional[int] = None

    @classmethod
    def for_world(cls, world: int, **options) -> "LayerKnobs":
        """Measured defaults: n_comm0 and group0 left to the
        adaptive chooser (measured split metadata, else the fitted cost model
        and 8-pair layer0 groups at EP=1 / EP>=8, 4-pair groups at EP=2/4)."""
        return cls(**options)

    def options(self) -> Dict[str, Optional[int]]:
        """The COMET_OPT_* values (None = library default)."""
        return {name: (None if getattr(self, name) is None else int(getattr(self, name))) for name in _lib.OPTIONS}

    def is_fused(self, world: int) -> bool:
        """Both layers in one persistent launch (comet_layers) -- the default,
        as in comet_forward -- unless world-1 combine CTAs are asked for or
        ``fused`` is False."""
        return self.fused is not False and not (world == 1 and self.n_comm1 > 0)


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
        self._applied: Optional[Dict[str, Optional[int]]] = None
        self.knobs = knobs or LayerKnobs.for_world(parallel.world_size)
        self.device = device
        self._xbuf = self.ctx.token_buffer()
        self._nc_cache: Dict[int, tuple] = {}

    def n_comm0(self, M: int) -> int:
        """Layer0 dispatch CTAs for a forward of M tokens: 0 at world 1 (no
        remote rows), the knob when set, else the adaptive chooser's n_c
        (``assigner.choose_split``: measured sweep, else the fitted cost
        model), cached per M."""
        return self.split_choice(M)[0]

    def split_choice(self, M: int):
        """(n_comm0, source) -- source "knob", "measured", "model" or "world1"."""
        if self.parallel.world_size == 1:
            return 0, "world1"
        if self.knobs.n_comm0 is not None:
            return self.knobs.n_comm0, "knob"
        return self._chosen(M)[:2]

    def group0(self, M: int) -> int:
        """Layer0 pair-group size: the knob when set, else the one measured
        with the chosen n_c (``assigner.choose_knobs``)."""
        if self.knobs.group0 is not None:
            return self.knobs.group0
        if self.parallel.world_size == 1:
            from .assigner import default_group0
            return default_group0(1)
        return self._chosen(M)[2]

    def _chosen(self, M: int):
        hit = self._nc_cache.get(M)
        if hit is None:
            from .assigner import choose_knobs
            blocks = self.knobs.grid or _lib.device_info(self.device)["sms"]
            split, src, g0 = choose_knobs(self.model, self.parallel, M, blocks)
            # the kernel needs an even count leaving >= one compute pair; a
            # reduced grid (ranks sharing one GPU) keeps half of it computing
            cap = blocks - 2 if self.knobs.grid is None else (blocks // 2) // 2 * 2
            nc = max(2, min(split.n_c, cap) // 2 * 2)
            hit = self._nc_cache[M] = (nc, src, g0)
        return hit

    @property
    def knobs(self) -> LayerKnobs:
        return self._knobs

    @knobs.setter
    def knobs(self, knobs: LayerKnobs) -> None:
        """Install knobs: the COMET_OPT_* fields go to the native context."""
        opts = knobs.options()
        if opts != self._applied:
            for name, value in opts.items():
                if self._applied is None or self._applied.get(name) != value:
                    self.ctx.set_option(name, value)
            self._applied = opts
        self._knobs = knobs

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
                         activation=self.act, n_comm0=self.n_comm0(M),
                         n_comm1=self.n_comm1(),
                         group0=self.group0(M), wave1=k.wave1, stream=stream)

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

    def forward_host(self, x_host, experts_host, combine_w=None, out=None, chunks=None,
                     mode: Optional[str] = None):
        """End-to-end form on HOST buffers (pinned for overlap): tokens and
        router output in, the result into ``out`` (bf16 [M_r, N], allocated
        pinned when None); asynchronous on the current stream like
        ``forward`` (synchronise it before reading ``out``).

        ``mode`` (single GPU; default "zerocopy" when ``out`` is pinned,
        contiguous bf16 and N % 512 == 0, else "chunks"):

        * "zerocopy": ONE launch with the host as the token-owning peer
          (``comet_forward_zerocopy``): dispatch CTAs read each token row once
          from pinned host memory over PCIe in the compute claim order and the
          fused combine writes output rows to ``out``.  A token tensor that is
          not pinned contiguous bf16 is first converted into a pinned staging
          buffer owned by the layer (the kernel reads it asynchronously).
        * "stream": ONE streamed launch (``comet_forward_host``): the token
          upload runs in 1024-token chunks whose landing the dispatch CTAs
          wait for, the download of each chunk starts as soon as the fused
          combine finished its rows.  Correct (tests) but slower than
          zerocopy.
        * "chunks": consecutive forwards over token chunks with the H2D of
          chunk c+1 and the D2H of chunk c-1 on two copy streams under the
          forward of chunk c (``chunks`` = an int for equal chunks or a list
          of sizes; default 3 equal chunks for M >= 6144).

        Multi-GPU ranks copy, run, copy."""
        torch = self.torch
        M = int(experts_host.shape[0])
        N = self.model.N
        lo_r, hi_r = self.token_range(M)
        if out is None:
            out = torch.empty(hi_r - lo_r, N, dtype=torch.bfloat16, pin_memory=True)
        if tuple(out.shape) != (hi_r - lo_r, N):
            raise ConfigurationError(f"out must be [{hi_r - lo_r}, {N}], got {tuple(out.shape)}")
        world = self.parallel.world_size
        out_direct = out.dtype == torch.bfloat16 and out.is_contiguous() and out.is_pinned()
        if mode is None:
            mode = "zerocopy" if chunks is None else "chunks"
        if mode not in ("zerocopy", "stream", "chunks"):
            raise ConfigurationError(f"forward_host mode {mode!r}: choose zerocopy, stream or chunks")
        single = world == 1 and self.n_pad == N and out_direct
        k = self.knobs
        if single and mode == "zerocopy" and N % 512 == 0 and self.model.topk <= 8:
            # one launch, the host as the token-owning peer (comet_forward_zerocopy)
            ex = experts_host if experts_host.dtype == torch.int32 else experts_host.to(torch.int32)
            cw = None if combine_w is None else combine_w.float().contiguous()
            xb = self._pinned_tokens(x_host, M)
            # 16-pair groups, layer1 one group behind (PCIe-paced dispatch: a
            # group spans two experts' tiles, whose token rows land together
            # with the per-token dedup; 3.50 -> 3.40 ms vs 8-pair groups, lag 3)
            self.ctx.forward_zerocopy(xb, ex.contiguous(), cw, out, M, self.weights.w0t, self.weights.w1t, self.act,
                                      n_comm0=k.zc_n_comm, group0=k.zc_group0, wave1=k.wave1)
            self._note_host_reader()
            return out
        if single and mode == "stream":
            # one launch streaming the upload / download (comet_forward_host)
            ex = experts_host if experts_host.dtype == torch.int32 else experts_host.to(torch.int32)
            cw = None if combine_w is None else combine_w.float().contiguous()
            xb = self._pinned_tokens(x_host, M)
            # the dispatch CTAs also reduce the combine (they do not join the
            # GEMMs here): a small count
            self.ctx.forward_host(xb, ex.contiguous(), cw, out, M, self.weights.w0t, self.weights.w1t,
                                  self.act, n_comm0=k.stream_n_comm, group0=self.group0(M),
                                  wave1=k.wave1, chunks=max(1, min(64, M // 1024)))
            self._note_host_reader()
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

    def _pinned_tokens(self, x_host, M: int):
        """``x_host`` as pinned contiguous bf16 host memory that stays alive
        while the kernel reads it: the caller's tensor when it already is,
        else a staging buffer owned by the layer (reused once the previous
        host-reading launch is done)."""
        torch = self.torch
        if (x_host.dtype == torch.bfloat16 and x_host.is_contiguous() and x_host.is_pinned()
                and x_host.device.type == "cpu"):
            return x_host
        st = getattr(self, "_x_stage", None)
        if st is None or st.shape[0] < M or st.shape[1] != x_host.shape[1]:
            st = torch.empty(max(M, 1), x_host.shape[1], dtype=torch.bfloat16, pin_memory=True)
            self._x_stage = st
        ev = getattr(self, "_host_reader", None)
        if ev is not None:
            ev.synchronize()  # the previous launch has finished reading the staging buffer
        st[:M].copy_(x_host.to("cpu"))
        return st[:M]

    def _note_host_reader(self) -> None:
        ev = self.torch.cuda.Event()
        ev.record(self.torch.cuda.current_stream(self.device))
        self._host_reader = ev

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


def invalidate_weight_cache(weights: Optional[ExpertWeights] = None) -> None:
    """Drop the prepared device copies of ``weights`` (all when None)."""
    if weights is None:
        _weight_cache.clear()
    else:
        _weight_cache.pop(weights, None)


def _rank_weights(weights, model: ModelConfig, parallel: ParallelSpec) -> List[RankWeights]:
    """Per-rank bf16 device copies.  ``weights`` is an ``ExpertWeights``
    (cached per instance: its arrays are made read-only while cached, so an
    in-place edit raises instead of silently using stale copies; call
    ``invalidate_weight_cache`` after replacing them) or a ``(w0, w1)`` pair
    of torch tensors, e.g. on the GPU for full-size shapes (not cached)."""
    if isinstance(weights, tuple):
        w0, w1 = weights
        return [RankWeights.from_full(w0, w1, model, parallel, r) for r in range(parallel.world_size)]
    key = (model, parallel)
    per = _weight_cache.get(weights)
    if per is None:
        per = {}
        _weight_cache[weights] = per
        for arr in (weights.w0, weights.w1):
            if isinstance(arr, np.ndarray):
                arr.flags.writeable = False
    if key not in per:
        per[key] = [RankWeights.from_full(weights.w0, weights.w1, model, parallel, r)
                    for r in range(parallel.world_size)]
    return per[key]


def _layers(model: ModelConfig, parallel: ParallelSpec, m_cap: int, rw: List[RankWeights], act: int):
    """Emulated rank layers for (model, parallel), sized for >= m_cap tokens
    (capacity rounded up to a power of two so varying M reuses the group;
    at most 4 groups are kept, least recently used evicted and freed)."""
    cap = 1 << max(0, int(m_cap - 1).bit_length())
    key = None
    for k in _group_cache:
        if k[0] == model and k[1] == parallel and k[2] >= m_cap:
            key = k
            break
    if key is None:
        while len(_group_cache) >= 4:
            old = next(iter(_group_cache))
            for layer in _group_cache.pop(old):
                layer.close()
        key = (model, parallel, cap)
        layers = [MoELayer(model, parallel, r, cap, rw[r]) for r in range(parallel.world_size)]
        if parallel.world_size > 1:
            _lib.Context.link_local([layer.ctx for layer in layers])
        _group_cache[key] = layers
    layers = _group_cache.pop(key)
    _group_cache[key] = layers  # most recently used last
    for r, layer in enumerate(layers):
        layer.weights = rw[r]
        layer.act = act
    return layers


def run_emulated(x, weights, routing: RoutingTable, parallel: ParallelSpec,
                 activation: Activation = None, combine_weights=None, knobs: Optional[LayerKnobs] = None):
    """Execute the layer with every rank of ``parallel`` on this GPU (shared
    by the three reference entry points).  ``weights``: ``ExpertWeights`` or
    a ``(w0 [E,N,K], w1 [E,K,N])`` pair of torch tensors.  Returns a torch
    fp32 [M, N]."""
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
        layer.knobs = knobs if knobs is not None else LayerKnobs.for_world(parallel.world_size)
        lo, hi = layer.token_range(M)
        layer.place_tokens(xt[lo:hi], M)
    _phase_forward(layers, ex, M, [out[slice(*layer.token_range(M))] for layer in layers], cw)
    torch.cuda.synchronize()
    return out[:, :model.N].float()


def index_flags(world: int, n_comm1: int) -> int:
    """Index-build flags of the forward hot path (index.cuh): combine token
    list only for world-1 combine CTAs; x_ready signal when world > 1; the
    layer1 pair order comet_forward uses (kIndexForwardOrder)."""
    return (2 if world == 1 and n_comm1 > 0 else 0) | (4 if world > 1 else 0) | 64


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
    if layers[0].knobs.is_fused(world):
        for layer, y in zip(layers, outs):
            k = layer.knobs
            layer.ctx.layers(layer.weights.w0t, layer.weights.w1t, cw, y, layer.act,
                             layer.n_comm0(M), layer.group0(M), k.wave1, stream=stream)
    else:
        for layer in layers:
            k = layer.knobs
            layer.ctx.layer0(layer.weights.w0t, layer.act, layer.n_comm0(M), layer.group0(M), stream=stream)
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


def _rank_layer(model: ModelConfig, par: ParallelSpec, M: int, w_local: RankWeights, activation: Activation,
                knobs: Optional[LayerKnobs]) -> "MoELayer":
    """This rank's cached layer for (model, parallel, activation), with a
    token capacity >= M (rounded up to a power of two, so varying batch sizes
    reuse it); the weights are passed per call.  Creating one is collective
    (``distributed.init_layer``); every rank takes the same branch because the
    decision depends only on arguments all ranks share.  At most two layers
    are kept (the older one is closed)."""
    from . import distributed
    act = activation_code(activation)
    key = (model, par, act)
    layer = _RANK_LAYERS.get(key)
    if layer is None or layer.m_cap < M:
        if layer is not None:
            _RANK_LAYERS.pop(key).close()
        while len(_RANK_LAYERS) >= 2:
            _RANK_LAYERS.pop(next(iter(_RANK_LAYERS))).close()
        cap = 1 << max(0, int(max(M, 1) - 1).bit_length())
        layer = distributed.init_layer(model, par, cap, w_local, activation=activation, knobs=knobs)
        _RANK_LAYERS[key] = layer
    layer.weights = w_local
    if knobs is not None:
        layer.knobs = knobs
    return layer


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
        layer = _rank_layer(routing.model, par, M, w_local, activation, knobs)
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
