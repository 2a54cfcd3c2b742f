"""GPU router front-end: gate logits -> router output.

The step in front of the fused layer: ``route_topk`` turns gate logits
``[M, E]`` (fp32 or bf16, on the GPU) into the reference's router output --
top-k expert ids stored ascending per token, ``RoutingTable.experts_per_token``
(routing.py:62-163) -- and the combine weights ``[M, topk]`` in the same
ascending-expert slot order that ``_combine`` folds (executor.py:102-120),
with one ``comet_router_topk`` launch (csrc/router.cu).  The result feeds
``MoELayer.forward`` / ``comet_index_build`` directly, with no host round
trip.

The reference has no router (``build_routing``, routing.py:283-307, is a
synthetic count generator), so selection is defined as a stable descending
sort (ties -> smaller expert id) and checked bit-exact against the oracle's
``router_topk``; weights are fp32 within 1e-6 of the fp64 oracle.
"""

from __future__ import annotations

from typing import Optional, Tuple

import numpy as np

from . import _lib
from .config import ConfigurationError, ModelConfig, ParallelSpec, WorkloadSpec
from .routing import RoutingTable

NORMS = {None: 0, "none": 0, "topk": 1, "all": 2}


def route_topk(logits, topk: int, norm: Optional[str] = "topk", experts=None, weights=None,
               stream=None) -> Tuple[object, Optional[object]]:
    """Device top-k routing.  ``logits``: torch CUDA tensor [M, E], float32
    or bfloat16.  ``norm``: ``"topk"`` (softmax over the selected logits,
    Mixtral), ``"all"`` (softmax over all E, selected entries; Qwen2-MoE
    without top-k renormalisation) or ``None`` (ids only).  Returns
    ``(experts int32 [M, topk], weights float32 [M, topk] or None)``;
    asynchronous on ``stream`` (default: the current stream)."""
    torch = _lib.require_device()
    if norm not in NORMS:
        raise ConfigurationError(f"unknown router norm {norm!r}; expected one of 'topk', 'all', None")
    if logits.dim() != 2:
        raise ConfigurationError(f"logits must be [M, E], got shape {tuple(logits.shape)}")
    if logits.dtype not in (torch.float32, torch.bfloat16):
        raise ConfigurationError(f"logits must be float32 or bfloat16, got {logits.dtype}")
    if not logits.is_cuda:
        raise ConfigurationError("logits must live on the GPU (there is no host router)")
    logits = logits.contiguous()
    M, E = logits.shape
    dev = logits.device
    if experts is None:
        experts = torch.empty(M, topk, dtype=torch.int32, device=dev)
    code = NORMS[norm]
    if code and weights is None:
        weights = torch.empty(M, topk, dtype=torch.float32, device=dev)
    if tuple(experts.shape) != (M, topk) or experts.dtype != torch.int32 or not experts.is_contiguous():
        raise ConfigurationError("experts buffer must be contiguous int32 [M, topk]")
    if code and (tuple(weights.shape) != (M, topk) or weights.dtype != torch.float32 or not weights.is_contiguous()):
        raise ConfigurationError("weights buffer must be contiguous float32 [M, topk]")
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    _lib.check(_lib.load().comet_router_topk(
        logits.data_ptr(), 1 if logits.dtype == torch.bfloat16 else 0, M, E, topk, code,
        experts.data_ptr(), weights.data_ptr() if code else None, s.cuda_stream))
    return experts, (weights if code else None)


def routing_from_logits(model: ModelConfig, parallel: ParallelSpec, logits, norm: Optional[str] = "topk",
                        seed: int = 0) -> Tuple[RoutingTable, Optional[np.ndarray]]:
    """Host-facing form: route on the GPU, wrap the ids as a validated
    ``RoutingTable`` (routing.py:146-163 checks) and return the combine
    weights as float64 numpy (the reference's ``combine_weights``)."""
    torch = _lib.require_device()
    if not isinstance(logits, torch.Tensor):
        logits = torch.as_tensor(np.asarray(logits, dtype=np.float32))
    if logits.shape[1] != model.E:
        raise ConfigurationError(f"logits have {logits.shape[1]} experts, model has E={model.E}")
    ex, w = route_topk(logits.cuda(), model.topk, norm)
    torch.cuda.synchronize()
    table = RoutingTable.from_array(model, parallel, WorkloadSpec(M=int(logits.shape[0]), seed=seed, std=0.0),
                                    ex.cpu().numpy())
    return table, (None if w is None else w.double().cpu().numpy())
