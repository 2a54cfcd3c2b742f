"""Reference computations for the GPU parity tests (test infrastructure)."""

import numpy as np

from oracle import moe_oracle as O


def bf16(a):
    return O.round_bf16(np.asarray(a, dtype=np.float32)).astype(np.float64)


def oracle_bf16_inputs(x, w0, w1, experts, activation=None, combine_weights=None, tp=1):
    """fp64 oracle on bf16-rounded inputs (isolates kernel error from input
    quantisation)."""
    args = (bf16(x), bf16(w0), bf16(w1), np.asarray(experts))
    if tp == 1:
        return O.layer_forward(*args, activation=activation, combine_weights=combine_weights)
    return O.layer_forward_tp(*args, tp, activation=activation, combine_weights=combine_weights)


def torch_reference(x, w0, w1, experts, activation=None, combine_w=None, tp=1):
    """Plain PyTorch fp32 reference of the same op (bf16 inputs, bf16 h and
    expert rows -- the storage points of the fused kernels).  ``tp`` > 1
    follows execute_tp_sharded (ref executor.py:221-246): K is cut into tp
    contiguous shards, each shard's expert row is its own bf16 partial, and
    the partials are summed in shard order before the combine."""
    import torch
    M, N = x.shape
    K = w0.shape[2]
    ks = K // tp
    xf = x.to(torch.bfloat16).float()
    y = torch.zeros(M, N, dtype=torch.float32, device=x.device)
    for e in range(w0.shape[0]):
        tok, slot = (experts == e).nonzero(as_tuple=True)
        if tok.numel() == 0:
            continue
        ye = torch.zeros(tok.numel(), N, dtype=torch.float32, device=x.device)
        for s in range(tp):
            h = xf[tok] @ w0[e, :, s * ks:(s + 1) * ks].to(torch.bfloat16).float()
            if activation == "tanh":
                h = torch.tanh(h)
            elif activation == "silu":
                h = h * torch.sigmoid(h)
            h = h.to(torch.bfloat16).float()
            ye += (h @ w1[e, s * ks:(s + 1) * ks].to(torch.bfloat16).float()).to(torch.bfloat16).float()
        if combine_w is not None:
            ye = ye * combine_w[tok, slot][:, None]
        y.index_add_(0, tok, ye)
    return y


# Tolerance (BASELINE.json north_star): bf16 in, fp32
# accumulate, bf16 intermediate; measured 3.3e-3 / 3.6e-3 max-normalised.
MAX_REL = 1e-2     # max|d| / max|ref|
FROB_REL = 5e-3    # ||d||_F / ||ref||_F


def assert_close(got, ref, max_rel=MAX_REL, frob_rel=FROB_REL, what=""):
    mx, fr = O.relative_error(np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64))
    assert mx <= max_rel and fr <= frob_rel, f"{what}: max-normalised {mx:.3e}, frobenius {fr:.3e}"
    return mx, fr
