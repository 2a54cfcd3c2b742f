"""Staged GPU bring-up check (prints PASS/FAIL per stage, never raises)."""
import os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_19811_b200 import _lib
from paper_2502_19811_b200 import config as C, routing as Rt
from oracle import moe_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def stage(name):
    def deco(fn):
        def run():
            t = time.time()
            try:
                fn()
                print(f"[PASS] {name} ({time.time()-t:.1f}s)", flush=True)
            except Exception:
                print(f"[FAIL] {name}", flush=True)
                traceback.print_exc()
        return run
    return deco


def prep_weights(w0, w1, e_lo, E_r, tp_idx, k_local):
    ks = slice(tp_idx * k_local, (tp_idx + 1) * k_local)
    w0t = w0[e_lo:e_lo + E_r, :, ks].transpose(1, 2).contiguous().to(torch.bfloat16)
    w1t = w1[e_lo:e_lo + E_r, ks, :].transpose(1, 2).contiguous().to(torch.bfloat16)
    return w0t, w1t


def torch_ref(x, w0, w1, experts, act=None, cw=None):
    """fp32 reference on bf16-rounded inputs, bf16 intermediate h (per expert)."""
    M, N = x.shape
    E = w0.shape[0]
    y = torch.zeros(M, N, dtype=torch.float32, device=x.device)
    xf = x.float()
    for e in range(E):
        tok, slot = (experts == e).nonzero(as_tuple=True)
        if tok.numel() == 0:
            continue
        h = xf[tok] @ w0[e].to(torch.bfloat16).float()
        if act == "tanh":
            h = torch.tanh(h)
        h = h.to(torch.bfloat16).float()
        ye = h @ w1[e].to(torch.bfloat16).float()
        ye = ye.to(torch.bfloat16).float()
        if cw is not None:
            ye = ye * cw[tok, slot][:, None]
        y.index_add_(0, tok, ye)
    return y


@stage("device info")
def s_info():
    print("   ", _lib.device_info(0))


@stage("index build vs reference fixtures")
def s_index():
    for name in ("c1", "mx_ep8_s032", "mx_ep1_s032", "ph_tp2ep4_s032", "qw_ep8_s032"):
        z = np.load(os.path.join(GOLD, f"index_{name}.npz"))
        E, topk, N, K, M, tp, ep, tr, tc = z["meta"].tolist()
        std = 0.0 if name == "c1" else 0.032
        r = Rt.build_routing(C.ModelConfig(L=1, E=E, topk=topk, N=N, K=K), C.ParallelSpec(tp, ep),
                             C.WorkloadSpec(M=M, seed=0, std=std))
        ex = torch.from_numpy(r.as_array().copy()).cuda()
        for rank in z["ranks"].tolist():
            ctx = _lib.Context(rank=rank, world=tp * ep, tp=tp, ep=ep, device=0, E=E, topk=topk,
                               N=N, K=K, m_cap=M)
            ctx.index_build(ex, M, tr, tc)
            got = ctx.download_index()
            bad = []
            for key in ("expert_counts", "transfer_counts", "row_offsets", "row_token", "row_src",
                        "n_local", "tiles0", "tiles1", "chunks"):
                if not np.array_equal(got[key], z[f"r{rank}_{key}"]):
                    bad.append(key)
            ora = O.index_for_rank(r.as_array(), E, tp, ep, rank, tr, tc, N)
            print(f"    {name} r{rank}: meta={got['meta'][:8].tolist()} mismatches={bad}")
            assert not bad, bad
            ctx.close()


def run_layer(E, topk, N, K, M, std=0.0, act=None, weighted=False, n_comm1=0, wave=4, group=16,
              seed=0, timing=False):
    model = C.ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    r = Rt.build_routing(model, C.ParallelSpec(1, 1), C.WorkloadSpec(M=M, seed=seed, std=std))
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
    w0 = torch.randn(E, N, K, device="cuda", generator=g) / N ** 0.5
    w1 = torch.randn(E, K, N, device="cuda", generator=g) / K ** 0.5
    ex = torch.from_numpy(r.as_array().copy()).cuda()
    cw = torch.rand(M, topk, device="cuda", generator=g) if weighted else None
    ctx = _lib.Context(rank=0, world=1, tp=1, ep=1, device=0, E=E, topk=topk, N=N, K=K, m_cap=M)
    w0t, w1t = prep_weights(w0, w1, 0, E, 0, K)
    ctx.token_buffer()[:M].copy_(x)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    a = _lib.ACTIVATIONS[act]
    ctx.forward(ex, M, w0t, w1t, cw, y, activation=a, n_comm0=n_comm1, n_comm1=n_comm1, group0=group, wave1=wave)
    torch.cuda.synchronize()
    ref = torch_ref(x, w0, w1, ex.long(), act, cw)
    mx, fr = O.relative_error(y.float().cpu().numpy(), ref.cpu().numpy())
    print(f"    E{E} top{topk} N{N} K{K} M{M} act={act} w={weighted}: max/max={mx:.2e} frob={fr:.2e}")
    if timing:
        for _ in range(3):
            ctx.forward(ex, M, w0t, w1t, cw, y, activation=a, n_comm0=n_comm1, n_comm1=n_comm1, group0=group, wave1=wave)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        n = 10
        st.record()
        for _ in range(n):
            ctx.forward(ex, M, w0t, w1t, cw, y, activation=a, n_comm0=n_comm1, n_comm1=n_comm1, group0=group, wave1=wave)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / n
        flops = 4.0 * M * topk * N * K
        print(f"    forward {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
    ctx.close()
    assert mx < 1e-2, mx


@stage("layer EP=1 small identity")
def s_small():
    run_layer(4, 2, 256, 512, 300)


@stage("layer EP=1 small tanh weighted")
def s_small2():
    run_layer(8, 3, 512, 1024, 1000, act="tanh", weighted=True)


@stage("layer EP=1 config1 shape")
def s_c1():
    run_layer(8, 2, 512, 1024, 512)


@stage("layer EP=1 Mixtral M=2048")
def s_mx_small():
    run_layer(8, 2, 4096, 14336, 2048, timing=True)


@stage("layer EP=1 Mixtral M=8192")
def s_mx():
    run_layer(8, 2, 4096, 14336, 8192, timing=True)
    run_layer(8, 2, 4096, 14336, 8192, timing=True, n_comm1=4)


@stage("layer EP=1 comm-CTA combine, tanh weighted")
def s_comm():
    run_layer(8, 3, 512, 1024, 1000, act="tanh", weighted=True, n_comm1=2)
    run_layer(8, 2, 4096, 14336, 1024, std=0.05, weighted=True, n_comm1=6)


if __name__ == "__main__":
    which = sys.argv[1:] or ["info", "index", "small", "small2", "c1", "mxs", "mx"]
    table = {"info": s_info, "index": s_index, "small": s_small, "small2": s_small2, "c1": s_c1,
             "mxs": s_mx_small, "mx": s_mx, "comm": s_comm}
    for w in which:
        table[w]()
