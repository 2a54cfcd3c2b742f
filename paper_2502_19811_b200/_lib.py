"""ctypes binding of libcomet_b200.so (include/comet_b200.h).

This is the only way the package reaches the GPU.  There is no CPU
fallback: if the library is missing or no CUDA device is visible, every
entry point raises ``NativeUnavailable`` (loudly, never silently computing
on the host).
"""

from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

from .config import ConfigurationError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcomet_b200.so")

COMET_OK, COMET_EINVAL, COMET_ECUDA, COMET_ECAP = 0, 1, 2, 3

ACTIVATIONS = {None: 0, "identity": 0, "none": 0, "relu": 1, "silu": 2, "gelu_tanh": 3, "gelu": 3, "tanh": 4}

META = {"rows": 0, "rows_pad": 1, "tiles0": 2, "pairs": 3, "pull": 4, "tiles1": 5, "chunks": 6, "combine_tok": 7}

# Exported symbols declared in include/comet_b200.h (checked by the CPU test suite).
EXPORTS = (
    "comet_last_error", "comet_version", "comet_ctx_create", "comet_ctx_destroy",
    "comet_symm_export", "comet_symm_import", "comet_link_local", "comet_token_buffer",
    "comet_routing_buffer", "comet_index_build", "comet_index_build_ex", "comet_index_sizes", "comet_index_download",
    "comet_signal_tokens_ready", "comet_layer0", "comet_layer1", "comet_layers", "comet_combine_finish", "comet_forward",
    "comet_hidden_buffer", "comet_yrows_buffer", "comet_hidden_rows_cap", "comet_device_info",
    "comet_timeline_enable", "comet_timeline_dump", "comet_router_topk", "comet_forward_host", "comet_forward_zerocopy",
    "comet_set_option", "comet_get_option", "comet_abort_waits", "comet_kernel_timing_enable",
    "comet_kernel_timing_read",
)

# Per-context kernel options (include/comet_b200.h COMET_OPT_*).
OPTIONS = {
    "fused": 0, "ksplit_max": 1, "split_tail0": 2, "split1": 3, "dedup": 4, "pull_local": 5, "fold_order": 6,
    "group1": 7, "chunk_rows": 8, "pdl": 9, "grid": 10, "fuse1": 11, "spin_timeout_ms": 12, "zc_dedup": 13,
    "zc_interleave": 14, "zc_download": 15, "zc_order": 16, "zc_fold_order": 17, "stream_fuse": 18, "sequential": 19,
    "streamk": 20, "fold_stride": 21,
}
OPT_DEFAULT = -2147483648
ROLES = ("load", "mma", "tmem_wait", "epilogue", "comm")


class NativeUnavailable(RuntimeError):
    """libcomet_b200.so is missing or cannot run (no sm_100a device)."""


class NativeError(RuntimeError):
    """A CUDA-side failure reported by the library."""


class CometConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("rank", "world", "tp", "ep", "device", "E", "topk", "N", "K", "m_cap")]


_P32 = ctypes.POINTER(ctypes.c_int32)


class CometIndexHost(ctypes.Structure):
    _fields_ = [("meta", ctypes.c_int32 * 16)] + [(n, _P32) for n in (
        "counts", "transfer", "row_off", "n_local", "row_token", "row_src",
        "tiles0", "tiles1", "chunks", "pairs0", "pull_token", "pull_src")]


_lib: Optional[ctypes.CDLL] = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library (no device needed) and declare every signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    vp, i32, c = ctypes.c_void_p, ctypes.c_int, ctypes
    sig = {
        "comet_last_error": ([], c.c_char_p),
        "comet_version": ([], i32),
        "comet_ctx_create": ([c.POINTER(CometConfig), c.POINTER(vp)], i32),
        "comet_ctx_destroy": ([vp], i32),
        "comet_symm_export": ([vp, vp], i32),
        "comet_symm_import": ([vp, vp], i32),
        "comet_link_local": ([c.POINTER(vp), i32], i32),
        "comet_token_buffer": ([vp], vp),
        "comet_routing_buffer": ([vp], vp),
        "comet_hidden_buffer": ([vp], vp),
        "comet_yrows_buffer": ([vp], vp),
        "comet_hidden_rows_cap": ([vp], c.c_int32),
        "comet_index_build": ([vp, vp, i32, i32, i32, vp], i32),
        "comet_index_build_ex": ([vp, vp, i32, i32, i32, i32, vp], i32),
        "comet_index_sizes": ([vp, _P32, vp], i32),
        "comet_index_download": ([vp, c.POINTER(CometIndexHost), vp], i32),
        "comet_signal_tokens_ready": ([vp, vp], i32),
        "comet_layer0": ([vp, vp, i32, i32, i32, vp], i32),
        "comet_layer1": ([vp, vp, vp, vp, i32, i32, vp], i32),
        "comet_combine_finish": ([vp, vp, vp], i32),
        "comet_layers": ([vp, vp, vp, vp, vp, i32, i32, i32, i32, vp], i32),
        "comet_forward": ([vp, vp, i32, vp, vp, vp, vp, i32, i32, i32, i32, i32, vp], i32),
        "comet_device_info": ([i32, _P32], i32),
        "comet_timeline_enable": ([vp, i32], i32),
        "comet_kernel_timing_enable": ([vp, i32], i32),
        "comet_kernel_timing_read": ([vp, vp, i32, vp], i32),
        "comet_timeline_dump": ([vp, vp, c.c_size_t], i32),
        "comet_router_topk": ([vp, i32, i32, i32, i32, i32, vp, vp, vp], i32),
        "comet_forward_host": ([vp, vp, vp, vp, vp, i32, vp, vp, i32, i32, i32, i32, i32, vp], i32),
        "comet_forward_zerocopy": ([vp, vp, vp, vp, vp, i32, vp, vp, i32, i32, i32, i32, vp], i32),
        "comet_set_option": ([vp, i32, i32], i32),
        "comet_get_option": ([vp, i32, c.POINTER(i32)], i32),
        "comet_abort_waits": ([i32], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == COMET_OK:
        return
    msg = load().comet_last_error().decode(errors="replace")
    if rc == COMET_EINVAL:
        raise ConfigurationError(msg)
    raise NativeError(f"libcomet_b200 error {rc}: {msg}")


def require_device():
    """Import torch and make sure a CUDA device is present (no fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the fused MoE layer runs only on sm_100a GPUs")
    load()
    return torch


def abort_waits(value: int = 1) -> None:
    """Make every device flag wait of this process trap at its next check
    (comet_abort_waits): for a watchdog that knows a peer rank is gone.
    ``abort_waits(0)`` clears it."""
    check(load().comet_abort_waits(int(value)))


def device_info(device: int = 0) -> Dict[str, int]:
    out = (ctypes.c_int32 * 4)()
    check(load().comet_device_info(device, out))
    return {"sms": out[0], "max_clusters": out[1], "cc": out[2], "smem": out[3]}


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


class Context:
    """One rank's native context (symmetric heap, index scratch, buffers)."""

    def __init__(self, *, rank: int, world: int, tp: int, ep: int, device: int,
                 E: int, topk: int, N: int, K: int, m_cap: int):
        self.torch = require_device()
        self.lib = load()
        self.cfg = CometConfig(rank, world, tp, ep, device, E, topk, N, K, m_cap)
        self.rank, self.world, self.tp, self.ep, self.device = rank, world, tp, ep, device
        self.E, self.topk, self.N, self.K, self.m_cap = E, topk, N, K, m_cap
        self.E_r = E // ep
        self.e_lo = (rank // tp) * self.E_r
        self.k_local = K // tp
        h = ctypes.c_void_p()
        check(self.lib.comet_ctx_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self.handle = h

    # -- lifetime ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.comet_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- options ------------------------------------------------------------
    def set_option(self, name: str, value) -> None:
        """Set a COMET_OPT_* option (None restores the library default)."""
        if name not in OPTIONS:
            raise ConfigurationError(f"unknown option {name!r}; choose from {sorted(OPTIONS)}")
        v = OPT_DEFAULT if value is None else int(value)
        check(self.lib.comet_set_option(self.handle, OPTIONS[name], v))

    def get_option(self, name: str) -> int:
        out = ctypes.c_int()
        check(self.lib.comet_get_option(self.handle, OPTIONS[name], ctypes.byref(out)))
        return out.value

    # -- buffers ------------------------------------------------------------
    def _view(self, ptr: int, shape, dtype):
        t = self.torch
        typestr = {t.bfloat16: "<f2", t.int32: "<i4", t.float32: "<f4"}[dtype]
        arr = t.as_tensor(_CudaArray(ptr, shape, typestr), device=f"cuda:{self.device}")
        return arr.view(dtype) if dtype == t.bfloat16 else arr

    def token_buffer(self):
        """[m_cap, N] bf16 token-slot buffer (symmetric)."""
        return self._view(self.lib.comet_token_buffer(self.handle), (self.m_cap, self.N), self.torch.bfloat16)

    def routing_buffer(self):
        return self._view(self.lib.comet_routing_buffer(self.handle), (self.m_cap * self.topk,), self.torch.int32)

    def hidden_buffer(self):
        rows = self.lib.comet_hidden_rows_cap(self.handle)
        return self._view(self.lib.comet_hidden_buffer(self.handle), (rows, self.k_local), self.torch.bfloat16)

    def yrows_buffer(self):
        rows = self.lib.comet_hidden_rows_cap(self.handle)
        return self._view(self.lib.comet_yrows_buffer(self.handle), (rows, self.N), self.torch.bfloat16)

    # -- symmetric heap -----------------------------------------------------
    def export_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(self.lib.comet_symm_export(self.handle, buf))
        return buf.raw

    def import_handles(self, handles: bytes) -> None:
        assert len(handles) == 64 * self.world
        check(self.lib.comet_symm_import(self.handle, ctypes.c_char_p(handles)))

    @staticmethod
    def link_local(ctxs) -> None:
        arr = (ctypes.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
        check(load().comet_link_local(arr, len(ctxs)))

    # -- index ----------------------------------------------------------------
    def _stream(self, stream=None) -> int:
        t = self.torch
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        return s.cuda_stream

    def index_build(self, experts_dev, M: int, tile_rows: int = 128, tile_cols: Optional[int] = None,
                    stream=None, flags: int = 3) -> None:
        """flags: bit0 reference tile lists, bit1 combine token list."""
        if tile_cols is None:  # reference default_tile_cols (resolver.py:35-39)
            tile_cols = 128 if self.N >= 512 else max(1, self.N // 4)
        check(self.lib.comet_index_build_ex(self.handle, ctypes.c_void_p(experts_dev.data_ptr()), M,
                                            tile_rows, tile_cols, flags, ctypes.c_void_p(self._stream(stream))))

    def index_meta(self, stream=None) -> np.ndarray:
        meta = (ctypes.c_int32 * 16)()
        check(self.lib.comet_index_sizes(self.handle, meta, ctypes.c_void_p(self._stream(stream))))
        return np.frombuffer(meta, dtype=np.int32).copy()

    def download_index(self, stream=None) -> Dict[str, np.ndarray]:
        """Host copy of the index in the oracle's flat form
        (oracle.moe_oracle.index_for_rank keys)."""
        m = self.index_meta(stream)
        n_rows, t0, t1, ch, pairs, pull = (int(m[META[k]]) for k in
                                           ("rows", "tiles0", "tiles1", "chunks", "pairs", "pull"))
        W = self.world
        bufs = {
            "counts": np.zeros(self.E, np.int32), "transfer": np.zeros(W * W, np.int32),
            "row_off": np.zeros(self.E_r + 1, np.int32), "n_local": np.zeros(self.E_r, np.int32),
            "row_token": np.zeros(max(n_rows, 1), np.int32), "row_src": np.zeros(max(n_rows, 1), np.int32),
            "tiles0": np.zeros(max(t0, 1) * 4, np.int32), "tiles1": np.zeros(max(t1, 1) * 6, np.int32),
            "chunks": np.zeros(max(ch, 1) * 4, np.int32), "pairs0": np.zeros(max(pairs, 1) * 4, np.int32),
            "pull_token": np.zeros(max(pull, 1), np.int32), "pull_src": np.zeros(max(pull, 1), np.int32),
        }
        h = CometIndexHost()
        for k, v in bufs.items():
            setattr(h, k, v.ctypes.data_as(_P32))
        check(self.lib.comet_index_download(self.handle, ctypes.byref(h), ctypes.c_void_p(self._stream(stream))))
        i64 = lambda a: a.astype(np.int64)  # noqa: E731
        return {
            "meta": np.frombuffer(h.meta, dtype=np.int32).copy(),
            "expert_counts": i64(bufs["counts"]),
            "transfer_counts": i64(bufs["transfer"]).reshape(W, W),
            "row_offsets": i64(bufs["row_off"]),
            "row_token": i64(bufs["row_token"][:n_rows]),
            "row_src": i64(bufs["row_src"][:n_rows]),
            "n_local": i64(bufs["n_local"]),
            "tiles0": i64(bufs["tiles0"][:t0 * 4]).reshape(t0, 4),
            "tiles1": i64(bufs["tiles1"][:t1 * 6]).reshape(t1, 6),
            "chunks": i64(bufs["chunks"][:ch * 4]).reshape(ch, 4),
            "pairs0": i64(bufs["pairs0"][:pairs * 4]).reshape(pairs, 4),
            "pull_token": i64(bufs["pull_token"][:pull]),
            "pull_src": i64(bufs["pull_src"][:pull]),
        }

    # -- layer ----------------------------------------------------------------
    def signal_tokens_ready(self, stream=None) -> None:
        check(self.lib.comet_signal_tokens_ready(self.handle, ctypes.c_void_p(self._stream(stream))))

    def layer0(self, w0t, activation: int = 0, n_comm: int = 2, group: int = 16, stream=None) -> None:
        check(self.lib.comet_layer0(self.handle, ctypes.c_void_p(w0t.data_ptr()), activation, n_comm, group,
                                    ctypes.c_void_p(self._stream(stream))))

    def layer1(self, w1t, combine_w, y_local, n_comm: int = 2, wave: int = 4, stream=None) -> None:
        cw = ctypes.c_void_p(combine_w.data_ptr()) if combine_w is not None else None
        check(self.lib.comet_layer1(self.handle, ctypes.c_void_p(w1t.data_ptr()), cw,
                                    ctypes.c_void_p(y_local.data_ptr()), n_comm, wave,
                                    ctypes.c_void_p(self._stream(stream))))

    def layers(self, w0t, w1t, combine_w, y_local, activation: int = 0, n_comm0: int = 2, group0: int = 4,
               wave1: int = 4, stream=None) -> None:
        """layer0 + layer1 in one persistent launch (comet_layers)."""
        cw = ctypes.c_void_p(combine_w.data_ptr()) if combine_w is not None else None
        check(self.lib.comet_layers(self.handle, ctypes.c_void_p(w0t.data_ptr()), ctypes.c_void_p(w1t.data_ptr()),
                                    cw, ctypes.c_void_p(y_local.data_ptr()), activation, n_comm0, group0, wave1,
                                    ctypes.c_void_p(self._stream(stream))))

    def forward_host(self, x_host, experts_host, combine_w_host, y_host, M: int, w0t, w1t, activation: int = 0,
                     n_comm0: int = 32, group0: int = 8, wave1: int = 4, chunks: int = 8, stream=None) -> None:
        """Streamed single-GPU forward on pinned host tensors (comet_forward_host)."""
        vp = ctypes.c_void_p
        check(self.lib.comet_forward_host(
            self.handle, vp(x_host.data_ptr()), vp(experts_host.data_ptr()),
            vp(combine_w_host.data_ptr()) if combine_w_host is not None else None, vp(y_host.data_ptr()), M,
            vp(w0t.data_ptr()), vp(w1t.data_ptr()), activation, n_comm0, group0, wave1, chunks,
            vp(self._stream(stream))))

    def forward_zerocopy(self, x_host, experts_host, combine_w_host, y_host, M: int, w0t, w1t, activation: int = 0,
                         n_comm0: int = 16, group0: int = 8, wave1: int = 4, stream=None) -> None:
        """Zero-copy single-GPU forward on pinned host tensors (comet_forward_zerocopy)."""
        vp = ctypes.c_void_p
        check(self.lib.comet_forward_zerocopy(
            self.handle, vp(x_host.data_ptr()), vp(experts_host.data_ptr()),
            vp(combine_w_host.data_ptr()) if combine_w_host is not None else None, vp(y_host.data_ptr()), M,
            vp(w0t.data_ptr()), vp(w1t.data_ptr()), activation, n_comm0, group0, wave1, vp(self._stream(stream))))

    def kernel_timing_enable(self, slots: int) -> None:
        """Bracket the next ``slots`` layer-kernel launches with CUDA events."""
        self._kt_slots = slots
        check(self.lib.comet_kernel_timing_enable(self.handle, slots))

    def kernel_timing_read(self):
        """Durations (ms) of the timed layer-kernel launches since enable/read."""
        cap = max(1, getattr(self, "_kt_slots", 0))
        buf = np.zeros(cap, dtype=np.float32)
        n = ctypes.c_int(0)
        check(self.lib.comet_kernel_timing_read(self.handle, buf.ctypes.data_as(ctypes.c_void_p), cap,
                                                ctypes.byref(n)))
        return buf[:n.value].tolist()

    def timeline_enable(self, cap: int) -> None:
        self._tl_cap = cap
        check(self.lib.comet_timeline_enable(self.handle, cap))

    def timeline_dump(self):
        """[(cta, role, task, start_ns, end_ns)] of the launches since enable/dump."""
        sms = device_info(self.device)["sms"]
        n = sms * len(ROLES) * self._tl_cap * 2
        buf = np.zeros(n, dtype=np.uint64)
        check(self.lib.comet_timeline_dump(self.handle, buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes))
        rec = buf.reshape(sms, len(ROLES), self._tl_cap, 2)
        out = []
        cta, role, idx = np.nonzero(rec[..., 1])
        for c, r, i in zip(cta.tolist(), role.tolist(), idx.tolist()):
            start, packed = int(rec[c, r, i, 0]), int(rec[c, r, i, 1])
            out.append((c, ROLES[r], (packed >> 40) - 1, start, start + (packed & ((1 << 40) - 1))))
        return out

    def combine_finish(self, y_local=None, stream=None) -> None:
        ptr = ctypes.c_void_p(y_local.data_ptr()) if y_local is not None else None
        check(self.lib.comet_combine_finish(self.handle, ptr, ctypes.c_void_p(self._stream(stream))))

    def forward(self, experts_dev, M: int, w0t, w1t, combine_w, y_local, activation: int = 0,
                n_comm0: int = 2, n_comm1: int = 2, group0: int = 16, wave1: int = 4, stream=None) -> None:
        cw = ctypes.c_void_p(combine_w.data_ptr()) if combine_w is not None else None
        check(self.lib.comet_forward(self.handle, ctypes.c_void_p(experts_dev.data_ptr()), M,
                                     ctypes.c_void_p(w0t.data_ptr()), ctypes.c_void_p(w1t.data_ptr()), cw,
                                     ctypes.c_void_p(y_local.data_ptr()), activation, n_comm0, n_comm1,
                                     group0, wave1, ctypes.c_void_p(self._stream(stream))))
