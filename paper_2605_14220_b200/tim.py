"""ctypes binding of libtim.so (include/tim.h).  Argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts torch
tensors into raw device pointers, picks the caller's current CUDA stream, sizes the
workspaces and maps status codes to exceptions.  Host tensors passed to ``logprob`` /
``correct`` are copied to the device first and results copied back (the end-to-end form
bench.py times), which is the only host<->device traffic this module issues.

Method: PAPER.md §2 (delta_t), §4.1 (P:349 recomputation, P:393 K1/K3), §4.2
(P:496-547 r_corr, L_TIS, L_RS, S_seq), App. A.4 (P:812-896 the four patch objectives,
tau_tok = 2, tau_seq = 0.001).
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("TIM_LIBRARY") or os.path.join(_HERE, "libtim.so")  # override: A/B builds

TIM_OK = 0
_STATUS = {0: "TIM_OK", 1: "TIM_ERR_NULL", 2: "TIM_ERR_SHAPE", 3: "TIM_ERR_ALIGN", 4: "TIM_ERR_VALUE",
           5: "TIM_ERR_WORKSPACE", 6: "TIM_ERR_CUDA", 7: "TIM_ERR_NCCL", 8: "TIM_ERR_UNSUPPORTED",
           9: "TIM_ERR_DATA"}
SEQ_NONE, SEQ_K1, SEQ_K3 = 0, 1, 3
AGG_SUM, AGG_MEAN = 0, 1


class TimError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str = ""):
        super().__init__(f"{where}: {_STATUS.get(code, code)} {msg}".strip())
        self.code = code


class CorrectCfgC(ctypes.Structure):
    _fields_ = [("tis", ctypes.c_int32), ("tok_rs", ctypes.c_int32), ("seq_rs", ctypes.c_int32),
                ("seq_agg", ctypes.c_int32), ("tis_cap", ctypes.c_double), ("log_tis_cap", ctypes.c_double),
                ("log_tok_lo", ctypes.c_double), ("log_tok_hi", ctypes.c_double), ("tau_seq", ctypes.c_double)]


class StatsC(ctypes.Structure):
    _fields_ = [("n_tok", ctypes.c_int64), ("n_resp_tok", ctypes.c_int64), ("n_seq", ctypes.c_int64),
                ("n_truncated", ctypes.c_int64), ("n_tok_rejected", ctypes.c_int64),
                ("n_seq_rejected", ctypes.c_int64), ("n_saturated", ctypes.c_int64),
                ("sum_abs_delta_fx", ctypes.c_int64 * 2), ("sum_k1_fx", ctypes.c_int64 * 2),
                ("sum_k3_fx", ctypes.c_int64 * 2), ("max_abs_delta", ctypes.c_double),
                ("mean_abs_delta", ctypes.c_double), ("mean_k1", ctypes.c_double), ("mean_k3", ctypes.c_double)]


STATS_BYTES = ctypes.sizeof(StatsC)  # 136
PARTIAL_HEADER_BYTES = 128
SEQ_PARTIAL_BYTES = 32

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F = ctypes.c_float
_SZ = ctypes.c_size_t

_SIGS = {
    "tim_status_string": (ctypes.c_char_p, [_I32]),
    "tim_abi_version": (ctypes.c_int, []),
    "tim_logprob_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_logprob_vocab_slices": (_I32, [_I32]),
    "tim_logprob": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, _F, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_sample_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_sample": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, ctypes.c_uint64, _F, _P, _P, _P, _P, _P, _SZ, _P,
                          _P]),
    "tim_stats_finalize": (_I32, [_P]),
    "tim_correct_workspace_bytes": (_SZ, [_I64, _I64, _I32]),
    "tim_mismatch_stats": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_correct": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_correct_partial_bytes": (_SZ, [_I64]),
    "tim_correct_local": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "tim_correct_finish": (_I32, [_P, _I32, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P]),
    "tim_tp_vocab_range": (_I32, [_I32, _I32, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "tim_l2_persisting": (_I32, [ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "tim_logprob_tp_partial_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_logprob_tp_partial": (_I32, [_P, _I64, _P, _I32, _I32, _I32, _I32, _P, _I64, _F, _P, _P, _P, _SZ, _P]),
    "tim_logprob_tp_merge": (_I32, [_P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_logprob_tp_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_logprob_tp": (_I32, [_P, _I64, _P, _I32, _I32, _P, _P, _I64, _F, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_rmsnorm": (_I32, [_P, _I64, _P, _F, _I32, _I64, _P, _P]),
    "tim_logprob_rmsnorm_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_logprob_rmsnorm": (_I32, [_P, _I64, _P, _F, _P, _I32, _I32, _P, _I64, _F, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_head_backward_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_head_backward": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, _F, _P, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_logprob_saved": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, _F, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "tim_head_backward_saved": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, _F, _P, _P, _P, _P, _P, _P, _P, _P,
                                       _SZ, _P, _P]),
    "tim_ppo_partial_bytes": (_SZ, [_I64, _I32]),
    "tim_ppo_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tim_ppo_loss": (_I32, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P,
                            _P]),
    "tim_ppo_local": (_I32, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "tim_ppo_finish": (_I32, [_P, _I32, _I64, _P, _P, _P, _P, _P]),
    "tim_ppo_stats_finalize": (_I32, [_P]),
    "tim_comm_unique_id": (_I32, [_P]),
    "tim_comm_init": (_I32, [_P, _I32, _I32, ctypes.POINTER(_P)]),
    "tim_comm_destroy": (_I32, [_P]),
    "tim_debug_logprob_logits": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, _P, _I64, _P, _P, _P, _SZ, _P]),
    "tim_debug_set_kernel": (_I32, [_I32, _I32]),
    "tim_debug_set_pad_small": (_I32, [_I32]),
    "tim_debug_set_tuning": (_I32, [_I32, _I32, _I32, _I32]),
    "tim_debug_set_schedule": (_I32, [_I32, _I32]),
    "tim_debug_set_cluster": (_I32, [_I32]),
    "tim_debug_set_gemm_slack": (_I32, [_I32]),
    "tim_debug_set_gemm_policy": (_I32, [_I32, _I32, _I32, _I32]),
    "tim_debug_set_die_groups": (_I32, [_I32]),
    "tim_debug_die_map": (_I32, [_P, _P]),
    "tim_debug_set_correct_split": (_I32, [_I32]),
}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load libtim.so (fails loudly: there is no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(_LIB_PATH):
                    raise RuntimeError(f"libtim.so not built ({_LIB_PATH}); run __graft_entry__.build()")
                L = ctypes.CDLL(_LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def _check(code: int, where: str):
    if code != TIM_OK:
        raise TimError(code, where, lib().tim_status_string(code).decode())


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def vocab_slices(vocab: int) -> int:
    return int(lib().tim_logprob_vocab_slices(vocab))


# ----------------------------------------------------------------------------------- workspaces --
_ws_cache: dict = {}


def _workspace(device, nbytes: int, tag: str) -> torch.Tensor:
    """Cached workspace per (device, CURRENT STREAM, tag).  Calls on different streams never share
    a buffer (the library's per-call header, progress counters and partials would race), and a
    buffer is allocated on -- and, when it grows, released to the caching allocator from -- the
    stream that uses it, so the reuse is stream-ordered."""
    stream = torch.cuda.current_stream(device)
    key = (str(device), stream.cuda_stream, tag)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(nbytes, 256) + 256, dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def new_status(device) -> torch.Tensor:
    """Zeroed device status word (tim_device_status, 16 B) as int64[2]: [code | reserved<<32, first_bad]."""
    return torch.zeros(2, dtype=torch.int64, device=device)


def read_status(st: torch.Tensor) -> tuple[int, int]:
    v = st.cpu().tolist()
    return int(v[0] & 0xFFFFFFFF), int(v[1])


# --------------------------------------------------------------------------------------- logprob --
def logprob(hidden: torch.Tensor, weight: torch.Tensor, ids: torch.Tensor, temperature: float = 1.0,
            temperatures: torch.Tensor | None = None, entropy: bool = True, out: tuple | None = None,
            status: torch.Tensor | None = None, device=None):
    """Per-token log pi(ids[t] | row t) and entropy (nats) -- tim_logprob.

    hidden [N, d] bf16 (rows may be strided), weight [V, d] bf16 contiguous, ids [N] int64.
    Host (CPU) inputs are copied to ``device`` and the results copied back.
    """
    host = not hidden.is_cuda
    dev = torch.device(device) if device is not None else (hidden.device if not host else torch.device("cuda"))
    if host and out is None and hidden.shape[0] >= 4 * _HOST_FIRST:
        return _logprob_from_host(hidden, weight, ids, temperature, temperatures, entropy, status, dev)
    if host:
        hidden = hidden.to(dev, non_blocking=True)
        ids = ids.to(dev, non_blocking=True)
        if temperatures is not None:
            temperatures = temperatures.to(dev, non_blocking=True)
    if not weight.is_cuda:
        weight = weight.to(dev, non_blocking=True)
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("hidden and weight must be bfloat16")
    if hidden.dim() != 2 or hidden.stride(1) != 1:
        raise ValueError("hidden must be [N, d] with unit inner stride")
    weight = weight.contiguous()
    ids = ids.to(torch.int64).contiguous()
    N, d = hidden.shape
    V = weight.shape[0]
    if weight.shape[1] != d or ids.numel() != N:
        raise ValueError(f"shape mismatch: hidden {tuple(hidden.shape)}, weight {tuple(weight.shape)}, ids {tuple(ids.shape)}")
    if temperatures is not None:
        temperatures = temperatures.to(torch.float32).contiguous()
    if out is None:
        lp = torch.empty(N, dtype=torch.float32, device=dev)
        ent = torch.empty(N, dtype=torch.float32, device=dev) if entropy else None
    else:
        lp, ent = out
    L = lib()
    wsb = L.tim_logprob_workspace_bytes(N, d, V)
    ws = _workspace(dev, wsb, "logprob")
    code = L.tim_logprob(_ptr(hidden), hidden.stride(0), _ptr(weight), d, V, _ptr(ids), N, float(temperature),
                         _ptr(temperatures), _ptr(lp), _ptr(ent), _ptr(ws), ws.numel(), _ptr(status), _stream(dev))
    _check(code, "tim_logprob")
    if host:
        lp = lp.to("cpu", non_blocking=False)
        ent = ent.to("cpu") if ent is not None else None
    return lp, ent


_HOST_CHUNK = int(os.environ.get("TIM_HOST_CHUNK", 524288))  # rows per host->device chunk (multiple of 256)
_HOST_FIRST = 8192           # the first chunks ramp up 8k, 16k, 32k: only a small copy is exposed
_copy_streams: dict = {}


def _logprob_from_host(hidden, weight, ids, temperature, temperatures, entropy, status, dev):
    """Host inputs: the H2D copy of chunk i + 1 (copy stream) overlaps tim_logprob on chunk i
    (caller's stream).  Rows are independent and the kernel is batch-invariant, so the chunked
    result is bit-identical to one call on the whole batch."""
    N, d = hidden.shape
    if not weight.is_cuda:
        weight = weight.to(dev, non_blocking=True)
    weight = weight.contiguous()
    cs = _copy_streams.get(str(dev))
    if cs is None:
        cs = _copy_streams[str(dev)] = torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)
    hd = torch.empty(N, d, dtype=torch.bfloat16, device=dev)
    ids_d = ids.to(dev, non_blocking=True).to(torch.int64)
    temps_d = temperatures.to(dev, non_blocking=True) if temperatures is not None else None
    cuts, a, step = [0], 0, _HOST_FIRST
    while a < N:
        a = min(N, a + step)
        cuts.append(a)
        step = min(2 * step, _HOST_CHUNK)
    evs = []
    cs.wait_stream(comp)
    with torch.cuda.stream(cs):
        for a, b in zip(cuts[:-1], cuts[1:]):
            hd[a:b].copy_(hidden[a:b], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            evs.append(e)
    lp = torch.empty(N, dtype=torch.float32, device=dev)
    ent = torch.empty(N, dtype=torch.float32, device=dev) if entropy else None
    for (a, b), e in zip(zip(cuts[:-1], cuts[1:]), evs):
        comp.wait_event(e)
        logprob(hd[a:b], weight, ids_d[a:b], temperature, temps_d[a:b] if temps_d is not None else None,
                entropy, out=(lp[a:b], ent[a:b] if ent is not None else None), status=status)
    return lp.cpu(), (ent.cpu() if ent is not None else None)


def sample(hidden: torch.Tensor, weight: torch.Tensor, row_keys: torch.Tensor, seed: int,
           temperature: float = 1.0, temperatures: torch.Tensor | None = None, entropy: bool = True,
           status: torch.Tensor | None = None):
    """Rollout-side twin -- tim_sample: Gumbel-max draw a_t ~ softmax(z_t / T) keyed by (seed,
    row_keys[t]); returns (ids int64, logp, entropy) with logp / entropy bit-identical to
    tim_logprob(ids)."""
    dev = hidden.device
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("hidden and weight must be bfloat16")
    if hidden.dim() != 2 or hidden.stride(1) != 1:
        raise ValueError("hidden must be [N, d] with unit inner stride")
    weight = weight.contiguous()
    N, d = hidden.shape
    V = weight.shape[0]
    row_keys = row_keys.to(device=dev, dtype=torch.int64).contiguous()
    if row_keys.numel() != N or weight.shape[1] != d:
        raise ValueError("shape mismatch")
    if temperatures is not None:
        temperatures = temperatures.to(device=dev, dtype=torch.float32).contiguous()
    ids = torch.empty(N, dtype=torch.int64, device=dev)
    lp = torch.empty(N, dtype=torch.float32, device=dev)
    ent = torch.empty(N, dtype=torch.float32, device=dev) if entropy else None
    L = lib()
    ws = _workspace(dev, L.tim_sample_workspace_bytes(N, d, V), "sample")
    _check(L.tim_sample(_ptr(hidden), hidden.stride(0), _ptr(weight), d, V, _ptr(row_keys), N,
                        ctypes.c_uint64(int(seed) % (1 << 64)), float(temperature), _ptr(temperatures), _ptr(ids),
                        _ptr(lp), _ptr(ent), _ptr(ws), ws.numel(), _ptr(status), _stream(dev)), "tim_sample")
    return ids, lp, ent


def l2_persisting(nbytes: int, device=None) -> int:
    """tim_l2_persisting: the device's persisting-L2 set-aside (application-level; see include/tim.h).
    Returns the granted size in bytes."""
    got = ctypes.c_int64(0)
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        _check(lib().tim_l2_persisting(int(nbytes), ctypes.byref(got)), "tim_l2_persisting")
    return int(got.value)


def tp_vocab_range(vocab: int, tp: int, rank: int) -> tuple[int, int]:
    """W rows [begin, end) owned by `rank` of a `tp`-way vocab-parallel head (whole slices)."""
    b, e = _I32(), _I32()
    _check(lib().tim_tp_vocab_range(vocab, tp, rank, ctypes.byref(b), ctypes.byref(e)), "tim_tp_vocab_range")
    return b.value, e.value


def logprob_tp_partial(hidden: torch.Tensor, weight_shard: torch.Tensor, vocab: int, tp: int, rank: int,
                       ids: torch.Tensor, temperature: float = 1.0, temperatures: torch.Tensor | None = None):
    """One rank of a vocab-parallel head: this rank's slice partials (uint8 block) -- tim_logprob_tp_partial."""
    dev = hidden.device
    N, d = hidden.shape
    b, e = tp_vocab_range(vocab, tp, rank)
    if hidden.dtype != torch.bfloat16 or weight_shard.dtype != torch.bfloat16:
        raise TypeError("hidden and weight_shard must be bfloat16")
    if weight_shard.dim() != 2 or weight_shard.shape[1] != d or weight_shard.shape[0] != e - b:
        raise ValueError(f"weight_shard must be W[{b}:{e}] ([{e - b}, {d}]: whole 256-row slices of the fixed "
                         f"split, tim_tp_vocab_range), got {tuple(weight_shard.shape)}")
    weight_shard = weight_shard.contiguous()
    ids = ids.to(device=dev, dtype=torch.int64).contiguous()
    if temperatures is not None:
        temperatures = temperatures.to(device=dev, dtype=torch.float32).contiguous()
    L = lib()
    part = torch.empty(max(1, int(L.tim_logprob_tp_partial_bytes(N, vocab, tp))), dtype=torch.uint8, device=dev)
    ws = _workspace(dev, 1024, "tp")
    _check(L.tim_logprob_tp_partial(_ptr(hidden), hidden.stride(0), _ptr(weight_shard), d, vocab, tp, rank, _ptr(ids),
                                    N, float(temperature), _ptr(temperatures), _ptr(part), _ptr(ws), ws.numel(),
                                    _stream(dev)), "tim_logprob_tp_partial")
    return part


def logprob_tp_merge(gathered: torch.Tensor, n_tok: int, vocab: int, ids: torch.Tensor,
                     temperatures: torch.Tensor | None = None, status: torch.Tensor | None = None):
    """Merge the all-gathered slice partials of every rank -- tim_logprob_tp_merge."""
    dev = gathered.device
    ids = ids.to(device=dev, dtype=torch.int64).contiguous()
    lp = torch.empty(n_tok, dtype=torch.float32, device=dev)
    ent = torch.empty(n_tok, dtype=torch.float32, device=dev)
    ws = _workspace(dev, 1024, "tp_merge")
    _check(lib().tim_logprob_tp_merge(_ptr(gathered), n_tok, vocab, _ptr(ids), _ptr(temperatures), _ptr(lp), _ptr(ent),
                                      _ptr(ws), ws.numel(), _ptr(status), _stream(dev)), "tim_logprob_tp_merge")
    return lp, ent


def logprob_tp(hidden: torch.Tensor, weight_shard: torch.Tensor, vocab: int, ids: torch.Tensor, comm: "Comm",
               temperature: float = 1.0, temperatures: torch.Tensor | None = None,
               status: torch.Tensor | None = None):
    """The whole vocab-parallel head over `comm` (tp = comm.nranks): this rank's slices, the NCCL
    all-gather of the slice partials inside libtim, the fixed-order merge -- tim_logprob_tp.  Every
    rank passes the same rows and gets logp / entropy of all of them, bitwise equal to logprob()."""
    dev = hidden.device
    N, d = hidden.shape
    tp, rank = comm.nranks, comm.rank
    b, e = tp_vocab_range(vocab, tp, rank)
    if hidden.dtype != torch.bfloat16 or weight_shard.dtype != torch.bfloat16:
        raise TypeError("hidden and weight_shard must be bfloat16")
    if weight_shard.dim() != 2 or weight_shard.shape[1] != d or weight_shard.shape[0] != e - b:
        raise ValueError(f"weight_shard must be W[{b}:{e}] ([{e - b}, {d}]: whole 256-row slices of the fixed "
                         f"split, tim_tp_vocab_range), got {tuple(weight_shard.shape)}")
    weight_shard = weight_shard.contiguous()
    ids = ids.to(device=dev, dtype=torch.int64).contiguous()
    if temperatures is not None:
        temperatures = temperatures.to(device=dev, dtype=torch.float32).contiguous()
    L = lib()
    lp = torch.empty(N, dtype=torch.float32, device=dev)
    ent = torch.empty(N, dtype=torch.float32, device=dev)
    ws = _workspace(dev, max(1024, int(L.tim_logprob_tp_workspace_bytes(N, vocab, tp))), "tp_full")
    _check(L.tim_logprob_tp(_ptr(hidden), hidden.stride(0), _ptr(weight_shard), d, vocab, comm.handle, _ptr(ids), N,
                            float(temperature), _ptr(temperatures), _ptr(lp), _ptr(ent), _ptr(ws), ws.numel(),
                            _ptr(status), _stream(dev)), "tim_logprob_tp")
    return lp, ent


def rmsnorm(hidden: torch.Tensor, gamma: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """Batch-invariant RMSNorm (HF Qwen3 semantics, bf16 in / out) -- tim_rmsnorm."""
    N, d = hidden.shape
    out = torch.empty(N, d, dtype=torch.bfloat16, device=hidden.device)
    gamma = gamma.to(device=hidden.device, dtype=torch.bfloat16).contiguous()
    _check(lib().tim_rmsnorm(_ptr(hidden), hidden.stride(0), _ptr(gamma), float(eps), d, N, _ptr(out),
                             _stream(hidden.device)), "tim_rmsnorm")
    return out


def logprob_rmsnorm(hidden: torch.Tensor, gamma: torch.Tensor, weight: torch.Tensor, ids: torch.Tensor,
                    eps: float = 1e-6, temperature: float = 1.0, temperatures: torch.Tensor | None = None,
                    status: torch.Tensor | None = None):
    """RMSNorm prologue + log-prob / entropy of the normalized rows -- tim_logprob_rmsnorm."""
    dev = hidden.device
    N, d = hidden.shape
    V = weight.shape[0]
    gamma = gamma.to(device=dev, dtype=torch.bfloat16).contiguous()
    weight = weight.contiguous()
    ids = ids.to(device=dev, dtype=torch.int64).contiguous()
    if temperatures is not None:
        temperatures = temperatures.to(device=dev, dtype=torch.float32).contiguous()
    lp = torch.empty(N, dtype=torch.float32, device=dev)
    ent = torch.empty(N, dtype=torch.float32, device=dev)
    L = lib()
    ws = _workspace(dev, L.tim_logprob_rmsnorm_workspace_bytes(N, d, V), "logprob_rmsnorm")
    _check(L.tim_logprob_rmsnorm(_ptr(hidden), hidden.stride(0), _ptr(gamma), float(eps), _ptr(weight), d, V,
                                 _ptr(ids), N, float(temperature), _ptr(temperatures), _ptr(lp), _ptr(ent), _ptr(ws),
                                 ws.numel(), _ptr(status), _stream(dev)), "tim_logprob_rmsnorm")
    return lp, ent


def logprob_saved(hidden: torch.Tensor, weight: torch.Tensor, ids: torch.Tensor, temperature: float = 1.0,
                  temperatures: torch.Tensor | None = None, status: torch.Tensor | None = None):
    """tim_logprob_saved: (logp, entropy, lse2) on the device; pass ``saved=(entropy, lse2)`` to
    head_backward to skip its forward pass."""
    dev = hidden.device
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("hidden and weight must be bfloat16")
    if hidden.dim() != 2 or hidden.stride(1) != 1:
        raise ValueError("hidden must be [N, d] with unit inner stride")
    weight = weight.contiguous()
    ids = ids.to(device=dev, dtype=torch.int64).contiguous()
    if temperatures is not None:
        temperatures = temperatures.to(device=dev, dtype=torch.float32).contiguous()
    N, d = hidden.shape
    V = weight.shape[0]
    if weight.shape[1] != d or ids.numel() != N:
        raise ValueError("shape mismatch")
    lp, ent, lse2 = (torch.empty(N, dtype=torch.float32, device=dev) for _ in range(3))
    L = lib()
    ws = _workspace(dev, L.tim_logprob_workspace_bytes(N, d, V), "logprob")
    _check(L.tim_logprob_saved(_ptr(hidden), hidden.stride(0), _ptr(weight), d, V, _ptr(ids), N, float(temperature),
                               _ptr(temperatures), _ptr(lp), _ptr(ent), _ptr(lse2), _ptr(ws), ws.numel(),
                               _ptr(status), _stream(dev)), "tim_logprob_saved")
    return lp, ent, lse2


def head_backward(hidden: torch.Tensor, weight: torch.Tensor, ids: torch.Tensor, grad_logp: torch.Tensor,
                  grad_entropy: torch.Tensor | None = None, temperature: float = 1.0,
                  temperatures: torch.Tensor | None = None, need_dhidden: bool = True, need_dweight: bool = True,
                  status: torch.Tensor | None = None, saved: tuple | None = None):
    """Backward of the head for L = sum_t grad_logp[t] logp_t + grad_entropy[t] H_t -- tim_head_backward,
    or tim_head_backward_saved when ``saved`` = (entropy, lse2) from logprob_saved on the same inputs.

    Returns (dhidden fp32 [N, d] or None, dweight fp32 [V, d] or None)."""
    dev = hidden.device
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("hidden and weight must be bfloat16")
    if hidden.dim() != 2 or hidden.stride(1) != 1:
        raise ValueError("hidden must be [N, d] with unit inner stride")
    weight = weight.contiguous()
    N, d = hidden.shape
    V = weight.shape[0]
    ids = ids.to(device=dev, dtype=torch.int64).contiguous()
    grad_logp = grad_logp.to(device=dev, dtype=torch.float32).contiguous()
    if grad_entropy is not None:
        grad_entropy = grad_entropy.to(device=dev, dtype=torch.float32).contiguous()
    if temperatures is not None:
        temperatures = temperatures.to(device=dev, dtype=torch.float32).contiguous()
    if ids.numel() != N or grad_logp.numel() != N or weight.shape[1] != d:
        raise ValueError("shape mismatch")
    dh = torch.empty(N, d, dtype=torch.float32, device=dev) if need_dhidden else None
    dw = torch.empty(V, d, dtype=torch.float32, device=dev) if need_dweight else None
    L = lib()
    ws = _workspace(dev, L.tim_head_backward_workspace_bytes(N, d, V), "head_backward")
    if saved is None:
        _check(L.tim_head_backward(_ptr(hidden), hidden.stride(0), _ptr(weight), d, V, _ptr(ids), N,
                                   float(temperature), _ptr(temperatures), _ptr(grad_logp), _ptr(grad_entropy),
                                   _ptr(dh), _ptr(dw), _ptr(ws), ws.numel(), _ptr(status), _stream(dev)),
               "tim_head_backward")
    else:
        ent, lse2 = (x.to(device=dev, dtype=torch.float32).contiguous() for x in saved)
        if ent.numel() != N or lse2.numel() != N:
            raise ValueError("saved (entropy, lse2) must have one value per token")
        _check(L.tim_head_backward_saved(_ptr(hidden), hidden.stride(0), _ptr(weight), d, V, _ptr(ids), N,
                                         float(temperature), _ptr(temperatures), _ptr(ent), _ptr(lse2),
                                         _ptr(grad_logp), _ptr(grad_entropy), _ptr(dh), _ptr(dw), _ptr(ws),
                                         ws.numel(), _ptr(status), _stream(dev)), "tim_head_backward_saved")
    return dh, dw


def debug_logits(hidden: torch.Tensor, weight: torch.Tensor, ids: torch.Tensor):
    """TEST ONLY (tim_debug.h): raw fp32 accumulators z = H W^T plus logp / entropy."""
    N, d = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    z = torch.full((N, V), float("nan"), dtype=torch.float32, device=dev)
    lp = torch.empty(N, dtype=torch.float32, device=dev)
    ent = torch.empty(N, dtype=torch.float32, device=dev)
    L = lib()
    ws = _workspace(dev, L.tim_logprob_workspace_bytes(N, d, V), "logprob")
    _check(L.tim_debug_logprob_logits(_ptr(hidden), hidden.stride(0), _ptr(weight), d, V, _ptr(ids), N, _ptr(z), V,
                                      _ptr(lp), _ptr(ent), _ptr(ws), ws.numel(), _stream(dev)), "tim_debug_logprob_logits")
    return z, lp, ent


def debug_set_tuning(h_policy: int = 0, w_policy: int = 0, sleep_waits: bool = False, sync_slack: int = 0):
    """Performance knobs (results unchanged): L2 policies for H / W loads, sleeping waits."""
    _check(lib().tim_debug_set_tuning(int(h_policy), int(w_policy), int(sleep_waits), int(sync_slack)),
           "tim_debug_set_tuning")


def debug_set_schedule(group: int = 0, demote: bool = False):
    """Schedule knobs (results unchanged): CTA pairs per M-tile group (0 = auto), L2 demotion."""
    _check(lib().tim_debug_set_schedule(int(group), int(demote)), "tim_debug_set_schedule")


def debug_set_cluster(pairs_per_cluster: int = 1):
    """Cluster shape knob (results unchanged): 2 = two CTA pairs sharing W through TMA multicast."""
    _check(lib().tim_debug_set_cluster(int(pairs_per_cluster)), "tim_debug_set_cluster")


def debug_set_gemm_slack(k_blocks: int = 128):
    """Head-backward GEMM progress gate (tim_debug_set_gemm_slack); never changes a result bit."""
    _check(lib().tim_debug_set_gemm_slack(int(k_blocks)), "tim_debug_set_gemm_slack")


def debug_set_gemm_policy(dh_a: int = 1, dh_b: int = 1, dw_a: int = 1, dw_b: int = 3):
    """Head-backward GEMM L2 policies (tim_debug_set_gemm_policy); never changes a result bit."""
    _check(lib().tim_debug_set_gemm_policy(int(dh_a), int(dh_b), int(dw_a), int(dw_b)), "tim_debug_set_gemm_policy")


def debug_set_die_groups(enable: bool = True):
    """Die-aware M-tile groups for G > 1 (tim_debug_set_die_groups); never changes a result bit."""
    _check(lib().tim_debug_set_die_groups(int(bool(enable))), "tim_debug_set_die_groups")


def debug_die_map():
    """(state, [die of SM s for s in 0..255]) from the per-device probe (tim_debug_die_map)."""
    st = ctypes.c_int32(0)
    mask = (ctypes.c_uint64 * 4)()
    _check(lib().tim_debug_die_map(ctypes.byref(st), mask), "tim_debug_die_map")
    return st.value, [(int(mask[s >> 6]) >> (s & 63)) & 1 for s in range(256)]


def debug_set_correct_split(split: bool = True):
    """P = 1 correction form (tim_debug_set_correct_split): True = the split local / finish / zero
    launches (default, the faster), False = one fused cooperative launch; never changes a result bit."""
    _check(lib().tim_debug_set_correct_split(int(bool(split))), "tim_debug_set_correct_split")


def debug_set_pad_small(enable: bool = True):
    """Small-batch H staging knob (tim_debug_set_pad_small); never changes a result bit."""
    _check(lib().tim_debug_set_pad_small(1 if enable else 0), "tim_debug_set_pad_small")


def debug_set_kernel(use_pair: bool = True, max_ctas: int = 0):
    """TEST ONLY: select the cta_group::2 (contract) or ::1 kernel and cap the persistent grid."""
    _check(lib().tim_debug_set_kernel(int(use_pair), int(max_ctas)), "tim_debug_set_kernel")


# -------------------------------------------------------------------------------- corrections --
@dataclasses.dataclass
class CorrectConfig:
    """tim_correct_cfg.  Paper values: tau_tok = 2, tau_seq = 0.001."""

    tis: bool = False
    tis_cap: float = 2.0
    tok_rs: bool = False
    tok_lo: float = 0.5
    tok_hi: float = 2.0
    seq_rs: int = SEQ_NONE
    seq_agg: int = AGG_SUM
    tau_seq: float = 1e-3

    def to_c(self) -> CorrectCfgC:
        return CorrectCfgC(int(self.tis), int(self.tok_rs), int(self.seq_rs), int(self.seq_agg),
                           float(self.tis_cap), math.log(self.tis_cap), math.log(self.tok_lo),
                           math.log(self.tok_hi), float(self.tau_seq))


# App. A.4.  The masking signal (num, den) is chosen by the caller:
# *-corr-ratio -> (train_old, rollout); *-ppo-ratio -> (current, rollout).
PRESETS = {
    "srs-k3-corr-ratio": CorrectConfig(seq_rs=SEQ_K3, seq_agg=AGG_SUM, tau_seq=1e-3),
    "srs-k3-ppo-ratio": CorrectConfig(seq_rs=SEQ_K3, seq_agg=AGG_SUM, tau_seq=1e-3),
    "tis-srs-k3-corr-ratio": CorrectConfig(tis=True, tis_cap=2.0, seq_rs=SEQ_K3, seq_agg=AGG_SUM, tau_seq=1e-3),
    "tis-srs-k1-corr-ratio": CorrectConfig(tis=True, tis_cap=2.0, seq_rs=SEQ_K1, seq_agg=AGG_SUM, tau_seq=1e-3),
}


def stats_from_bytes(raw: torch.Tensor) -> dict:
    """Host copy of a device tim_stats (uint8[136]) -> finalized dict (tim_stats_finalize)."""
    st = StatsC.from_buffer_copy(bytes(raw.cpu().numpy().tobytes()))
    _check(lib().tim_stats_finalize(ctypes.byref(st)), "tim_stats_finalize")

    def i128(a):
        return int(a[0]) % (1 << 64) + (int(a[1]) << 64)

    return {
        "n_tok": st.n_tok, "n_resp_tok": st.n_resp_tok, "n_seq": st.n_seq, "n_truncated": st.n_truncated,
        "n_tok_rejected": st.n_tok_rejected, "n_seq_rejected": st.n_seq_rejected, "n_saturated": st.n_saturated,
        "sum_abs_delta": i128(st.sum_abs_delta_fx), "sum_k1": i128(st.sum_k1_fx), "sum_k3": i128(st.sum_k3_fx),
        "max_abs_delta": st.max_abs_delta, "mean_abs_delta": st.mean_abs_delta, "mean_k1": st.mean_k1,
        "mean_k3": st.mean_k3,
    }


def _prep_correct(lp_num, lp_den, cu_seqlens, resp_mask, dev):
    """Every tensor argument is moved to `dev` (a no-op when already there): a host pointer must
    never reach a kernel, whatever mix of host and device tensors the caller passes."""
    host = not lp_num.is_cuda
    lp_num = lp_num.to(dev, non_blocking=True)
    lp_den = lp_den.to(dev, non_blocking=True)
    if resp_mask is not None:
        resp_mask = resp_mask.to(dev, non_blocking=True)
    cu_seqlens = cu_seqlens.to(dev, non_blocking=True)
    if lp_den.numel() != lp_num.numel() or (resp_mask is not None and resp_mask.numel() != lp_num.numel()):
        raise ValueError("lp_num, lp_den and resp_mask must have one value per token")
    lp_num = lp_num.to(torch.float32).contiguous()
    lp_den = lp_den.to(torch.float32).contiguous()
    cu_seqlens = cu_seqlens.to(torch.int64).contiguous()
    if resp_mask is not None:
        resp_mask = resp_mask.to(torch.uint8).contiguous()
    return host, lp_num, lp_den, cu_seqlens, resp_mask


def correct(lp_num: torch.Tensor, lp_den: torch.Tensor, cu_seqlens: torch.Tensor, cfg: CorrectConfig,
            resp_mask: torch.Tensor | None = None, tok_begin: int = 0, comm: "Comm | None" = None,
            status: torch.Tensor | None = None, return_stats: bool = True, device=None, out: dict | None = None):
    """TIS / token-RS / sequence-RS coefficients and statistics -- tim_correct.

    Returns dict(tis_w, tok_keep, seq_keep, coeff, seq_score, stats_raw[, stats]).  With
    ``return_stats`` the device stats are copied to the host (this synchronizes)."""
    dev = torch.device(device) if device is not None else (lp_num.device if lp_num.is_cuda else torch.device("cuda"))
    host, lp_num, lp_den, cu_seqlens, resp_mask = _prep_correct(lp_num, lp_den, cu_seqlens, resp_mask, dev)
    n = lp_num.numel()
    S = cu_seqlens.numel() - 1
    nranks = comm.nranks if comm is not None else 1
    if out is None:
        out = {
            "tis_w": torch.empty(n, dtype=torch.float32, device=dev),
            "tok_keep": torch.empty(n, dtype=torch.uint8, device=dev),
            "seq_keep": torch.empty(S, dtype=torch.uint8, device=dev),
            "coeff": torch.empty(n, dtype=torch.float32, device=dev),
            "seq_score": torch.empty(S, dtype=torch.float64, device=dev),
            "stats_raw": torch.zeros(STATS_BYTES, dtype=torch.uint8, device=dev),
        }
    L = lib()
    ws = _workspace(dev, L.tim_correct_workspace_bytes(n, S, nranks), "correct")
    c = cfg.to_c()
    code = L.tim_correct(_ptr(lp_num), _ptr(lp_den), _ptr(cu_seqlens), S, int(tok_begin), n, _ptr(resp_mask),
                         ctypes.byref(c), comm.handle if comm is not None else None, _ptr(out["tis_w"]),
                         _ptr(out["tok_keep"]), _ptr(out["seq_keep"]), _ptr(out["coeff"]), _ptr(out["seq_score"]),
                         _ptr(out["stats_raw"]), _ptr(ws), ws.numel(), _ptr(status), _stream(dev))
    _check(code, "tim_correct")
    res = dict(out)
    if return_stats:
        res["stats"] = stats_from_bytes(out["stats_raw"])
    if host:
        res = {k: (v.cpu() if isinstance(v, torch.Tensor) else v) for k, v in res.items()}
    return res


def mismatch_stats(lp_num, lp_den, cu_seqlens, resp_mask=None, tok_begin: int = 0, comm=None, status=None,
                   device=None) -> dict:
    """delta statistics only -- tim_mismatch_stats (synchronizes to return host values)."""
    dev = torch.device(device) if device is not None else (lp_num.device if lp_num.is_cuda else torch.device("cuda"))
    _, lp_num, lp_den, cu_seqlens, resp_mask = _prep_correct(lp_num, lp_den, cu_seqlens, resp_mask, dev)
    n = lp_num.numel()
    S = cu_seqlens.numel() - 1
    nranks = comm.nranks if comm is not None else 1
    L = lib()
    ws = _workspace(dev, L.tim_correct_workspace_bytes(n, S, nranks), "correct")
    raw = torch.zeros(STATS_BYTES, dtype=torch.uint8, device=dev)
    _check(L.tim_mismatch_stats(_ptr(lp_num), _ptr(lp_den), _ptr(cu_seqlens), S, int(tok_begin), n, _ptr(resp_mask),
                                comm.handle if comm is not None else None, _ptr(raw), _ptr(ws), ws.numel(),
                                _ptr(status), _stream(dev)), "tim_mismatch_stats")
    return stats_from_bytes(raw)


# ------------------------------------------------------------------------------ PPO (NEXT-2) --
class PpoCfgC(ctypes.Structure):
    _fields_ = [("clip_lo", ctypes.c_double), ("clip_hi", ctypes.c_double), ("hist_lo", ctypes.c_double),
                ("hist_inv_width", ctypes.c_double), ("hist_bins", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class PpoStatsC(ctypes.Structure):
    _fields_ = [("n_tok", ctypes.c_int64), ("n_contrib", ctypes.c_int64), ("n_clipped", ctypes.c_int64),
                ("n_zero_adv", ctypes.c_int64), ("n_saturated", ctypes.c_int64), ("n_seq", ctypes.c_int64),
                ("n_seq_contrib", ctypes.c_int64), ("sum_loss_fx", ctypes.c_int64 * 2),
                ("sum_k1_fx", ctypes.c_int64 * 2), ("sum_k3_fx", ctypes.c_int64 * 2), ("batch_loss", ctypes.c_double),
                ("clip_frac", ctypes.c_double), ("mean_k1", ctypes.c_double), ("mean_k3", ctypes.c_double)]


PPO_STATS_BYTES = ctypes.sizeof(PpoStatsC)


@dataclasses.dataclass
class PPOConfig:
    """tim_ppo_cfg: clip(r, 1 - eps, 1 + eps) (eq:ppo_loss) and the C(r) histogram range."""

    eps: float = 0.2
    hist_lo: float = -1.0
    hist_hi: float = 1.0
    hist_bins: int = 64

    def to_c(self) -> PpoCfgC:
        return PpoCfgC(1.0 - self.eps, 1.0 + self.eps, float(self.hist_lo),
                       self.hist_bins / (self.hist_hi - self.hist_lo), int(self.hist_bins), 0)


def ppo_stats_from_bytes(raw: torch.Tensor) -> dict:
    st = PpoStatsC.from_buffer_copy(bytes(raw.cpu().numpy().tobytes()))
    _check(lib().tim_ppo_stats_finalize(ctypes.byref(st)), "tim_ppo_stats_finalize")

    def i128(a):
        return int(a[0]) % (1 << 64) + (int(a[1]) << 64)

    return {"n_tok": st.n_tok, "n_contrib": st.n_contrib, "n_clipped": st.n_clipped, "n_zero_adv": st.n_zero_adv,
            "n_saturated": st.n_saturated, "n_seq": st.n_seq, "n_seq_contrib": st.n_seq_contrib,
            "sum_loss": i128(st.sum_loss_fx), "sum_k1": i128(st.sum_k1_fx), "sum_k3": i128(st.sum_k3_fx),
            "batch_loss": st.batch_loss, "clip_frac": st.clip_frac, "mean_k1": st.mean_k1, "mean_k3": st.mean_k3}


def ppo_loss(lp_cur: torch.Tensor, lp_old: torch.Tensor, advantages: torch.Tensor, cu_seqlens: torch.Tensor,
             cfg: PPOConfig, coeff: torch.Tensor | None = None, resp_mask: torch.Tensor | None = None,
             tok_begin: int = 0, comm: "Comm | None" = None, status: torch.Tensor | None = None,
             return_stats: bool = True):
    """Fused clipped surrogate + diagnostics -- tim_ppo_loss (device tensors)."""
    dev = lp_cur.device
    _, lp_cur, lp_old, cu_seqlens, resp_mask = _prep_correct(lp_cur, lp_old, cu_seqlens, resp_mask, dev)
    adv = advantages.to(device=dev, dtype=torch.float32).contiguous()
    if coeff is not None:
        coeff = coeff.to(device=dev, dtype=torch.float32).contiguous()
    n = lp_cur.numel()
    S = cu_seqlens.numel() - 1
    nranks = comm.nranks if comm is not None else 1
    c = cfg.to_c()
    out = {"loss": torch.empty(n, dtype=torch.float32, device=dev),
           "grad": torch.empty(n, dtype=torch.float32, device=dev),
           "clipped": torch.empty(n, dtype=torch.uint8, device=dev),
           "seq_loss": torch.empty(S, dtype=torch.float64, device=dev),
           "hist": torch.empty(2, cfg.hist_bins + 2, dtype=torch.int64, device=dev),
           "stats_raw": torch.zeros(PPO_STATS_BYTES, dtype=torch.uint8, device=dev)}
    L = lib()
    ws = _workspace(dev, L.tim_ppo_workspace_bytes(S, cfg.hist_bins, nranks), "ppo")
    _check(L.tim_ppo_loss(_ptr(lp_cur), _ptr(lp_old), _ptr(adv), _ptr(coeff), _ptr(resp_mask), _ptr(cu_seqlens), S,
                          int(tok_begin), n, ctypes.byref(c), comm.handle if comm is not None else None,
                          _ptr(out["loss"]), _ptr(out["grad"]), _ptr(out["clipped"]), _ptr(out["seq_loss"]),
                          _ptr(out["hist"]), _ptr(out["stats_raw"]), _ptr(ws), ws.numel(), _ptr(status),
                          _stream(dev)), "tim_ppo_loss")
    if return_stats:
        out["stats"] = ppo_stats_from_bytes(out["stats_raw"])
    return out


def ppo_local(lp_cur, lp_old, advantages, cu_seqlens, cfg: PPOConfig, coeff=None, resp_mask=None,
              tok_begin: int = 0, status=None):
    """Split form, pass 1 of tim_ppo_loss: per-token outputs + this rank's exact partial block."""
    dev = lp_cur.device
    _, lp_cur, lp_old, cu_seqlens, resp_mask = _prep_correct(lp_cur, lp_old, cu_seqlens, resp_mask, dev)
    adv = advantages.to(device=dev, dtype=torch.float32).contiguous()
    if coeff is not None:
        coeff = coeff.to(device=dev, dtype=torch.float32).contiguous()
    n = lp_cur.numel()
    S = cu_seqlens.numel() - 1
    c = cfg.to_c()
    out = {"loss": torch.empty(n, dtype=torch.float32, device=dev),
           "grad": torch.empty(n, dtype=torch.float32, device=dev),
           "clipped": torch.empty(n, dtype=torch.uint8, device=dev),
           "partial": torch.empty(int(lib().tim_ppo_partial_bytes(S, cfg.hist_bins)), dtype=torch.uint8, device=dev)}
    _check(lib().tim_ppo_local(_ptr(lp_cur), _ptr(lp_old), _ptr(adv), _ptr(coeff), _ptr(resp_mask), _ptr(cu_seqlens),
                               S, int(tok_begin), n, ctypes.byref(c), _ptr(out["loss"]), _ptr(out["grad"]),
                               _ptr(out["clipped"]), _ptr(out["partial"]), _ptr(status), _stream(dev)),
           "tim_ppo_local")
    return out


def ppo_finish(gathered: torch.Tensor, nranks: int, n_seq: int, cfg: PPOConfig):
    """Split form, pass 2: exact rank-ordered combine -> sequence losses, histogram, stats."""
    dev = gathered.device
    c = cfg.to_c()
    out = {"seq_loss": torch.empty(n_seq, dtype=torch.float64, device=dev),
           "hist": torch.empty(2, cfg.hist_bins + 2, dtype=torch.int64, device=dev),
           "stats_raw": torch.zeros(PPO_STATS_BYTES, dtype=torch.uint8, device=dev)}
    _check(lib().tim_ppo_finish(_ptr(gathered), int(nranks), int(n_seq), ctypes.byref(c), _ptr(out["seq_loss"]),
                                _ptr(out["hist"]), _ptr(out["stats_raw"]), _stream(dev)), "tim_ppo_finish")
    return out


def partial_bytes(n_seq: int) -> int:
    return int(lib().tim_correct_partial_bytes(n_seq))


def correct_local(lp_num, lp_den, cu_seqlens, cfg: CorrectConfig, resp_mask=None, tok_begin: int = 0,
                  status=None):
    """Split form, pass 1: per-token outputs + this rank's exact partial block (uint8 tensor)."""
    dev = lp_num.device
    _, lp_num, lp_den, cu_seqlens, resp_mask = _prep_correct(lp_num, lp_den, cu_seqlens, resp_mask, dev)
    n = lp_num.numel()
    S = cu_seqlens.numel() - 1
    tis_w = torch.empty(n, dtype=torch.float32, device=dev)
    tok_keep = torch.empty(n, dtype=torch.uint8, device=dev)
    coeff = torch.empty(n, dtype=torch.float32, device=dev)
    part = torch.empty(partial_bytes(S), dtype=torch.uint8, device=dev)
    c = cfg.to_c()
    _check(lib().tim_correct_local(_ptr(lp_num), _ptr(lp_den), _ptr(cu_seqlens), S, int(tok_begin), n,
                                   _ptr(resp_mask), ctypes.byref(c), _ptr(tis_w), _ptr(tok_keep), _ptr(coeff),
                                   _ptr(part), _ptr(status), _stream(dev)), "tim_correct_local")
    return {"tis_w": tis_w, "tok_keep": tok_keep, "coeff": coeff, "partial": part}


def exchange_partials(partial: torch.Tensor, group=None) -> tuple[torch.Tensor, int]:
    """All-gather every rank's partial block, in rank order, over torch.distributed (plumbing only:
    the blocks are exact integers, so any collective algorithm gives identical bits)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return partial, 1
    world = dist.get_world_size(group)
    if world == 1:
        return partial, 1
    if dist.get_backend(group) == "gloo":  # gloo lacks all_gather_into_tensor on some builds
        parts = [torch.empty_like(partial) for _ in range(world)]
        dist.all_gather(parts, partial, group=group)
        return torch.cat(parts), world
    gathered = torch.empty(world * partial.numel(), dtype=partial.dtype, device=partial.device)
    dist.all_gather_into_tensor(gathered, partial, group=group)
    return gathered, world


def correct_finish(gathered: torch.Tensor, nranks: int, cu_seqlens, cfg: CorrectConfig, coeff: torch.Tensor,
                   tok_begin: int = 0):
    """Split form, pass 2: exact combine, sequence decisions, coeff zeroing, stats."""
    dev = coeff.device
    cu = cu_seqlens.to(dev).to(torch.int64).contiguous()
    S = cu.numel() - 1
    seq_keep = torch.empty(S, dtype=torch.uint8, device=dev)
    seq_score = torch.empty(S, dtype=torch.float64, device=dev)
    raw = torch.zeros(STATS_BYTES, dtype=torch.uint8, device=dev)
    c = cfg.to_c()
    _check(lib().tim_correct_finish(_ptr(gathered), int(nranks), _ptr(cu), S, int(tok_begin), coeff.numel(),
                                    ctypes.byref(c), _ptr(coeff), _ptr(seq_keep), _ptr(seq_score), _ptr(raw),
                                    _stream(dev)), "tim_correct_finish")
    return {"seq_keep": seq_keep, "seq_score": seq_score, "stats_raw": raw}


def shard_range(n_tok: int, nranks: int, rank: int, align: int = 256) -> tuple[int, int]:
    """Token range [a, b) of `rank`: floor(r N / P) rounded down to `align` (balance only; correctness
    never depends on where the cut falls -- sequences may straddle ranks)."""
    if nranks < 1 or not (0 <= rank < nranks):
        raise ValueError("bad rank")

    def cut(r):
        if r >= nranks:
            return n_tok
        c = (r * n_tok) // nranks
        return min(n_tok, (c // align) * align)

    return cut(rank), cut(rank + 1)


class Comm:
    """NCCL communicator owned by libtim (tim_comm_init); bootstrap via torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib().tim_comm_unique_id(uid), "tim_comm_unique_id")
        obj = [bytes(uid.raw)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = ctypes.create_string_buffer(obj[0], 128)
        h = ctypes.c_void_p()
        _check(lib().tim_comm_init(uid, self.nranks, self.rank, ctypes.byref(h)), "tim_comm_init")
        self.handle = h

    def close(self):
        if self.handle:
            lib().tim_comm_destroy(self.handle)
            self.handle = None
