"""CPU-only checks of the C ABI (no compute call needs a GPU here).

The library must load, export every symbol include/tim.h and include/tim_debug.h declare, and
reject bad arguments synchronously before touching the device (tim.h "Conventions").
"""
import ctypes
import math
import os
import re

import pytest

from paper_2605_14220_b200 import tim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("tim.h", "tim_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(tim_[a-z0-9_]+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def L():
    return tim.lib()


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert {"tim_logprob", "tim_mismatch_stats", "tim_correct", "tim_comm_init", "tim_comm_destroy",
            "tim_stats_finalize"} <= names
    for n in sorted(names):
        assert hasattr(L, n), n
        assert n in tim._SIGS, f"binding lacks a signature for {n}"


def test_version_and_strings(L):
    assert L.tim_abi_version() == 1
    for code in range(10):
        assert L.tim_status_string(code).decode().startswith(tim._STATUS[code])


def test_workspace_sizes(L):
    assert L.tim_logprob_vocab_slices(151936) == 64   # 594 tiles of 256 -> 64 slices of 9-10 tiles
    assert L.tim_logprob_vocab_slices(1024) == 4      # 4 tiles of 256 -> 4 slices
    assert L.tim_logprob_vocab_slices(1) == 1
    assert L.tim_logprob_workspace_bytes(1000, 2048, 151936) == 1024 + 64 * 1000 * 16
    # n_tok < 256 with n_tok % 128 in [1, 32]: + a zero-padded copy of H in whole 128-row boxes
    assert L.tim_logprob_workspace_bytes(20, 2048, 151936) == 1024 + 64 * 20 * 16 + 256 + 128 * 2048 * 2
    assert L.tim_logprob_workspace_bytes(130, 256, 1024) == 1024 + 4 * 130 * 16 + 256 + 256 * 256 * 2
    assert L.tim_logprob_workspace_bytes(100, 2048, 151936) == 1024 + 64 * 100 * 16
    assert L.tim_logprob_workspace_bytes(128, 2048, 151936) == 1024 + 64 * 128 * 16
    assert L.tim_logprob_workspace_bytes(300, 2048, 151936) == 1024 + 64 * 300 * 16
    assert L.tim_sample_workspace_bytes(1, 64, 1024) == 1024 + 2 * 4 * 16 + 256 + 128 * 64 * 2
    assert L.tim_correct_partial_bytes(5) == 128 + 5 * 32
    assert L.tim_correct_workspace_bytes(100, 5, 1) == 512 * 2
    assert L.tim_correct_workspace_bytes(100, 5, 4) == 512 * 5


P = ctypes.c_void_p


def _lp(L, hidden=P(4096), ld=256, weight=P(8192), d=256, V=1024, ids=P(16), n=10, T=1.0, out=P(32),
        ws=P(1 << 20), wsb=1 << 30):
    return L.tim_logprob(hidden, ld, weight, d, V, ids, n, T, None, out, None, ws, wsb, None, None)


def test_logprob_argument_errors_are_synchronous(L):
    assert _lp(L, hidden=None) == 1
    assert _lp(L, ids=None) == 1
    assert _lp(L, d=200, ld=200) == 2            # hidden % 64
    assert _lp(L, V=0) == 2
    assert _lp(L, n=-1) == 2
    assert _lp(L, ld=128) == 2                    # ld_hidden < hidden
    assert _lp(L, T=0.0) == 4 and _lp(L, T=float("nan")) == 4
    assert _lp(L, hidden=P(4104)) == 3            # not 16-B aligned
    assert _lp(L, ld=260) == 3                    # pitch*2 % 16
    assert _lp(L, n=0) == 0                       # empty batch: no launch
    assert _lp(L, wsb=100) == 5


def _bw(L, hidden=P(4096), weight=P(8192), d=256, V=1024, ids=P(16), n=10, T=1.0, gl=P(32), dh=P(64),
        dw=P(128), ws=P(1 << 20), wsb=1 << 40):
    return L.tim_head_backward(hidden, 256, weight, d, V, ids, n, T, None, gl, None, dh, dw, ws, wsb, None, None)


def test_head_backward_argument_errors_are_synchronous(L):
    assert _bw(L, dh=None, dw=None) == 1
    assert _bw(L, gl=None) == 1 and _bw(L, ids=None) == 1 and _bw(L, weight=None) == 1
    assert _bw(L, d=200) == 2 and _bw(L, V=0) == 2 and _bw(L, n=-1) == 2
    assert _bw(L, T=-1.0) == 4
    assert _bw(L, dh=P(68)) == 3 and _bw(L, ws=P(4096 + 16)) == 3
    assert _bw(L, wsb=1000) == 5
    assert _bw(L, n=0, dw=None) == 0                   # empty batch, dhidden only: nothing to do
    # saved-forward variants: the saved per-token values are required
    assert L.tim_head_backward_saved(P(4096), 256, P(8192), 256, 1024, P(16), 10, 1.0, None, None, P(256), P(32),
                                     None, P(64), P(128), P(1 << 20), 1 << 40, None, None) == 1
    assert L.tim_head_backward_saved(P(4096), 256, P(8192), 256, 1024, P(16), 10, 1.0, None, P(256), None, P(32),
                                     None, P(64), P(128), P(1 << 20), 1 << 40, None, None) == 1
    assert L.tim_logprob_saved(P(4096), 256, P(8192), 256, 1024, P(16), 10, 1.0, None, P(32), P(64), None,
                               P(1 << 20), 1 << 30, None, None) == 1
    # workspace: forward partials + 3 per-token vectors + one bf16 G block of <= 4 GiB
    nb = (1 << 32) // (2 * 151936) // 256 * 256
    assert nb == 14080
    assert L.tim_head_backward_workspace_bytes(100000, 2048, 151936) == \
        (1024 + 64 * nb * 16) + 3 * nb * 4 + nb * 151936 * 2
    assert L.tim_head_backward_workspace_bytes(1, 2048, 1000) == (1024 + 4 * 256 * 16) + 3 * 1024 + 256 * 1000 * 2


def _cfg(**kw):
    c = tim.CorrectConfig(**kw).to_c()
    return c


def test_correct_argument_errors_are_synchronous(L):
    c = _cfg(seq_rs=tim.SEQ_K3)
    args = dict(num=P(4096), den=P(8192), cu=P(16), S=2, tb=0, n=10, resp=None)

    def call(cfg=c, **kw):
        a = dict(args, **kw)
        return L.tim_correct_local(a["num"], a["den"], a["cu"], a["S"], a["tb"], a["n"], a["resp"],
                                   ctypes.byref(cfg) if cfg is not None else None, None, None, None,
                                   P(1 << 16), None, None)

    assert call(num=None) == 1
    assert call(cfg=None) == 1
    assert call(n=-3) == 2
    assert call(S=0) == 2
    assert call(num=P(4098)) == 3                 # fp32 array not 4-B aligned
    bad = _cfg(seq_rs=tim.SEQ_K3, tau_seq=2000.0)
    assert call(cfg=bad) == 4
    bad2 = _cfg(tok_rs=True, tok_lo=2.0, tok_hi=1.0)
    assert call(cfg=bad2) == 4
    bad3 = tim.CorrectCfgC(0, 0, 2, 0, 2.0, math.log(2), 0, 0, 1e-3)   # seq_rs = 2 is not a tim_seq_rs
    assert call(cfg=bad3) == 4


def test_stats_finalize_rounding(L):
    st = tim.StatsC()
    st.n_resp_tok = 3
    big = (1 << 90) + 12345
    st.sum_abs_delta_fx[0] = ctypes.c_int64(big & ((1 << 64) - 1) if big & (1 << 63) == 0 else (big & ((1 << 64) - 1)) - (1 << 64)).value
    st.sum_abs_delta_fx[1] = big >> 64
    neg = -(3 << 52) - 1
    st.sum_k1_fx[0] = ctypes.c_int64(neg).value
    st.sum_k1_fx[1] = -1
    assert L.tim_stats_finalize(ctypes.byref(st)) == 0
    assert st.mean_abs_delta == (float(big) * 2.0 ** -52) / 3
    assert st.mean_k1 == (float(neg) * 2.0 ** -52) / 3
    assert st.mean_k3 == 0.0


def test_shard_range_covers_tokens():
    for n in (0, 1, 255, 256, 1000, 262144, 8388609):
        for P_ in (1, 2, 3, 4, 8):
            cuts = [tim.shard_range(n, P_, r) for r in range(P_)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            for (a, b), (c, d) in zip(cuts[:-1], cuts[1:]):
                assert b == c and a <= b


def test_tp_vocab_ranges_partition_the_vocabulary():
    for V in (300, 1000, 4096, 151936, 152064):
        S = tim.lib().tim_logprob_vocab_slices(V)
        for tp in (1, 2, 4, 8):
            if S % tp:
                continue
            rs = [tim.tp_vocab_range(V, tp, r) for r in range(tp)]
            assert rs[0][0] == 0 and rs[-1][1] == V
            for (a, b), (c, d) in zip(rs[:-1], rs[1:]):
                assert b == c and a % 256 == 0 and a < b


def test_missing_library_fails_loudly():
    """No CPU fallback: without the built library every entry point raises (checked in a fresh
    interpreter whose TIM_LIBRARY points nowhere)."""
    import subprocess
    import sys
    code = ("from paper_2605_14220_b200 import tim\n"
            "try:\n    tim.lib()\nexcept RuntimeError as e:\n    print('raised', 'not built' in str(e))\n")
    env = dict(os.environ, TIM_LIBRARY=os.path.join(ROOT, "no_such_libtim.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert "raised True" in r.stdout, r.stdout + r.stderr


def test_debug_knobs_validate_arguments(L):
    """Performance knobs reject out-of-range values synchronously and accept their defaults."""
    assert L.tim_debug_set_pad_small(2) == 4 and L.tim_debug_set_pad_small(-1) == 4
    assert L.tim_debug_set_pad_small(1) == 0
    assert L.tim_debug_set_tuning(4, 2, 0, 4) == 4 and L.tim_debug_set_tuning(3, 2, 0, -1) == 4
    assert L.tim_debug_set_tuning(3, 2, 8, 4) == 4          # sleep bits 0..7
    assert L.tim_debug_set_tuning(3, 2, 0, 4) == 0          # the defaults
    assert L.tim_debug_set_kernel(2, 0) == 4 and L.tim_debug_set_kernel(1, -1) == 4
    assert L.tim_debug_set_kernel(1, 0) == 0


def test_tp_partial_rejects_a_shard_of_the_wrong_split():
    """a standard even vocab-parallel shard (V / tp rows) is not the fixed split of
    whole 256-row slices; the binding rejects it before any launch (no GPU needed)."""
    import torch
    from paper_2605_14220_b200 import tim
    V, tp, d = 151936, 8, 128
    b, e = tim.tp_vocab_range(V, tp, 0)
    assert (b, e) == (0, 18944)
    H = torch.zeros(4, d, dtype=torch.bfloat16)
    ids = torch.zeros(4, dtype=torch.int64)
    with pytest.raises(ValueError):
        tim.logprob_tp_partial(H, torch.zeros(V // tp, d, dtype=torch.bfloat16), V, tp, 0, ids)
    with pytest.raises(ValueError):
        tim.logprob_tp_partial(H, torch.zeros(e - b, d + 64, dtype=torch.bfloat16), V, tp, 0, ids)
    with pytest.raises(TypeError):
        tim.logprob_tp_partial(H, torch.zeros(e - b, d, dtype=torch.float32), V, tp, 0, ids)


def test_l2_persisting_rejects_negative_size_before_any_cuda_call(L):
    L.tim_l2_persisting.argtypes = [ctypes.c_int64, ctypes.c_void_p]
    assert L.tim_l2_persisting(-1, None) == 4     # TIM_ERR_VALUE, no device touched
