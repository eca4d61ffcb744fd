"""World-size-2 CPU test of the N > 1 host path over a real torch.distributed (gloo) group.

Each rank takes its token shard (tim.shard_range; sequences straddle the cut), computes its
exact partials with the oracle, packs them in the partial-block byte layout of include/tim.h
(tim_partial_header + n_seq x tim_seq_partial), exchanges the blocks with the product's
``exchange_partials`` and combines them: every rank must reproduce the single-process result
(§4.2 sequence rejection over whole trajectories) bit for bit.
"""
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import correct as oc


def _pack(glob, seq):
    m = struct.unpack("<Q", struct.pack("<d", glob["max_abs_delta"]))[0]

    def i128(v):
        v %= 1 << 128
        return [v & ((1 << 64) - 1), v >> 64]

    words = [glob["n_tok"], glob["n_resp_tok"], glob["n_truncated"], glob["n_tok_rejected"], glob["n_saturated"], m]
    words += i128(glob["sum_abs_delta"]) + i128(glob["sum_k1"]) + i128(glob["sum_k3"]) + [0, 0, 0, 0]
    for s in range(seq.shape[0]):
        words += i128(int(seq[s, 0])) + [int(seq[s, 1]), int(seq[s, 2])]
    raw = b"".join(struct.pack("<Q", w % (1 << 64)) for w in words)
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8)


def _unpack(raw: bytes, n_seq: int):
    w = struct.unpack(f"<{len(raw) // 8}Q", raw)

    def s64(x):
        return x - (1 << 64) if x >> 63 else x

    def i128(lo, hi):
        return lo + (s64(hi) << 64)

    glob = {"n_tok": s64(w[0]), "n_resp_tok": s64(w[1]), "n_truncated": s64(w[2]), "n_tok_rejected": s64(w[3]),
            "n_saturated": s64(w[4]), "max_abs_delta": struct.unpack("<d", struct.pack("<Q", w[5]))[0],
            "sum_abs_delta": i128(w[6], w[7]), "sum_k1": i128(w[8], w[9]), "sum_k3": i128(w[10], w[11])}
    seq = np.zeros((n_seq, 3), dtype=object)
    for s in range(n_seq):
        b = 16 + 4 * s
        seq[s] = [i128(w[b], w[b + 1]), s64(w[b + 2]), s64(w[b + 3])]
    return glob, seq


def _data():
    rng = np.random.default_rng(11)
    cu = np.array([0, 900, 1500, 1501, 3900, 5000, 5000, 7001])
    N = int(cu[-1])
    den = -np.abs(rng.normal(0, 2, N)).astype(np.float32)
    num = (den + rng.laplace(0, 3e-3, N) * (rng.random(N) < 0.5)).astype(np.float32)
    mask = (rng.random(N) < 0.85).astype(np.uint8)
    cfg = oc.Cfg(tis=True, tok_rs=True, log_tok_lo=np.log(0.9), log_tok_hi=np.log(1.1), seq_rs=oc.SEQ_K3,
                 seq_agg=oc.AGG_MEAN, tau_seq=1e-5)
    return cu, num, den, mask, cfg


def _worker(rank, world, port, q):
    from paper_2605_14220_b200 import tim
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cu, num, den, mask, cfg = _data()
        N = int(cu[-1])
        a, b = tim.shard_range(N, world, rank, align=1)
        _, g, s = oc.local_partials(num[a:b], den[a:b], cu, cfg, mask[a:b], a)
        block = _pack(g, s)
        gathered, P = tim.exchange_partials(block)
        assert P == world and gathered.numel() == world * block.numel()
        raw = gathered.numpy().tobytes()
        bb = block.numel()
        parts = [_unpack(raw[r * bb:(r + 1) * bb], len(cu) - 1) for r in range(world)]
        glob, seq = oc.combine(parts)
        keep, score = oc.decide(seq, cfg)
        stats = oc.finalize_stats(glob, keep, len(cu) - 1)
        full = oc.correct(num, den, cu, cfg, mask)
        ok = (np.array_equal(keep, full["seq_keep"]) and np.array_equal(score, full["seq_score"])
              and stats == full["stats"] and (seq == full["seq_partials"]).all())
        q.put((rank, bool(ok), int(keep.sum()), (a, b)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_two_rank_exchange_reproduces_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _, _ in res), res
    bounds = (0, 900, 1500, 1501, 3900, 5000, 7001)
    for r in range(world - 1):
        assert res[r][3][1] == res[r + 1][3][0]
    assert any(res[r][3][1] not in bounds for r in range(world - 1))   # a cut falls mid-sequence
    assert len({k for _, _, k, _ in res}) == 1
