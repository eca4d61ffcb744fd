"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no log-softmax, no ratio, no
TIS/RS rule). It only draws random hidden states, head weights, token ids,
sequence boundaries, response masks and log-prob perturbations with the
shapes and value distributions of the paper's workloads (SURVEY.md §8(d),
BASELINE.json ``configs``; App. A.1 ``tab:exp_setup`` P:710-729).

Every generator takes an explicit seed and returns torch tensors on the
requested device.  The oracle receives host copies; the CUDA path receives
device copies of the very same values.
"""
from __future__ import annotations

import dataclasses
import math

import torch

SEED_BASE = 20260000  # seed per config = 20260000 + config index


@dataclasses.dataclass(frozen=True)
class HeadConfig:
    """One BASELINE.json config (shape of an lm_head workload)."""

    name: str
    index: int          # position in BASELINE.json "configs" (seed offset)
    hidden: int         # d
    vocab: int          # V
    n_seq: int          # S
    seq_len: int        # tokens per sequence (prompt + response)
    prompt_len: int     # resp_mask == 0 on this prefix (tab:exp_setup)

    @property
    def n_tok(self) -> int:
        return self.n_seq * self.seq_len

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index


# BASELINE.json configs[0..3]; the sweep (configs[4]) reuses c1's shape.
CONFIGS = {
    "toy": HeadConfig("toy", 0, 256, 1024, 4, 64, 16),
    "c1": HeadConfig("c1", 1, 2048, 151936, 64, 4096, 1024),
    "c2": HeadConfig("c2", 2, 4096, 151936, 256, 8192, 1024),
    "c3": HeadConfig("c3", 3, 2048, 151936, 512, 16384, 2048),
}
SWEEP_INDEX = 4


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def head_weight(vocab: int, hidden: int, seed: int, device="cpu", sigma: float = 0.02) -> torch.Tensor:
    """W [V, d] bf16 ~ N(0, sigma^2) ("flat" mode)."""
    g = _gen(seed * 7 + 1, device)
    w = torch.randn(vocab, hidden, generator=g, device=device, dtype=torch.float32)
    return (w * sigma).to(torch.bfloat16)


def token_ids(n: int, vocab: int, seed: int, device="cpu", tail_frac: float = 0.01) -> torch.Tensor:
    """Uniform ids in [0, V); a fraction is forced into the last 256-wide vocab tile
    so the vocab-tail masking is exercised (SURVEY §8(d) "Ids")."""
    g = _gen(seed * 7 + 2, device)
    ids = torch.randint(0, vocab, (n,), generator=g, device=device, dtype=torch.int64)
    if n and tail_frac > 0:
        tail0 = ((vocab - 1) // 256) * 256
        pick = torch.rand(n, generator=g, device=device) < tail_frac
        tail = torch.randint(tail0, vocab, (n,), generator=g, device=device, dtype=torch.int64)
        ids = torch.where(pick, tail, ids)
    return ids


def hidden_states(n: int, hidden: int, seed: int, device="cpu", weight: torch.Tensor | None = None,
                  ids: torch.Tensor | None = None, mode: str = "flat", scale: float = 1.0,
                  target_sd: float = 2.5, chunk: int = 65536) -> torch.Tensor:
    """H [n, d] bf16.

    flat:   H = bf16(N(0,1))  (unit-RMS, like post-RMSNorm states)
    peaked: H_t = bf16(N(0,1) + beta_t * w_{a_t} / ||w_{a_t}||^2), beta_t = ln V + d*sigma^2/2 + l_t,
            l_t ~ N(0, target_sd^2): the target logit sits l_t above the background
            log-sum-exp, so most logp sit near 0 as in Table 1.
    """
    out = torch.empty(n, hidden, device=device, dtype=torch.bfloat16)
    g = _gen(seed * 7 + 3, device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        h = torch.randn(b - a, hidden, generator=g, device=device, dtype=torch.float32) * scale
        if mode == "peaked":
            assert weight is not None and ids is not None
            w = weight[ids[a:b].to(weight.device)].to(device=device, dtype=torch.float32)
            nrm2 = (w * w).sum(dim=1, keepdim=True).clamp_min(1e-30)
            vocab = weight.shape[0]
            sig2 = float((weight[: min(4096, vocab)].float() ** 2).mean())
            lt = torch.randn(b - a, 1, generator=g, device=device, dtype=torch.float32) * target_sd
            beta = math.log(vocab) + hidden * sig2 / 2.0 + lt
            h = h + beta * w / nrm2
        elif mode != "flat":
            raise ValueError(mode)
        out[a:b] = h.to(torch.bfloat16)
    return out


ROW_CHUNK = 65536  # rows per independently seeded chunk of a global batch (global_rows)


def global_rows(n_total: int, hidden: int, vocab: int, seed: int, a: int, b: int, weight: torch.Tensor,
                device="cpu", mode: str = "peaked") -> tuple[torch.Tensor, torch.Tensor]:
    """(H [b - a, d], ids [b - a]) = rows [a, b) of an n_total-row global batch in which every
    ROW_CHUNK-row chunk is drawn from its own seed, so any partition of the rows over ranks (a
    strong-scaling shard, a cut inside a sequence) reproduces exactly the same values."""
    if not (0 <= a <= b <= n_total):
        raise ValueError("bad row range")
    Hs, Is = [], []
    for c in range(a // ROW_CHUNK, (b - 1) // ROW_CHUNK + 1 if b > a else a // ROW_CHUNK):
        lo, hi = c * ROW_CHUNK, min(n_total, (c + 1) * ROW_CHUNK)
        sc = seed * 1009 + c
        idc = token_ids(hi - lo, vocab, sc, device=device)
        hc = hidden_states(hi - lo, hidden, sc, device=device, weight=weight, ids=idc, mode=mode)
        x0, x1 = max(a, lo) - lo, min(b, hi) - lo
        Hs.append(hc[x0:x1])
        Is.append(idc[x0:x1])
    if not Hs:
        return (torch.empty(0, hidden, dtype=torch.bfloat16, device=device),
                torch.empty(0, dtype=torch.int64, device=device))
    return torch.cat(Hs), torch.cat(Is)


def cu_seqlens(n_seq: int, seq_len: int, seed: int = 0, variable: bool = False, device="cpu") -> torch.Tensor:
    """int64 [S+1] prefix offsets; equal lengths, or L_s ~ U[L/8, L] when variable."""
    if variable:
        g = _gen(seed * 7 + 4, "cpu")
        lens = torch.randint(max(1, seq_len // 8), seq_len + 1, (n_seq,), generator=g, dtype=torch.int64)
    else:
        lens = torch.full((n_seq,), seq_len, dtype=torch.int64)
    cu = torch.zeros(n_seq + 1, dtype=torch.int64)
    cu[1:] = torch.cumsum(lens, 0)
    return cu.to(device)


def resp_mask(cu: torch.Tensor, prompt_len: int, device="cpu") -> torch.Tensor:
    """u8 [N]: 0 on the first prompt_len tokens of every sequence, 1 on the response."""
    cu = cu.cpu()
    n = int(cu[-1])
    m = torch.ones(n, dtype=torch.uint8)
    for s in range(cu.numel() - 1):
        a = int(cu[s])
        b = min(int(cu[s + 1]), a + prompt_len)
        m[a:b] = 0
    return m.to(device)


def perturb_bf16(lp: torch.Tensor) -> torch.Tensor:
    """P1: trainer log-prob = fp32(bf16_RNE(rollout log-prob))."""
    return lp.to(torch.bfloat16).to(torch.float32)


def perturb_hidden_ulp(H: torch.Tensor, p: float, seed: int) -> torch.Tensor:
    """P2: move random bf16 elements of H by one ulp (+-1 on the bit pattern) with probability
    p; the trainer side then re-scores the perturbed rows (an upstream-kernel
    style mismatch)."""
    g = _gen(seed * 7 + 7, H.device)
    bits = H.contiguous().view(torch.int16)
    flip = torch.rand(bits.shape, generator=g, device=H.device) < p
    step = torch.where(torch.rand(bits.shape, generator=g, device=H.device) < 0.5, -1, 1).to(torch.int16)
    return torch.where(flip, bits + step, bits).view(torch.bfloat16)


def perturb_laplace_mix(lp: torch.Tensor, seed: int, p_zero: float = 0.5, small: float = 2e-3,
                        p_big: float = 0.001, big: float = 0.25) -> torch.Tensor:
    """P3: delta = 0 w.p. p_zero, else Laplace(0, small) w.p. (1-p_zero-p_big), else
    Laplace(0, big) w.p. p_big; trainer log-prob clamped <= 0 (fig:delta_t_batch shape)."""
    g = _gen(seed * 7 + 5, lp.device)
    n = lp.numel()
    u = torch.rand(n, generator=g, device=lp.device)
    e = torch.empty(n, device=lp.device).exponential_(1.0, generator=g)
    sgn = torch.where(torch.rand(n, generator=g, device=lp.device) < 0.5, -1.0, 1.0)
    lap = sgn * e
    scale = torch.where(u < p_zero, torch.zeros_like(u),
                        torch.where(u < 1.0 - p_big, torch.full_like(u, small), torch.full_like(u, big)))
    return torch.clamp(lp + (lap * scale).to(lp.dtype), max=0.0)


def policy_move(lp: torch.Tensor, seed: int, sd: float = 0.01) -> torch.Tensor:
    """Synthetic current-policy log-prob (lp_cur) for the r_ppo masking signal (C4 grid)."""
    g = _gen(seed * 7 + 6, lp.device)
    return torch.clamp(lp + torch.randn(lp.shape, generator=g, device=lp.device) * sd, max=0.0)
