"""B200-native batch-invariant log-prob recomputation + TIS/RS corrections (arxiv 2605.14220).

The compute lives in ``libtim.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/tim.h``); ``paper_2605_14220_b200.tim`` is a thin ctypes binding that only
marshals torch tensors / streams into that ABI.  There is no CPU fallback: on a GPU box
the package fails loudly if the library is missing.
"""
from .tim import (  # noqa: F401
    CorrectConfig, Comm, TimError, PRESETS, PPOConfig, logprob, sample, correct, mismatch_stats, correct_local,
    ppo_loss, ppo_local, ppo_finish, rmsnorm, logprob_rmsnorm, head_backward, tp_vocab_range, logprob_tp_partial, logprob_tp_merge,
    correct_finish, exchange_partials, lib, library_path, shard_range, vocab_slices,
)
