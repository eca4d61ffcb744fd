"""fp64 CPU oracle for the batch-invariant log-prob + TIS/RS hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2605_14220_b200``) never imports, calls or links
anything here, and this package never imports the product path: the two
share no code, constants or helpers.  Only ``synth`` (seeded input
generators, no method arithmetic) serves both.

Modules
  logprob  -- PAPER.md §2 / §4.1: per-token log-prob of the
              sampled id under the temperature-scaled softmax, and the entropy
              (SURVEY.md §8(c) C.1).  Plain definition in fp64.
  correct  -- PAPER.md §2 delta_t, §4.1 K1/K3, §4.2 r_corr,
              L_TIS, L_RS, S_seq, App. A.4: the
              decision-path arithmetic contract of SURVEY.md §8(c) C.3 written
              out step by step, masks, counts and statistics.
  exact    -- arbitrary-precision (mpmath / fractions) evaluations of the same
              real-number definitions, used only to pin the two modules above.

Parity status: every function is pinned by ``tests/test_oracle_*.py``
(closed forms, brute force, paper-printed Table 1 values, invariants).  No
function is "parity unpinned".
"""
