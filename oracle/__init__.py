"""fp64 CPU oracle for the SART multi-branch decode hot path (arXiv 2505.13326).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path
(``paper_2505_13326_b200``) may import, call, link or execute anything under
``oracle/``.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it.

It is a plain, slow, obviously correct restatement of the paper:

* ``orderstats``  Lemma 1 and the expected stop length.
* ``philox``      Philox4x32-10 counter-based generator and the Gumbel-max
                  sampler (the paper says only "stochastic
                  sampling").
* ``model``       textbook pre-norm decoder step, softmax attention over
                  [shared prefix ; branch suffix], PRM head.
* ``engine``      Algorithm 1 with the two-phase pruning of
                  P:188-198, early stopping, the block allocator
                  and commitment admission (readings R23, R34),
                  majority vote / max-reward aggregation.

It shares no code with the CUDA path.  Inputs come from ``synth/``.

Parity pins: see tests/test_oracle_*.py.  Parts that are conventions rather
than mathematics -- the PRM head standing in for Qwen2.5-Math-PRM-7B, answer
extraction, free-stack order, the commitment policy -- are "parity unpinned"
beyond their invariants (DESIGN.md §Oracle pins).
"""
