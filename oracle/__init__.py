"""CPU oracle for the RFT trainer loss path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2505_17826_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs use it, and only as the checker (or the timed CPU
baseline), never as the product path.

Parity status: PINNED.  ``tests/golden/*.npz`` were produced by
``tests/golden/make_golden.py``, which imports the reference (``triad``,
/root/reference/pkg/src) in the build container and runs its own
``group_loss`` / ``combine_reports`` / ``loss_sft`` / ``loss_dpo`` /
``regularizer_g``.  ``tests/test_oracle.py`` checks this oracle against every
fixture and against the reference tests' frozen known-answer values.
The north_star-only pieces (GRPO std, RLOO, PPO clip, k1/k2/k3/abs KL,
entropy bonus, token/sequence-mean aggregation) have no reference source; they
are pinned only through the exact reductions of SURVEY.md section 8c and by
finite differences (see tests/test_oracle.py).
"""
