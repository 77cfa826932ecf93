"""CPU oracle for the pipeline hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product (paper_2412_14374_b200) never imports it:
its compute path is libpp200.so and it fails loudly without it.

Contents
  ffn.py  float64 numpy restatement of the reference's op interpreter and
          serial accumulation loop (pkg/src/pipecraft/executor.py:50-134) for
          the FFN vocabulary.  Pinned bit-for-bit against the reference's own
          golden fixture (pkg/tests/fixtures/golden_seed0.json) and against
          run_reference outputs generated here (tests/golden/numerics.json,
          tests/golden/make_golden.py).
  gpt.py  float64 numpy GPT-2 forward/backward (embedding, pre-LN block with
          causal attention and tanh-GELU MLP, tied LM head with summed
          cross-entropy) and the same serial accumulation loop.  The reference
          has no GPT ops, so this half is PARITY UNPINNED by the reference; it
          is pinned instead by central finite differences (tests/test_oracle.py,
          the reference's own FD method, pkg/tests/test_ir.py:32-49) and by
          torch.autograd float64 on the same inputs.
"""
