"""CPU checkers for the B200 decode path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import anything under ``oracle/``; the product package never does.

* ``plan_oracle``   -- exhaustive prefetch selection and exact-rational budget
                       re-derivation (restating the reference's
                       ``pkg/src/pipemax/oracle.py``), used to check the
                       scheduler's selectors.
* ``forward_ref``   -- fp32 numpy decode forward of the Llama / Qwen3 shapes
                       (HF semantics, see its header), one token at a time --
                       the checker for the sm_100a kernels at small shapes.
* ``forward_seq``   -- the same forward in matrix form over whole teacher-
                       forced sequences (fp32 torch, CPU or GPU), the checker
                       at real model shapes.
  The reference has no model math; both restatements are
  pinned to ``transformers`` 5.5.0's own Qwen3/Llama forward through the
  committed logits fixtures ``tests/golden/hf_*.npz``
  (``tests/golden/make_hf_golden.py``, ``tests/test_oracle_hf.py``).
"""
