"""CPU checkers for the B200 decode path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import anything under ``oracle/``; the product package never does.

* ``plan_oracle``   -- exhaustive prefetch selection and exact-rational budget
                       re-derivation (restating the reference's
                       ``pkg/src/pipemax/oracle.py``), used to check the
                       scheduler's selectors.
* ``forward_ref``   -- fp32 numpy decode forward of the Llama / Qwen3 shapes
                       (HF semantics, see its header) -- the checker for the
                       sm_100a kernels.  PARITY UNPINNED by the reference: the
                       reference has no model math.
* ``kv_ref``        -- byte-level model of the paged, block-first KV pool
                       (append/gather/offload) used for bit-exact checks.
"""
