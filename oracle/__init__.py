"""CPU oracle for the AMUSD draft/verify decode path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2410_17375_b200`` imports this package. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may use it, and only as the checker or the timed CPU
baseline -- never as the thing measured on the GPU path.

Contents
--------
specdec_oracle   restatement of the reference protocol (``pkg/src/specdec``):
                 splitmix64 hash-chain and agreement models, AR / sync-SD /
                 async (virtual-clock and threaded) engines, trace schema.
                 PINNED: checked bit-exactly against tests/golden/*.json, which
                 oracle/make_golden.py generates by running the unmodified
                 reference.
ref_decoder      numpy fp32 Llama-style decoder behind the same model
                 interface. PARITY UNPINNED: the reference contains no
                 transformer arithmetic; this is the
                 builder's own restatement of the public Llama-3 architecture.
"""
