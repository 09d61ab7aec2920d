"""CPU oracle for the tensor-parallel hot path — TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the algorithms the GPU path must reproduce:

* ``tp``      — SPEC.md:390-516 (tensor_parallel module): the five collectives,
                DistributedLinear forward/backward, dim-sharded DistributedEmbedding,
                distributed LayerNorm, attention / MLP / transformer layer in speed
                and memory modes, plan_replacement; plus the builder-defined
                vocab-parallel embedding and cross-entropy.
                fp64 torch CPU tensors, simulated ranks in ascending order
                (SPEC.md:509).
* ``philox``  — numpy Philox4x32-10 and the logical-coordinate dropout masks the
                kernels draw (bit-exact).
* ``philox_grid.c`` — C restatement of the same masks (oracle/Makefile ->
                libphilox_grid.so), so 24-layer oracle stacks draw their masks fast;
                tests/test_philox.py checks it against the numpy version.
* ``tpcheck``  — the SPEC's tensor-parallel invariant suite as a CLI
                (``python -m oracle.tpcheck``; JSON report, exit 5 on violation;
                ``--gpu`` adds the sm_100a kernels at T = 1).
The partition / topology / schedule rows need no restatement here: the reference
itself is importable in this container and tests/golden/make_golden.py generates
tests/golden/reference_golden.json from it, against which the product's vendored
copies are checked bit-exactly.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2111_05972_b200``) never does: it fails loudly if libsmpk.so is absent.

Parity pinning: the reference ships no tests (pkg/pyproject.toml:24-25 points at
a missing tests/ dir), so the TP rows are pinned by the SPEC's worked examples
and tolerances, which tests/test_oracle.py checks,
and the partition/topology/schedule rows by golden vectors generated from the
reference code itself (tests/golden/).
"""
