"""TEST INFRASTRUCTURE — the CPU oracle for the TEAL decode hot path.

Nothing under ``oracle/`` is part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg (and its
``--impl reference`` arm) may import it, and only as the checker / the timed
CPU reference — never as the thing measured on the GPU or shipped.

Contents
--------
* :mod:`oracle.actsparse_ref` — a numpy restatement of the reference
  algorithms on the path (``sparsify``, ``realized_sparsity``,
  ``sparsify_batched``, ``_skip_gemv``, ``matmul_dense``, ``traffic_model``,
  ``ActivationHistogram.record/threshold``, ``gaussian_threshold``, the block
  forward of ``model._forward`` and Algorithm 1 ``greedy_optimize``), each
  function citing the reference file:line it follows.
* ``oracle/teal_oracle.c`` — a plain-C restatement of ``_skip_gemv`` /
  ``_gemv_colmajor`` (single thread, fp32, ascending column order) used as the
  CPU baseline (``cpu_baseline.kind = "port"``); an OpenMP variant splits
  output rows across host threads (disjoint outputs, allowed by SPEC.md:502).

Pinning
-------
The restatement is pinned against golden vectors produced by the real
reference (``actsparse`` 0.1.0 imported from ``/root/reference/pkg/src`` in the
build container) by ``tests/golden/make_golden.py``; the fixtures live in
``tests/golden/*.npz`` and ``tests/test_oracle_golden.py`` checks the oracle
against them on CPU.
"""
