"""CPU oracle for the structural-plasticity hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference algorithm (``sparsewire`` 0.1.0 under
``/root/reference/pkg/src/sparsewire``) in plain numpy / Python loops and, for
the heavy kernels, in plain C (``oracle/c/oracle.c``).  Every function cites
the reference ``file:line`` it follows.

Parity status: PINNED.  The restatement is checked against golden vectors
produced by running the real reference in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``) and against the
reference's own known-answer tests (``pkg/tests/test_rng.py:118-123`` etc.).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / CPU baseline.  The product package
``paper_2510_19764_b200`` never imports it and has no CPU fallback.
"""
