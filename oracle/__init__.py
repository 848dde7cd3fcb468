"""CPU ORACLE — test infrastructure only, never part of the product path.

This package restates, on the CPU, the reference algorithm of the ExpertFlow
hot path (``moesim``, /root/reference/pkg/src/moesim) so that the B200
product in ``paper_2510_26730_b200`` can be checked against it.

Who may import it (enforced by review and by ``tests/test_layout.py``):
  * ``tests/`` — parity checker;
  * ``__graft_entry__.smoke()`` — one tiny parity check on cuda:0;
  * ``bench.py`` — only its ``cpu_baseline`` leg and the ``--impl reference``
    arm, which time this restatement on the host cores.

Pinning: every function cites the reference file:line it follows, and
``tests/test_oracle_golden.py`` checks the restatement against golden vectors
produced by the real reference (``tests/golden/make_golden.py`` imports
``moesim`` from /root/reference in the build container and writes JSON
fixtures) plus the published README CSV (``pkg/README.md:84-88``).  Decision
logic (routing sets, N_e, predictions, S, cache trace, event stream) is
therefore **parity pinned**.  Layer arithmetic (router GEMV, SwiGLU experts,
permute/combine) has no reference counterpart: its oracle in
``oracle/numerics.py`` is a float64 restatement of public model conventions
and is "parity unpinned" by the reference.
"""
