"""Float64 CPU oracle for arXiv 2507.09165 (PSD-cone projection by composite
polynomial filtering).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2507_09165_b200``) never imports this package and shares no code,
tables or helpers with it.

Every function follows a passage of the paper (``P:L<n>`` = line *n* of
``/root/reference/PAPER.md``; Doc C, lines 337-1205, is the authority) and is
written as the plain definition or the paper's algorithm step by step, in
float64, with numpy matmul / eigh as the only library primitives.

Modules
-------
tables    -- Tables 1-2 coefficients transcribed from the paper.
chain     -- Algorithm 2: bound, rescale, T stages, reconstruction.
certify   -- e_float certificate over every float32 in [-1,1],
             C kernel ``certify.c`` (plain loops, OpenMP).
remez     -- Algorithm 1 sequential Remez + App. A.
admm      -- the SDP consumer: three-step ADMM with the filter as Pi; the
             fused S/X update of psd_admm_update and the full iteration for the pins.
polar     -- the polar factor of a general square matrix by the same composite odd filter
             (f(A) = sum_j c_j A (A^T A)^j per stage).
spectral  -- Higham closed form via numpy eigh, spectral operator
             (P:L381-399), Hadamard-conjugated structured oracle for large n.

Parity pins: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against paper-printed values, closed forms,
invariants or a library routine.  None is "parity unpinned".
"""
