"""CPU oracle for the MPML hot path of arXiv 2503.05533 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2503_05533_b200`` never imports it, and the two share no code: the
oracle is written from the paper (``/root/reference/PAPER.md``, cited as
``P:n``) and the readings listed in DESIGN.md section 3 (cited as ``Rk``).

Modules
-------
``oracle.c`` / ``core.py``  per-sample arithmetic in plain C (binary64 unless a
                            precision is being emulated): Philox RNG, KL field,
                            generic P1 element assembly, banded/dense Cholesky,
                            textbook MINRES, Algorithm 1 with emulated rounding.
``mlmc.py``                 estimators Eq. (3)/(4), the eps_l schedule
                            Eqs. (14)-(16), the N_l update and Algorithm 2.
``mg.py``                   NEXT-4: multigrid-preconditioned CG by the textbook
                            definitions (P1 prolongation, Galerkin P^T A P,
                            red-black Gauss-Seidel V(1,1)), numpy / scipy.sparse.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` (see DESIGN.md section 4 for the pin list).
"""
