"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (fp64) of what the hot
path of arxiv 2207.07847 ("PEGP/MSP") computes, written from PAPER.md alone.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import, call, link or execute
anything under ``oracle/``.  The product path (``paper_2207_07847_b200``)
never imports it and shares no code with it (no common kernels, headers,
helpers or constant generators); the two meet only through the seeded input
generators in ``inputs/``, which hold none of the method's arithmetic.

Module map (each function cites the PAPER.md passage it follows):

* ``graph``       -- §2.1  L_G = B^T W B, incidence, quadratic form
* ``aggregation`` -- §2.2  MWM aggregation (C: oracle/c/mwm_oracle.c),
                     prolongations P^l_{l-1}, P^l (Eq. def:P), composite P(mu)
* ``expansion``   -- §3.1 Eq. def:L_ell (L_G~), §3.2 PEGP H~ and L^-_mu,
                     §3.3 MSP T~, Theorem 3.1 lift / project
* ``precond``     -- Eq. graphL_precsys R ~ pseudo-inverse: R_X = P L_X^+ P^T
* ``pcg``         -- textbook preconditioned CG (§1 "Conjugate
                     Gradient (CG) method"; BASELINE north_star "PCG")
* ``spectral``    -- dense pencils for Lemma dim_G_tilde / upper / lower and
                     Theorem MSP_cond, Tables 1-2

Parity pins live in ``tests/test_oracle_*.py`` (run with ``-m "not gpu"``).
"""
