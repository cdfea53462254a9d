"""CPU oracle for the bulk neighborhood-sampling triangle estimator (arXiv 1308.2166).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call,
link or execute anything in this package.  The product path
(``paper_1308_2166_b200``) never routes through it and shares no code with it.

Contents (each function cites the PAPER.md passage it follows):

* ``rng``        -- Philox4x32-10 counter-based generator and Lemire's unbiased
                    bounded integer; the fixed draw mapping of DESIGN.md
                    reading R7/R8 (the paper is silent on the RNG).
* ``nbsi``       -- the *conceptual* per-estimator algorithm of §4.2-§4.4
                    (PAPER.md:520-569, 742-767, 835-845), brute force over W.
* ``rankall``    -- literal rankAll (Lemma rank-all), scan with
                    resets (App. B), the rank definition
                     and the substream naming.
* ``exact``      -- ground truth: tau, Gamma_S(e), C(t) and an exact
                    rational enumeration of one estimator's outcome distribution.
* ``indexed``    -- ctypes front end of ``indexed.c``: the paper's *bulk* algorithm
                    (sort + scan-with-resets + multisearch by binary search),
                    OpenMP over estimators.  This is the oracle timed as the
                    CPU baseline.

* ``ed``         -- the event-driven mode (reading R17): the sequential
                    neighborhood-sampling rule per edge, with the two reservoir coins
                    replaced by skip-sampled replacement times; exact enumeration of its outcome law.
* ``edc``        -- ctypes front end of ``ed.c``: the same mode walked event by event per estimator
                    (OpenMP), the GPU event mode's parity oracle at full size.

The two oracles (``nbsi`` brute force, ``indexed.c`` bulk) are independent of
each other and are required to agree bit-for-bit; both are pinned by the tests
in ``tests/test_oracle_*.py``.
"""
