"""CPU oracle for the randomized range finder / randomized SVD hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_0909_4061_b200/`` imports
this package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs may use it, and only as the checker
or as the timed CPU reference arm -- never as the product path.

See ``oracle/lowrank_oracle.py`` for the restatement (every function cites
the reference file:line it follows) and ``oracle/fixtures.py`` for the
seeded synthetic matrices of BASELINE.json's five configs.
"""
