"""ORACLE / TEST INFRASTRUCTURE.

``oracle.ref`` drives the unmodified reference library compiled into
``oracle/_ref``; ``oracle.restated`` is the CPU restatement of the hot path
(gmg_oracle.c).  Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's
CPU-baseline / ``--impl reference`` leg may import this package — the product
(``paper_1609_04809_b200``) never does.
"""
