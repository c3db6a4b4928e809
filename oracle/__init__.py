"""CPU oracle for the Fisher-BT likelihood engine — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or the
timed CPU baseline.  The product path (``paper_2601_11437_b200``) never imports
it and has no CPU fallback.

``oracle.maternmle_cpu`` restates the reference algorithm of arXiv 2601.11437's
``maternmle`` package in numpy/scipy, citing the reference file:line it follows.
Third-party arithmetic it shares with the reference: scipy.special ``kv`` /
``gamma`` / ``digamma`` and LAPACK ``dpotrf`` / ``dtrsm`` via scipy (scipy 1.18.1,
scipy-openblas 0.3.31.dev in this image; the reference pins only scipy>=1.10).
It is pinned against (a) the committed golden fixtures in ``tests/golden/``,
produced by the unmodified reference (``tests/golden/make_golden.py``), and
(b) the live reference package whenever ``/root/reference`` is present.
"""
