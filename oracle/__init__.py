"""CPU oracle for the P2ENet + splat hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference ``splatforge`` algorithm (read-only mount,
``/root/reference/pkg/src/splatforge``) in plain numpy (``voxel.py``,
``net.py``, ``raster.py``) and C (``raster_oracle.c``, compiled by
``oracle/Makefile`` into ``oracle/_build/liboracle_raster.so``). Every function
cites the reference file:line it follows.

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` leg, and only as the checker or the timed
CPU baseline. The product path (``paper_2409_16504_b200``) never imports it and
has no CPU fallback.

Pinning: ``tests/golden/make_golden.py`` imports the real reference in the build
container and records its outputs (exact integer arrays, SHA-256 digests of the
float64 arrays, and the three frame KATs from
``pkg/frontend/fixtures/frames.json``); ``tests/test_oracle.py`` checks this
restatement against them bit-for-bit (integer/ordering/raster outputs) or to
1e-12 (BLAS-dependent network outputs).
"""
