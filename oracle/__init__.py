"""ORACLE -- test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation (numpy / scipy) of what the
B200 hot path computes, written from PAPER.md (arxiv 1411.3923, Alexandersen & Lazarov,
"Robust topology optimisation of microstructural details without length scale separation
- using a spectral coarse basis preconditioner").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from this package.  The product path
(``paper_1411_3923_b200``) never imports it and shares no code with it; the only shared
module is ``workloads`` (seeded input generators, no method arithmetic).

Every function cites the PAPER.md line(s) / equation it follows.  Where the paper is
silent or ambiguous the reading taken is listed in DESIGN.md §"Readings" and referenced
here as R<n>.

Parity status: all functions are pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``)
against closed forms, invariants, brute force or paper-printed values; none is
"parity unpinned".
"""
