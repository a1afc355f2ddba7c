"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the GPU self-join
computes, written from PAPER.md (arxiv 1809.09930) and nothing else.  They
share no code with the CUDA path (`paper_1809_09930_b200/`) and never import
it.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything from here; the
product path must never route through it.

Modules
-------
brute  -- the definition (§3.1 "Problem Statement", l.104-110):
          nested-loop O(|D|^2) epsilon self-join, fp64, with the
          |d^2-eps^2| <= 1e-12 eps^2 ambiguity band split out.
grid   -- Algorithm 1 (§4.5, l.573-612) step by step: REORDER (§4.2),
          constructIndex over k of n dims (§3.2.1, §4.1), getAdjCells with
          binary search (§3.2.1, §5.6), calcDistancePts with SORTIDU (§4.3)
          and SHORTC (§4.4), batching arithmetic (§3.2.2), selectivity (§5.2),
          and the entity partitioning assignment (§6.2).

Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
