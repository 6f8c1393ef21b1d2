"""FP64 CPU oracle for the compressed FMM-FFT translation stage of
arXiv 2010.00520 (Qian & Yucel), written from /root/reference/PAPER.md.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import, call or
execute anything in this package.  The product (`paper_2010_00520_b200/`,
`include/`, the CUDA library) never imports it and shares no code with it.

Citations: `P:n` = PAPER.md line n.  Readings of ambiguous passages follow
SURVEY.md §8(c) and are listed in DESIGN.md ("Readings").

Modules
-------
fmm        direction grid, multipole count, eq. (7) operator, circulant grid, FFT
tensor     unfold / fold / i-mode product eq. (10) / mode-3 contraction eq. (12)
decomp     Alg. 1 Tucker-SVD, Alg. 2 H-Tucker-SVD, Alg. 3 TT-SVD, truncation rule
restore    dense eqs. (8), (9), (11), (13), (14) and the slice chains of Figs. 3-4
translate  eq. (5) by brute-force circular direct sum and by FP64 FFT; eq. (6) sum
memory     compressed-memory count
aggregate  eq. (4) aggregation and eq. (6) disaggregation around eq. (5)

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py; none is "parity unpinned".
"""
