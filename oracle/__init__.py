"""ORACLE -- plain, slow, CPU reference for the implicit LISL/HJB step of arXiv:1605.04821.

THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import or execute anything here.
It shares no code with the CUDA path (`paper_1605_04821_b200/`); the only common dependency
is the seeded input generator `synth/`, which holds no method arithmetic.

Every function cites the PAPER.md passage it follows ("P:n" = PAPER.md line n).  Where the
paper is silent or ambiguous the reading is the one listed in DESIGN.md §3 (Readings).

Parity-pin status (see tests/test_oracle_*.py and DESIGN.md §4):
    scheme.truncation_mu / truncation_weights  pinned (worked examples, D4 identities)
    scheme.interp_weights                      pinned (affine exactness, partition of unity)
    scheme.lhat_rows / apply_operator          pinned (constants, quadratics closed form D5,
                                               1D closed form P:751-769, node-landing Laplacian)
    system.assemble                            pinned (M-matrix pattern, row sums, dense inverse)
    system.solve                               pinned (dense LU on tiny grids, residual)
    howard.control_search / howard_step        pinned (brute-force policy enumeration, Problem B ties)
    howard.march                               pinned (Table 4a / Table 4-B errors; O(h) rate)
    howard.control_search(idx=sample).R        the nonlinear-residual certificate R_j(U) on sampled rows
                                               (full-size GPU checks); pinned (D6 bound against the
                                               exact discrete solution, test_residual_certificate_bound)
"""
