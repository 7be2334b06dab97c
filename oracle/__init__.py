"""CPU ORACLE for the Nys-IP-PMM hot path (arXiv 2404.14524) — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 numpy/scipy implementations of what the CUDA path
computes, each function citing the PAPER.md passage it follows (P:n = PAPER.md line n,
S:n = SPEC.md line n, SURVEY §8(c) A-ids = the readings adopted where the paper is silent).

Rules:
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / --impl reference
    leg may import anything from this package.  The product path
    (`paper_2404_14524_b200`, `csrc/`) never imports, links or calls it.
  * It shares no code with the CUDA path: no kernels, helpers, constants or generators.
    Inputs come from `synth/` (seeded generators only); the counter-based Gaussian
    generator used for the sketch test matrix is re-implemented here independently
    (oracle/rng.py) from the one in csrc/.
  * No blocking, fusion or reordering beyond what the paper's formulas state.

Modules
  linops    normal-equation operator N_k + delta I
  nystrom   Alg. 1 randomized Nystrom approximation, Alg. 2 / eq. preconditioner
  pcg       textbook preconditioned CG
  ippmm     Alg. 3 / 4 / 5 Nys-IP-PMM for x >= 0 (App. B)
  rng       Philox4x32-10 + Box-Muller Gaussian test matrix Omega_k
  partial_chol  partial Cholesky preconditioner of Chol-IP-PMM
  active_set brute-force active-set enumeration for tiny QPs
  ssn       exact f* of a Q > 0 separable QP by dual semismooth Newton (independent pin, §8(c) P9)
  svm       config 2's A = [Xt, -Xt, I, -I] as an operator + the exact Woodbury path D (A23)
"""
