"""CPU oracle for the SU(N) unfold of the GKSL master equation (arXiv:1812.11626).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_1812_11626_b200``) never imports it and has no CPU fallback.

The oracle shares no code with the CUDA path.  It computes the plain
definition (Eq. 1, basis P:135-144, Eq. 5, Eq. 9
P:194-198):

    Q_sm = Tr(F_s L(F_m)),   K_s = Tr(F_s L(I/N)),   s, m = 1..M,  M = N^2 - 1
    L(X) = -i[H, X] + sum_p gamma_p (L_p X L_p^+ - 1/2 {L_p^+ L_p, X})

so that dv/dt = Q v + K for rho = I/N + sum_j v_j F_j.

Modules
  basis      generators F_s (canonical order, R4/R5), Tr(F_s A)
             projection, brute-force f_mns / d_mns (Eq. 4).
  dense      O1: dense textbook evaluation of the trace definition (N <= 64).
  paper_eqs  the paper's own component formulas Eq. 6 (q_sn), Eq. 10 (r_sm,
             with the R1 reading) and Eq. 11 (k_s, with the R2 reading) from
             brute-force f, d -- used only to pin O1 to the paper's equations.
  gks        O3: the same trace definition for a generator given by a dense rate
             matrix A over the basis (Eq. 7), L_D(X) = sum_jk a_jk
             (F_j X F_k - 1/2 {F_k F_j, X}); the oracle of the batched dense unfold
             (SURVEY §8(f) F3).
  sparse     O2: the same trace definition with CSR operators, column by
             column (L(F_m) touches only the <= 2 matrix units of F_m, or the
             l+1 diagonal units of D^l), in plain C with OpenMP (sparse_o2.c).
             This is the timed CPU baseline.

Every function cites the PAPER.md line (P:n) it follows.  Pins (tests/
test_oracle_*.py, -m "not gpu"): N=2 Bloch equations, SU(3) Gell-Mann
structure constants, NZ_F / NZ_D closed forms of P:335, total (anti)symmetry
of f/d, orthonormality, the paper's Eqs. 6/10/11 with brute-force f/d,
trace preservation, rho-level apply check, O1 == O2.
"""
