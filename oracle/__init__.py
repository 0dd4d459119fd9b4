"""CPU oracle for DiffPD's PD forward/backward hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 numpy/scipy implementation of what the path computes,
written from PAPER.md (arXiv 2101.05917).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with the CUDA
path (``paper_2101_05917_b200``) and never imports it; the only shared module
is ``pd_inputs`` (seeded inputs, no method arithmetic).

Modules
  fem      — trilinear hex shape gradients, G (x -> F), lumped mass M, A.
  energy   — corotated projection (polar via SVD), its derivative, muscle projection.
  pd       — y, local step, RHS d, objective g, grad g, PD forward (Alg. 1 for contact).
  adjoint  — A_N = A - dA assembled, direct adjoint solve, parameter gradients.

Every function cites the PAPER.md line (P:n) / equation label it follows;
readings where the paper is silent or garbled are SURVEY.md §8(c) items,
restated in DESIGN.md §2.  Pins: tests/test_oracle_*.py (``-m "not gpu"``).
Parity unpinned: full-horizon c5 (only a prefix is run on the host), and
absolute agreement with any paper number (no shared meshes).
"""
