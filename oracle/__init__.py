"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 / complex128 numpy implementation of what the LDBP hot
path computes, written from the paper (Häger & Pfister, arXiv 2010.14258; citations
``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n).  It shares no code
with the CUDA path (``paper_2010_14258_b200/``) and neither imports the other.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The product
path must never route through it.

Modules
  physics   units, L_eff, EDFA noise PSD, CD memory T_cd                (Eq. 15)
  steps     log step sizes, half-step merge, LS filter init, gamma' init (Example 1)
  channel   RRC shaping, asymmetric SSFM, EDFA, brick-wall LPF/decimate  (Eqs. 4-6, 11)
  ldbp      direct-form LDBP forward, adjoint, MSE, Adam, masks, gauges  (Eq. 7)
  receiver  matched filter + downsample, genie phase, effective SNR       (Eqs. 12-14)
  essm      learned enhanced SSM: filtered nonlinear steps + adjoint     (Eq. nl_filtered)

Pins: tests/test_oracle_*.py check every function against what the paper and mathematics fix
(worked examples in tests/golden/, closed forms, invariants, special cases, finite
differences).  Functions without such a pin say "parity unpinned" in their docstring.
"""
