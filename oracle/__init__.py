"""oracle/ -- plain, slow, obviously-correct CPU implementations of what libpattn computes.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import anything under oracle/.  The
product path (paper_2511_11581_b200) never imports it, and nothing here imports
the product path: the two share no code.  Inputs come from `workloads/` (seeded
generators, no attention arithmetic) or from the tests themselves.

Modules
  attention  fp64 paged causal attention (Eq. 1/2; terminology P:304-317),
             C + OpenMP (pattn_oracle.c) behind ctypes.
  brute      the same definition in pure Python (math.fsum) for tiny inputs -- an
             independent second implementation used to pin `attention`.
  softmax    the paper's tiled softmax and segment merge in
             fp64 numpy, followed step by step.
  metadata   batch metadata / Q-block counts / sequence lookup / head mapping
             (P:171-178).

Pins: tests/test_oracle_pins.py, tests/test_oracle_softmax.py, tests/test_oracle_metadata.py.
Parity status of every function is listed in DESIGN.md §4 ("parity unpinned" rows: none).
"""
