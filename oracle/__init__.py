"""CPU oracle for the PDHCG hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package; the shipped solver (paper_2506_06258_b200) never does.

* pdhcg_oracle.c — plain-C restatement of the reference's fused chunk
  (/root/reference/pkg/src/market_eq/kernels.py:22-145), bit-identical to it.
* solve.py — numpy restatement of the reference's restarted solve loop
  (driver.py:271-377, adaptive.py, kkt.py:29-87, exchange.py:75-156),
  driving the C chunk.  It issues the same numpy operations in the same
  order as the reference, so on the same instance it reproduces the
  reference's SolveReport bit for bit (pinned in tests/test_oracle.py
  against tests/golden/, which oracle/gen_golden.py produced by running
  the reference itself in the build container).
"""
