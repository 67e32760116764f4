"""TEST INFRASTRUCTURE ONLY — the CPU oracle for TeraPipe's hot path (arXiv 2102.07988).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import or execute anything in this package. The product path (paper_2102_07988_b200/) never
imports it and shares no code with it: the two meet only at the seeded inputs in synth/.

Contents:
  model.py  — plain fp64 numpy unsliced GPT forward/backward (Eq. 1-3) plus a
              step-by-step sliced reference of the same layer maths used to
              check invariant (a) on the CPU.
  plan.py   — Algorithm 1, the t_max enumeration with pruning and
              epsilon-thinning, brute force over all compositions, the closed
              form of Eq. 5 and a flow-shop schedule simulator.
  bf_compositions.c — the same brute force as plan.py, in plain C, for n = 32 units
              (2^31 compositions, the tiny config of BASELINE.json:7 at g = 1).

Parity status of each function is in its docstring and in DESIGN.md ("Oracle pins").
"""
